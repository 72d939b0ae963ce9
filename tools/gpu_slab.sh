set -x
mkdir -p gpurun_out/r02p
timeout 900 python -m pytest tests -m gpu -x -q -k "slab" > gpurun_out/r02p/pytest_slab.log 2>&1; echo rc=$? >> gpurun_out/r02p/pytest_slab.log
timeout 600 python tools/slab_overhead.py c3 10 > gpurun_out/r02p/slab_overhead.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02p/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02p/pytest_gpu.log
