# quick C3 legs: gather (n=1), gather n=2 (384), paired (n=1); then the GPU tests
OUT=gpurun_out/${1:-quick}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 20"
timeout 600 python bench.py $Q --pi-kernel gather > $OUT/c3_gather.json 2> $OUT/c3_gather.err
timeout 600 python bench.py $Q --pi-kernel gather --pi-block 384 --n-subdiv 2 > $OUT/c3n2_gather384.json 2> $OUT/c3n2.err
timeout 600 python bench.py $Q --pi-kernel paired > $OUT/c3_paired.json 2> $OUT/c3_paired.err
if [ "${2:-}" = tests ]; then timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log; fi
