OUT=gpurun_out/${1:-tuned}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 600 python bench.py $Q --steps 100 --config c1 > $OUT/c1_tuned.json 2>/dev/null
timeout 600 python bench.py $Q --steps 30 > $OUT/c3_tuned.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
