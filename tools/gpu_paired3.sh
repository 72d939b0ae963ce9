OUT=gpurun_out/${1:-p3}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 30 --pi-kernel paired"
for r in 1 2 3; do timeout 600 python bench.py $Q > $OUT/paired_$r.json 2>/dev/null; done
