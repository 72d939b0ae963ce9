OUT=gpurun_out/${1:-e2e}; mkdir -p $OUT
Q="--no-cpu-baseline --collapsed-step 0 --fp64-steps 0 --steps 5 --pi-kernel paired"
for c in 4 8 16 32; do timeout 600 python bench.py $Q --e2e-chunks $c > $OUT/e2e_c$c.json 2>/dev/null; done
