OUT=gpurun_out/${1:-cfg}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 30"
for c in c1 c2 c4_1 c5; do timeout 900 python bench.py $Q --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
