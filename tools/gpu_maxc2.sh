OUT=gpurun_out/${1:-maxc2}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 30"
timeout 600 python bench.py $Q --config c1 > $OUT/bench_c1.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel paired > $OUT/c3_paired.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel gather > $OUT/c3_gather.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel gather --pi-block 384 --n-subdiv 2 > $OUT/c3n2.json 2>/dev/null
timeout 900 python tools/collapsed_bench.py 6000 30 384 > $OUT/collapsed384.txt 2>&1
