OUT=gpurun_out/${1:-c1}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 100 --config c1"
timeout 600 python bench.py $Q --pi-kernel gather --pi-block 128 > $OUT/c1_g128.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel gather --pi-block 256 > $OUT/c1_g256.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel gather --pi-block 384 > $OUT/c1_g384.json 2>/dev/null
timeout 600 python bench.py $Q --pi-kernel paired > $OUT/c1_paired.json 2>/dev/null
timeout 600 python bench.py $Q > $OUT/c1_tuned.json 2>/dev/null
