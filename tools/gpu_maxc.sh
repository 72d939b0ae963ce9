OUT=gpurun_out/${1:-maxc}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 20"
for m in 1000 6 7 8; do
  SPHB_BLOCK_MAXC=$m timeout 600 python bench.py $Q --pi-kernel gather > $OUT/c3_gather_m$m.json 2>/dev/null
  SPHB_BLOCK_MAXC=$m timeout 600 python bench.py $Q --pi-kernel paired > $OUT/c3_paired_m$m.json 2>/dev/null
done
for m in 1000 12 13 14; do
  SPHB_BLOCK_MAXC=$m timeout 600 python bench.py $Q --pi-kernel gather --pi-block 384 --n-subdiv 2 > $OUT/c3n2_m$m.json 2>/dev/null
done
for m in 1000 6 8; do SPHB_BLOCK_MAXC=$m timeout 900 python tools/collapsed_bench.py 6000 30 384 > $OUT/collapsed_m$m.txt 2>&1; done
