# h/2 gather 384 at rest: ncu --set full, every source line (for region sums)
OUT=gpurun_out/${1:-n2full}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/interact_n2 python bench.py $Q --steps 1 --warmup 3 --n-subdiv 2 --pi-kernel gather > $OUT/ncu_n2.log 2>&1
python tools/ncu_lines.py $OUT/interact_n2.ncu-rep 100000 > $OUT/n2_lines_all.txt 2>&1
ncu -i $OUT/interact_n2.ncu-rep --page source --csv --print-source sass > $OUT/n2_sass.csv 2>/dev/null
gzip -f $OUT/n2_sass.csv
rm -f $OUT/*.ncu-rep
