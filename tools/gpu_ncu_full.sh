# one k_interact launch (C3 at rest, step 3): ncu --set full, every source line + the SASS page
# usage: gpu_ncu_full.sh OUTDIR "bench.py args"
OUT=gpurun_out/${1:-full}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/k python bench.py $Q --steps 1 --warmup 3 $2 > $OUT/ncu.log 2>&1
python tools/ncu_lines.py $OUT/k.ncu-rep 100000 > $OUT/lines_all.txt 2>&1
python tools/ncu_regions.py $OUT/k.ncu-rep > $OUT/regions.txt 2>&1
ncu -i $OUT/k.ncu-rep --page source --csv --print-source sass > $OUT/sass.csv 2>/dev/null
gzip -f $OUT/sass.csv
rm -f $OUT/*.ncu-rep
