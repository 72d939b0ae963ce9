# ncu --set full + per-source-line attribution of the interaction kernel: paired (n=1) and
# gather 384 (h/2 cells); only the summaries come back
OUT=gpurun_out/${1:-lines}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/paired python bench.py $Q --steps 1 --warmup 3 --pi-kernel paired > $OUT/ncu_paired.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/n2 python bench.py $Q --steps 1 --warmup 3 --n-subdiv 2 --pi-kernel gather > $OUT/ncu_n2.log 2>&1
for r in paired n2; do
  python tools/ncu_lines.py $OUT/$r.ncu-rep 70 > $OUT/${r}_lines.txt 2>&1
  python tools/ncu_regions.py $OUT/$r.ncu-rep > $OUT/${r}_regions.txt 2>&1
done
rm -f $OUT/*.ncu-rep
