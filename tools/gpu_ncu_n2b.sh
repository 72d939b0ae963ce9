OUT=gpurun_out/${1:-r02ac}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/interact_n2 python bench.py $Q --steps 1 --warmup 3 --n-subdiv 2 --pi-kernel gather > $OUT/ncu_n2.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/interact_n1g python bench.py $Q --steps 1 --warmup 3 --pi-kernel gather > $OUT/ncu_n1g.log 2>&1
python tools/ncu_lines.py $OUT/interact_n2.ncu-rep 60 > $OUT/n2_lines.txt 2>&1
python tools/ncu_lines.py $OUT/interact_n1g.ncu-rep 60 > $OUT/n1g_lines.txt 2>&1
python tools/ncu_regions.py $OUT/interact_n1g.ncu-rep > $OUT/n1g_regions.txt 2>&1
rm -f $OUT/*.ncu-rep
