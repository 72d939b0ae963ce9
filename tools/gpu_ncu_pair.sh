# ncu --set full of the interaction kernel at C3: the h/2 gather (384 bricks) and the paired build (n=1)
OUT=gpurun_out/${1:-r02v}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/interact_n2 python bench.py $Q --steps 1 --warmup 3 --n-subdiv 2 --pi-kernel gather > $OUT/ncu_n2.log 2>&1
python tools/ncu_regions.py $OUT/interact_n2.ncu-rep > $OUT/interact_n2_regions.txt 2>&1; rm -f $OUT/interact_n2.ncu-rep
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
  -o $OUT/interact_paired python bench.py $Q --steps 1 --warmup 3 --pi-kernel paired > $OUT/ncu_paired.log 2>&1
python tools/ncu_regions.py $OUT/interact_paired.ncu-rep > $OUT/interact_paired_regions.txt 2>&1
