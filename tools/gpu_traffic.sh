# DRAM bytes per launch of the interaction kernel (the bench's roofline.traffic), current builds
O=gpurun_out/${1:-traffic}; mkdir -p $O
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 1 --warmup 3"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:k_interact -s 2 -c 1 --csv python bench.py $Q --pi-kernel paired > $O/n1_paired.csv 2> $O/n1.err
timeout 900 ncu --metrics $M --clock-control none -k regex:k_interact -s 2 -c 1 --csv python bench.py $Q --n-subdiv 2 --pi-kernel gather > $O/n2_gather.csv 2> $O/n2.err
timeout 900 ncu --metrics $M --clock-control none -k regex:k_interact -s 2 -c 1 --csv python bench.py $Q --pi-kernel gather > $O/n1_gather.csv 2> $O/n1g.err
grep -h "dram__\|gpu__time" $O/*.csv
