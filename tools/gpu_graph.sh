OUT=gpurun_out/${1:-r02w}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 30"
timeout 600 python bench.py $Q --graph off > $OUT/c3_graph_off.json 2> $OUT/off.err
timeout 600 python bench.py $Q --graph on > $OUT/c3_graph_on.json 2> $OUT/on.err
timeout 600 python bench.py $Q --graph off > $OUT/c3_graph_off2.json 2> $OUT/off2.err
timeout 600 python bench.py $Q --graph on > $OUT/c3_graph_on2.json 2> $OUT/on2.err
