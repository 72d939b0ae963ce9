# Round-end style pass: default bench line (all legs), h/2 bench, reference arm, ncu launch list,
# the 1-rank slab path through torchrun, smoke
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --n-subdiv 2 --no-cpu-baseline --collapsed-step 0 --fp64-steps 0 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --slab-path --no-cpu-baseline --e2e-steps 0 > $OUT/bench_slab1.json 2> $OUT/bench_slab1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 > $OUT/ncu_bench.log 2>&1
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches.txt 2>&1
