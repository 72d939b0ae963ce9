# X-slab checks on one GPU: compute-sanitizer over the step kernels (incl. the edge-band
# exchange through two virtual ranks) and the N-rank bench path with two gloo ranks
OUT=gpurun_out/${1:-r02q}; mkdir -p $OUT
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_steps.py > $OUT/memcheck.txt 2>&1; echo rc=$? >> $OUT/memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_steps.py > $OUT/racecheck.txt 2>&1; echo rc=$? >> $OUT/racecheck.txt
SPHB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/bench_n2_gloo.json 2> $OUT/bench_n2_gloo.err; echo rc=$? >> $OUT/bench_n2_gloo.err
