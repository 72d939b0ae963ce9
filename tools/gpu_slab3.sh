OUT=gpurun_out/${1:-r02aa}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "slab" > $OUT/pytest_slab.log 2>&1; echo rc=$? >> $OUT/pytest_slab.log
SPHB_DIST_BACKEND=gloo SPHB_SLAB_TRANSPORT=peer timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 0 > $OUT/bench_n2_peer.json 2> $OUT/bench_n2_peer.err; echo rc=$? >> $OUT/bench_n2_peer.err
