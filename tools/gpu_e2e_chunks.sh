# e2e (host round trip) throughput vs the number of pipelined row chunks, C3
set -u
O=gpurun_out/e2ec; mkdir -p $O
for c in 8 16 32 64; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --collapsed-step 0 --fp64-steps 0 \
    --e2e-steps 20 --e2e-chunks $c > $O/c$c.json 2> $O/c$c.err
  python -c "import json; d=json.loads(open('$O/c$c.json').read().strip().splitlines()[-1]); print($c, d['value']/1e6, d['e2e']['value']/1e6)"
done
