# Interaction blocking A/B over the BASELINE configurations at rest: ms/step, PI ms and the
# lane use of both builds.  bash tools/block_matrix.sh [configs...]
set -u
cfgs="${*:-c1 c2 c3 c4_1 c5}"
for c in $cfgs; do
  for pb in 128 384; do
    st=20; [ "$c" = c5 ] && st=6
    timeout 400 python bench.py --config $c --pi-block $pb --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $pb, round(d['ms_per_step'],3), round(d['stage_ms']['pi'],3), d['config'].get('pi_lane_use'))"
  done
done
