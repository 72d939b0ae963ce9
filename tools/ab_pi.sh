#!/bin/bash
# A/B of interaction builds at C3 (quick bench legs, no CPU / e2e / collapsed / FP64 extras).
# Usage (under gpurun): bash tools/ab_pi.sh TAG "ARGS1" "ARGS2" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
k=0
for a in "$@"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --collapsed-step 0 \
    --fp64-steps 0 $a > $OUT/ab_$k.json 2> $OUT/ab_$k.err
  python - "$OUT/ab_$k.json" "$a" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} {d['value']/1e6:8.1f}M  ms {d['ms_per_step']:.3f}  pi {d['stage_ms']['pi']:.3f}  "
          f"lane {d['build'].get('pi_lane_use')}  frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  k=$((k+1))
done | tee $OUT/ab_summary.txt
