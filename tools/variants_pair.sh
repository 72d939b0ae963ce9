#!/bin/bash
# A/B of the paired interaction build (EXTRAP flags override the Makefile's -D values):
# bench.py --pi-kernel paired at C3 per variant, restoring the default build at the end.
# Usage (under gpurun): bash tools/variants_pair.sh TAG "" "-DV8_NG=3" ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
C=paper_1110_3711_b200/csrc
for v in "$@"; do
  rm -f $C/interact512p.o
  if ! make -s -C $C EXTRAP="$v" > $OUT/build.log 2>&1; then echo "build fail: $v" | tee -a $OUT/variants.txt; continue; fi
  regs=$(grep -A2 "v12ILb1ELb1ELb0" $C/interact512p.ptxas.log | grep -o "Used [0-9]* registers")
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --fp64-steps 0 \
    --collapsed-step ${COLLAPSED:-0} --pi-kernel paired 2> $OUT/err.txt | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
c = d.get('collapsed') or {}
print(f'{sys.argv[1]:44s} {sys.argv[2]:22s} {d[\"value\"]/1e6:7.1f}M pi {d[\"stage_ms\"][\"pi\"]:.3f} collapsed pi {c.get(\"stage_ms\", {}).get(\"pi\", 0):.3f}')
" "$v" "$regs" | tee -a $OUT/variants.txt
done
rm -f $C/interact512p.o; make -s -C $C > /dev/null 2>&1
