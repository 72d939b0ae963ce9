# A/B of the 384-target interaction build (EXTRAL flags): collapsed-state C3 (after 5000
# steps) and C3 at rest (bench, 384-target blocks forced).  bash tools/variants_large.sh "" "-D..."
set -u
mkdir -p gpurun_out/varL
for v in "$@"; do
  make -s -C paper_1110_3711_b200/csrc clean >/dev/null; make -s -C paper_1110_3711_b200/csrc EXTRAL="$v" > /dev/null 2>&1 || echo "build fail $v"
  echo "== $v" >> gpurun_out/varL/res.txt
  timeout 600 python tools/collapsed_bench.py 5000 200 384 >> gpurun_out/varL/res.txt 2>&1
  timeout 300 python bench.py --pi-block 384 --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rest (384):', d['ms_per_step'], d['stage_ms']['pi'])" >> gpurun_out/varL/res.txt 2>&1
done
