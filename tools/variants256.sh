# A/B of the 256-target interaction build (EXTRA256 flags): collapsed-state C3 (after 5000
# steps) and C3 at rest (bench, 256-target blocks forced).  bash tools/variants256.sh "" "-D..."
set -u
mkdir -p gpurun_out/var256
for v in "$@"; do
  make -s -C paper_1110_3711_b200/csrc clean >/dev/null; make -s -C paper_1110_3711_b200/csrc EXTRA256="$v" > /dev/null 2>&1 || echo "build fail $v"
  echo "== $v" >> gpurun_out/var256/res.txt
  timeout 600 python tools/collapsed_bench.py 5000 200 256 >> gpurun_out/var256/res.txt 2>&1
  timeout 300 python bench.py --pi-block 256 --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rest (256):', d['ms_per_step'], d['stage_ms']['pi'])" >> gpurun_out/var256/res.txt 2>&1
done
