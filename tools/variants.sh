set -u
mkdir -p gpurun_out/var
for v in "$@"; do
  make -s -C paper_1110_3711_b200/csrc clean >/dev/null; make -s -C paper_1110_3711_b200/csrc EXTRA="$v" > /dev/null 2>&1 || echo "build fail $v"
  echo "== $v" >> gpurun_out/var/res.txt
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'])" >> gpurun_out/var/res.txt 2>&1
done
