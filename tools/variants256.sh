set -u
mkdir -p gpurun_out/var256
for v in "$@"; do
  make -s -C paper_1110_3711_b200/csrc clean >/dev/null; make -s -C paper_1110_3711_b200/csrc EXTRA256="$v" > /dev/null 2>&1 || echo "build fail $v"
  echo "== $v" >> gpurun_out/var256/res.txt
  timeout 600 python tools/collapsed_bench.py 5000 200 256 >> gpurun_out/var256/res.txt 2>&1
done
