#!/bin/bash
# One GPU-box pass: parity tests, default bench line, ncu launch list + one full k_interact capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh TAG [tests|bench|ncu ...]
set -u
TAG=${1:-run}; shift || true
WHAT=${*:-tests bench ncu full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
for w in $WHAT; do case $w in
tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log ;;
ref) timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/ref.err ;;
bench2) timeout 900 python bench.py --n-subdiv 2 --no-cpu-baseline > $OUT/bench_n2.json 2> $OUT/bench_n2.err ;;
ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
       --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_bench.log 2>&1 ;;
full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 1 \
       -o $OUT/interact python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_full.log 2>&1 ;;
nlsu) timeout 1200 ncu --set full --clock-control none --import-source on \
       -k "regex:k_reorder|k_integrate|k_radix|k_cell_keys|k_scan" -s 12 -c 10 \
       -o $OUT/nlsu python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_nlsu.log 2>&1 ;;
esac; done
ls -la $OUT
