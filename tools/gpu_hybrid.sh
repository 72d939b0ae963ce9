# hybrid n = 1 blocking (SPHB_HYBRID_T): parity subset, then PI A/B at rest and collapsed
set -u
O=gpurun_out/hyb; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "blocking or production or pi384 or collapsed or drift or counters" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -2 $O/pytest.log
cat > /tmp/hyb_ab.py <<'PY'
import os, sys, subprocess
PY
for T in 0 32 48 64; do SPHB_HYBRID_T=$T python tools/pi_ab.py 1 0 20 gather/384,gather/256 > $O/rest_T$T.txt 2>&1; done
grep -H rest $O/rest_T*.txt
