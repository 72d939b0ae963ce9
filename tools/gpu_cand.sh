set -u
O=gpurun_out/cand; mkdir -p $O
python tools/pi_ab.py 1 6000 10 gather/384,paired/512 > $O/n1.txt 2>&1
python tools/pi_ab.py 2 3000 10 gather/384 > $O/n2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -n 4 $O/n1.txt $O/n2.txt; tail -n 3 $O/pytest_gpu.log
