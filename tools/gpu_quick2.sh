# quick legs + the collapsed state (gather 384) + GPU tests
OUT=gpurun_out/${1:-quick2}; mkdir -p $OUT
bash tools/gpu_quick.sh $1 ${2:-}
timeout 900 python tools/collapsed_bench.py 6000 50 384 > $OUT/collapsed384.txt 2>&1
