OUT=gpurun_out/${1:-final2}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_bench_contract.py -m gpu -x -q > $OUT/pytest_bench.log 2>&1; echo rc=$? >> $OUT/pytest_bench.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
