OUT=gpurun_out/${1:-slab4}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "slab" > $OUT/pytest_slab.log 2>&1; echo rc=$? >> $OUT/pytest_slab.log
