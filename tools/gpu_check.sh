# quick bench legs + GPU tests + memcheck of the step kernels
OUT=gpurun_out/${1:-check}; mkdir -p $OUT
bash tools/gpu_quick.sh $1 tests
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_steps.py > $OUT/memcheck.txt 2>&1; echo rc=$? >> $OUT/memcheck.txt
