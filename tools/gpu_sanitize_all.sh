OUT=gpurun_out/${1:-san}; mkdir -p $OUT
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_steps.py > $OUT/$t.txt 2>&1; echo rc=$? >> $OUT/$t.txt
done
