# same-box A/B of two prebuilt libraries: paper_1110_3711_b200/libsphb200_old.so vs the current one
set -u
O=gpurun_out/${1:-ablib}; mkdir -p $O
L=paper_1110_3711_b200
cp $L/libsphb200.so /tmp/libsphb200_new.so
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp $L/libsphb200_old.so $L/libsphb200.so; else cp /tmp/libsphb200_new.so $L/libsphb200.so; fi
    python tools/pi_ab.py 1 0 20 gather/384,paired/512 > $O/${v}_n1_$rep.txt 2>&1
    python tools/pi_ab.py 2 0 20 gather/384 > $O/${v}_n2_$rep.txt 2>&1
  done
done
cp /tmp/libsphb200_new.so $L/libsphb200.so
grep -H "rest" $O/*.txt
