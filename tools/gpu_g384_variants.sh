# gather-384 build variants (prebuilt libsphb200_v*.so) vs the shipped build, PI collapsed (step 6000)
set -u
O=gpurun_out/gv; mkdir -p $O
L=paper_1110_3711_b200
cp $L/libsphb200.so /tmp/base.so
for v in base A B C D; do
  if [ $v = base ]; then cp /tmp/base.so $L/libsphb200.so; else cp $L/libsphb200_v$v.so $L/libsphb200.so; fi
  python tools/pi_ab.py 1 6000 20 gather/384 2>&1 | grep -E "rest|step6000" | sed "s/^/$v /" >> $O/res.txt
done
cp /tmp/base.so $L/libsphb200.so
cat $O/res.txt
