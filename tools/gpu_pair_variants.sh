# paired-kernel build variants (prebuilt libsphb200_v*.so) vs the shipped build, PI at rest
set -u
O=gpurun_out/pv; mkdir -p $O
L=paper_1110_3711_b200
cp $L/libsphb200.so /tmp/base.so
for rep in 1 2; do
  for v in base A B C D; do
    if [ $v = base ]; then cp /tmp/base.so $L/libsphb200.so; else cp $L/libsphb200_v$v.so $L/libsphb200.so; fi
    python tools/pi_ab.py 1 0 20 paired/512 2>&1 | grep rest | sed "s/^/$v /" >> $O/res.txt
  done
done
cp /tmp/base.so $L/libsphb200.so
cat $O/res.txt
