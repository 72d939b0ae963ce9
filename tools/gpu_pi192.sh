# A/B of a 2-CTA/SM 192-target gather build (in the pi256 slot; prebuilt libsphb200_v192*.so)
# against gather 384 / paired 512, at rest and collapsed, n_subdiv 1 and 2
set -u
O=gpurun_out/pi192; mkdir -p $O
L=paper_1110_3711_b200
cp $L/libsphb200.so /tmp/libsphb200_default.so
python tools/pi_ab.py 1 6000 10 gather/256,gather/384,paired/512 > $O/default.txt 2>&1
python tools/pi_ab.py 2 3000 10 gather/256,gather/384 > $O/default_n2.txt 2>&1
for v in v192 v192ng1; do
  cp $L/libsphb200_$v.so $L/libsphb200.so
  python tools/pi_ab.py 1 6000 10 gather/256 > $O/$v.txt 2>&1
  python tools/pi_ab.py 2 3000 10 gather/256 > $O/${v}_n2.txt 2>&1
done
cp /tmp/libsphb200_default.so $L/libsphb200.so
tail -n 8 $O/*.txt
