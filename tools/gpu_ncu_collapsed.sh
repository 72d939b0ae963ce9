OUT=gpurun_out/${1:-collapsed}; mkdir -p $OUT
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_interact \
  -o $OUT/coll python tools/collapsed_profile.py 6000 384 > $OUT/ncu_coll.log 2>&1
python tools/ncu_lines.py $OUT/coll.ncu-rep 50 > $OUT/coll_lines.txt 2>&1
python tools/ncu_regions.py $OUT/coll.ncu-rep > $OUT/coll_regions.txt 2>&1
rm -f $OUT/*.ncu-rep
