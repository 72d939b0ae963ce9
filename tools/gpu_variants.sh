# Interaction-kernel variants at C3 (quick bench legs, no CPU baseline / e2e / collapsed / fp64)
OUT=gpurun_out/${1:-r02r}; mkdir -p $OUT
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 20"
for k in gather paired symmetric; do
  timeout 600 python bench.py $Q --pi-kernel $k > $OUT/c3_$k.json 2> $OUT/c3_$k.err
done
for b in 128 256 384; do
  timeout 600 python bench.py $Q --pi-kernel gather --pi-block $b --n-subdiv 2 > $OUT/c3n2_gather$b.json 2> $OUT/c3n2_gather$b.err
done
timeout 600 python bench.py $Q --pi-kernel paired --n-subdiv 2 > $OUT/c3n2_paired.json 2> $OUT/c3n2_paired.err
timeout 600 python bench.py $Q --slab-path > $OUT/c3_slab1.json 2> $OUT/c3_slab1.err
