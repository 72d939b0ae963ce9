# same-box A/B of C1/C2 throughput: the worktree _oldwt (an older commit, its own build) vs HEAD
set -u
O=gpurun_out/abc1; mkdir -p $O
Q="--no-cpu-baseline --e2e-steps 0 --collapsed-step 0 --fp64-steps 0 --steps 30"
for rep in 1 2; do
  for c in c1; do
    (cd _oldwt && timeout 600 python bench.py $Q --config $c > ../$O/old_${c}_$rep.json 2>/dev/null)
    timeout 600 python bench.py $Q --config $c > $O/new_${c}_$rep.json 2>/dev/null
  done
done
python tools/show_bench.py $O/*.json
