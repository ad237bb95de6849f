# K1 time per launch for every BASELINE config at its CG (t=1) and multi-RHS t
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  for t in 1 8 16; do
    timeout 300 python tools/profile_k1.py --config $c --t $t --reps 3 2>&1 | tail -1
  done
done
for c in cfg2 cfg3; do timeout 300 python tools/cg_profile.py --config $c --iters 100 2>&1 | tail -1; done
