# drain-lag / accumulation-group sweep of K1-TC on cfg4 t=16
for g in 4 8; do for lag in 1 2 4 8; do
  [ $lag -gt $g ] && continue
  echo "G=$g DLAG=$lag $(LGP_TC_G=$g LGP_TC_DLAG=$lag timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
done; done
