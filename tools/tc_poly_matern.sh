# K1-TC exponentials on the FMA pipe (LGP_TC_POLY, per 16 entries) for Matern trees (2 MUFU / entry)
for p in 2 4 6 8; do
  echo "poly=$p $(LGP_TC_POLY=$p timeout 300 python tools/profile_k1.py --config cfg5 --t 8 --reps 2 2>&1 | tail -1)"
  echo "poly=$p $(LGP_TC_POLY=$p timeout 100 python tools/profile_k1.py --config cfg2 --t 16 --reps 3 2>&1 | tail -1)"
done
