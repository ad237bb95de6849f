# K1-TC: entries per 16 whose exp2 runs on the FMA pipe (LGP_TC_POLY), cfg4 t=16
for p in 0 2 4; do
  echo "POLY=$p $(LGP_TC_POLY=$p timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
done
