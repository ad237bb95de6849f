# K1-TC-sym: exp2 entries per 16 on the FMA pipe (cfg4 / cfg2-like t=1)
for p in 0 2 4 6; do
  echo "poly=$p cfg4 $(LGP_TS_POLY=$p timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
done
echo "cfg2 $(timeout 100 python tools/profile_k1.py --config cfg2 --t 1 --reps 3 2>&1 | tail -1)"
echo "cfg2 poly4 $(LGP_TS_POLY=4 timeout 100 python tools/profile_k1.py --config cfg2 --t 1 --reps 3 2>&1 | tail -1)"
