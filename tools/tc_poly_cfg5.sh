# K1-TC FMA-pipe exp2 share for the Matern-3/2 tree (cfg5, t=8) and RBF (cfg4, t=16)
for p in 0 2 4 6 8; do
  echo "cfg5 POLY=$p $(LGP_TC_POLY=$p timeout 200 python tools/profile_k1.py --config cfg5 --t 8 --reps 2 2>&1 | tail -1)"
done
