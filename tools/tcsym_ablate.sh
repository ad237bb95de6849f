# K1-TC-sym ablations (timing only; bit 1: no column butterfly, 2: no exp, 4: no per-chunk WG barrier)
for ab in 0 1 2 4 3 7; do
  echo "ablate=$ab $(LGP_TS_ABLATE=$ab timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
done
