# K1-TC-sym: FP32 -> FP64 widening by integer re-bias (0) vs F2F conversion (1)
for w in 0 1; do
  echo "widen=$w cfg4 $(LGP_TS_WIDEN=$w timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
done
