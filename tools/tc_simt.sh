# K1-TC: chunks whose distances run on the FMA pipe (bit c%8 of LGP_TC_SIMT_MASK), cfg4 t=16
for m in 0 0x08 0x48 0x49 0x55; do
  echo "MASK=$m $(LGP_TC_SIMT_MASK=$m timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
done
