# K1-TC v5 (mma.sync distance tiles, NWG epilogue warpgroups) vs v4: parity + time
for n in 3 4; do
  LGP_TC_V5=1 LGP_T4_NWG=$n LGP_TC_WATCHDOG=1 timeout 300 python -m pytest tests/test_gpu_matvec.py -x -q -k "tensor_core_matvec_parity or cfg4_rows" 2>&1 | tail -1
  echo "V5 NWG=$n $(LGP_TC_V5=1 LGP_T4_NWG=$n timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
  echo "V5 NWG=$n $(LGP_TC_V5=1 LGP_T4_NWG=$n timeout 200 python tools/profile_k1.py --config cfg5 --t 8 --reps 2 2>&1 | tail -1)"
done
echo "V4 $(timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
