# K1-TC distance tiles via mma.sync for the chunks in mask LGP_TC_HMMA (bit c % 8): parity + time
LGP_TC_HMMA=0x88 LGP_TC_WATCHDOG=1 timeout 300 python -m pytest tests/test_gpu_matvec.py -x -q -k "tensor_core_matvec_parity or cfg4_rows" 2>&1 | tail -1
for h in 0 0x80 0x88 0xAA 0xFF; do
  echo "HMMA=$h $(LGP_TC_HMMA=$h timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
done
