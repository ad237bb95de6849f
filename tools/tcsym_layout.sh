# K1-TC-sym TMEM read layout: 16x256b tiles (1, default) vs 32x32b rows (0); parity + cfg4/cfg5 t=1 timing + CG
LGP_TC_WATCHDOG=1 timeout 300 python -m pytest tests/test_gpu_solvers.py -q -x -k "symmetric_tensor_core" 2>&1 | tail -3
for l in 1 0; do
  echo "layout=$l cfg4 $(LGP_TS_LAYOUT=$l timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
  echo "layout=$l cfg5 $(LGP_TS_LAYOUT=$l timeout 200 python tools/profile_k1.py --config cfg5 --t 1 --reps 2 2>&1 | tail -1)"
done
for l in 1 0; do echo "layout=$l CG $(LGP_TS_LAYOUT=$l timeout 300 python tools/cg_tc_check.py 2>&1 | tail -1)"; done
