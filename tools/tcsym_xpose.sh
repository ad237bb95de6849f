# K1-TC-sym column reduction: shared-memory transpose (1) vs butterfly (0), cfg4 t=1; parity
for x in 1 0; do echo "xpose=$x $(LGP_TS_XPOSE=$x timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"; done
echo "xpose=1 nwg=3 $(LGP_TS_NWG=3 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
LGP_TC_WATCHDOG=1 timeout 300 python -m pytest tests/test_gpu_solvers.py -q -x -k "symmetric_tensor_core" 2>&1 | tail -2
