# symmetric tensor-core CG matvec: epilogue warpgroups 2 vs 3 (cfg4 t=1), parity test
for n in 3 4; do
  echo "NWG=$n $(LGP_TCSYM=1 LGP_TS_NWG=$n timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
done
echo "SIMT $(timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
LGP_TC_WATCHDOG=1 timeout 300 python -m pytest tests/test_gpu_solvers.py -q -x -k "tensor_core" 2>&1 | tail -1
for n in 3 4; do
  echo "cfg5 NWG=$n $(LGP_TCSYM=1 LGP_TS_NWG=$n timeout 200 python tools/profile_k1.py --config cfg5 --t 1 --reps 2 2>&1 | tail -1)"
done
echo "cfg5 SIMT $(timeout 200 python tools/profile_k1.py --config cfg5 --t 1 --reps 2 2>&1 | tail -1)"
