# K1-TC-sym: second-half TMEM prefetch (LGP_TS_PF) x epilogue warpgroups (cfg4 t=1)
echo "PF=0 NWG=4 $(timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "PF=1 NWG=3 $(LGP_TS_PF=1 LGP_TS_NWG=3 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "PF=1 NWG=4 $(LGP_TS_PF=1 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
LGP_TS_PF=1 LGP_TS_NWG=3 timeout 300 python -m pytest tests/test_gpu_solvers.py -q -x -k "symmetric_tensor_core_cg_dims" 2>&1 | tail -1
