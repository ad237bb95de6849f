# symmetric tensor-core CG matvec: epilogue warpgroups 3 vs 4 (cfg4 and cfg5, t=1)
for n in 3 4; do
  echo "NWG=$n $(LGP_TS_NWG=$n timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
  echo "cfg5 NWG=$n $(LGP_TS_NWG=$n timeout 200 python tools/profile_k1.py --config cfg5 --t 1 --reps 2 2>&1 | tail -1)"
done
echo "SIMT-sym $(LGP_NO_TCSYM=1 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
