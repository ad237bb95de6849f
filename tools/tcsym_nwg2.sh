# K1-TC-sym (16x256b layout): epilogue warpgroups / S buffers (cfg4 t=1)
echo "NWG=4 NSB=8 $(timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "NWG=4 NSB=4 $(LGP_TS_NSB=4 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "NWG=5 NSB=5 $(LGP_TS_NWG=5 LGP_TS_NSB=5 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "NWG=3 NSB=6 $(LGP_TS_NWG=3 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
echo "NWG=2 NSB=8 $(LGP_TS_NWG=2 LGP_TS_NSB=8 timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
