for cfg in "LGP_TC_NSB=4" "LGP_TC_NSB=6" "LGP_TC_NSB=6 LGP_TC_G=8" "LGP_TC_NSB=6 LGP_TC_PRIO=2"; do echo "$cfg $(env $cfg timeout 100 python tools/profile_k1.py --t 16 --reps 2 2>&1 | tail -1)"; done
echo "trace NSB6: $(LGP_TC_NSB=6 LGP_TC_TRACE=1 timeout 100 python tools/profile_k1.py --t 16 --reps 1 2>&1 | head -1)"
