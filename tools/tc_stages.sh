for st in 4 6 8 12; do echo "STAGES=$st $(LGP_TC_STAGES=$st timeout 100 python tools/profile_k1.py --t 16 --reps 2 2>&1 | tail -1)"; done
