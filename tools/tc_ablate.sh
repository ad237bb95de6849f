for ab in 0 1 2 4 3 5 6 7; do echo "ABLATE=$ab $(LGP_TC_ABLATE=$ab timeout 100 python tools/profile_k1.py --t 16 --reps 2 2>&1 | tail -1)"; done
