for tune in "8,128,64,4,3" "8,128,64,4,4" "8,128,32,6,3" "8,128,64,3,3" "6,128,64,4,4" "12,128,64,4,2" "8,64,64,4,6" "10,128,64,4,3"; do echo "T1 $tune $(LGP_TUNE=$tune timeout 100 python tools/profile_k1.py --t 1 --reps 2 2>&1 | tail -1)"; done
for tune in "4,128,64,4,2" "4,128,64,4,3" "2,256,64,4,2"; do echo "T4 $tune $(LGP_TUNE=$tune timeout 100 python tools/profile_k1.py --t 4 --reps 2 2>&1 | tail -1)"; done
echo "T4 default NO_SYM $(timeout 100 python tools/profile_k1.py --t 4 --reps 2 --flags 16 2>&1 | tail -1)"
