p() { echo "$1 t=$2: $(env $1 timeout 100 python tools/profile_k1.py --t $2 --reps 5 2>&1 | tail -1)"; }
p "" 16
p "LGP_TC_NWG=4 LGP_TC_NCI=2" 16
p "LGP_TC_NWG=4 LGP_TC_NCI=2 LGP_TC_D2B=1" 16
p "LGP_TC_NCI=2" 16
p "LGP_TC_NWG=4 LGP_TC_NCI=2" 8
p "" 8
echo "cfg5: $(timeout 200 python tools/profile_k1.py --config cfg5 --reps 2 2>&1 | tail -1)"
echo "cfg5 nwg4: $(LGP_TC_NWG=4 LGP_TC_NCI=2 timeout 200 python tools/profile_k1.py --config cfg5 --reps 2 2>&1 | tail -1)"
