#!/bin/bash
# ncu --set full of the bench kernel (K1-TC, cfg4 t = 16), raw and source pages
# exported as CSV (run after the same command exited 0 without ncu)
mkdir -p gpurun_out
K="python tools/profile_k1.py --t 16 --reps 1"
$K > gpurun_out/plain_k1tc.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:lgp_matvec_tc -c 1 \
    -o gpurun_out/k1tc $K > gpurun_out/ncu_k1tc.log 2>&1
ncu -i gpurun_out/k1tc.ncu-rep --page raw --csv > gpurun_out/k1tc_raw.csv
cat gpurun_out/plain_k1tc.log
