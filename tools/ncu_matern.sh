#!/bin/bash
# ncu --set full of K1-TC on a Matern tree (cfg2: matern52 D=4, t=16) after a plain run
set -e
K="python tools/profile_k1.py --config cfg2 --t 16 --reps 1"
$K > gpurun_out/plain_m52.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lgp_matvec_tc -c 1 \
    -o gpurun_out/k1tc_m52 $K > gpurun_out/ncu_m52.log 2>&1
ncu -i gpurun_out/k1tc_m52.ncu-rep --page raw --csv > gpurun_out/k1tc_m52_raw.csv
ncu -i gpurun_out/k1tc_m52.ncu-rep --page source --csv > gpurun_out/k1tc_m52_source.csv 2>/dev/null || true
cat gpurun_out/plain_m52.log
