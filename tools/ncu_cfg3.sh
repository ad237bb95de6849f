#!/bin/bash
# ncu --set full of K1-TC with Periodic features (cfg3, t = 16) after a plain run
set -e
K="python tools/profile_k1.py --config cfg3 --t 16 --reps 1"
$K > gpurun_out/plain_cfg3.log 2>&1
ncu --set full --clock-control none -k regex:lgp_matvec_tc -c 1 -o gpurun_out/k1tc_cfg3 $K > gpurun_out/ncu_cfg3.log 2>&1
ncu -i gpurun_out/k1tc_cfg3.ncu-rep --page raw --csv > gpurun_out/k1tc_cfg3_raw.csv
cat gpurun_out/plain_cfg3.log
