#!/bin/bash
# ncu capture of the symmetric tensor-core K1 (cfg4, t = 1) after a plain run
set -e
K="python tools/profile_k1.py --t 1 --reps 1"
$K > gpurun_out/plain_tcsym.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lgp_matvec_tcsym -c 1 \
    -o gpurun_out/tcsym $K > gpurun_out/ncu_tcsym.log 2>&1
ncu -i gpurun_out/tcsym.ncu-rep --page raw --csv > gpurun_out/tcsym_raw.csv
ncu -i gpurun_out/tcsym.ncu-rep --page source --csv > gpurun_out/tcsym_source.csv 2>/dev/null || true
cat gpurun_out/plain_tcsym.log
