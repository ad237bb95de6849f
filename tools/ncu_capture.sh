#!/bin/bash
# ncu evidence for the round (run under gpurun, 1 GPU):
#  1. launch list of the bench command (cold-cache, serialised: compare shares)
#  2. one --set full capture of the top kernel (K1-TC on cfg4, t = 16)
# Each ncu run follows a plain run of the same command that exited 0.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
K="python tools/profile_k1.py --t 16 --reps 1"
$K > gpurun_out/plain_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lgp_matvec_tc -c 1 \
    -o gpurun_out/k1tc $K > gpurun_out/ncu_k1tc.log 2>&1
ncu -i gpurun_out/k1tc.ncu-rep --page raw --csv > gpurun_out/k1tc_raw.csv
ncu -i gpurun_out/k1tc.ncu-rep --page source --csv > gpurun_out/k1tc_source.csv 2>/dev/null || true
echo done
