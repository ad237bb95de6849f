#!/bin/bash
# launch list of a fixed-budget device CG at full size (after a plain run of the same command):
# per-iteration kernels and their device times (cold-cache, serialised: compare shares)
set -e
CFG=${1:-cfg4}
K="python tools/cg_profile.py --config $CFG --iters 12"
$K > gpurun_out/plain_cg_$CFG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/cg_launches_$CFG.csv $K > gpurun_out/ncu_cg_$CFG.log 2>&1
cat gpurun_out/plain_cg_$CFG.log
