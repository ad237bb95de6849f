#!/bin/bash
# launch list of the fused CG iteration with caches NOT flushed between kernels
# (--cache-control none: the records K1-TC-sym just wrote are still in L2, as
# in a real solve), after a plain run of the same command
set -e
CFG=${1:-cfg4}
K="python tools/cg_profile.py --config $CFG --iters 12"
$K > gpurun_out/plain_cgw_$CFG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/cg_launches_warm_$CFG.csv $K > gpurun_out/ncu_cgw_$CFG.log 2>&1
python tools/launch_summary.py gpurun_out/cg_launches_warm_$CFG.csv
