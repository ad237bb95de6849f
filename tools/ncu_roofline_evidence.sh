#!/bin/bash
# ncu evidence for the K1-TC roofline denominator: the tcgen05.ld microbenchmark
# (tools/tmem_bench.cu, mode 0: 8 warps per SM loop tcgen05.ld 32x32b.x32) and the
# bench kernel (K1-TC, cfg4 t = 16), both --set full, raw pages exported as CSV.
set -e
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o gpurun_out/tmem_bench tools/tmem_bench.cu
gpurun_out/tmem_bench 0 > gpurun_out/tmem_bench_plain.log 2>&1
ncu --set full --clock-control none -k regex:kern -s 1 -c 1 -o gpurun_out/tmem_bench gpurun_out/tmem_bench 0 \
    > gpurun_out/ncu_tmem_bench.log 2>&1
ncu -i gpurun_out/tmem_bench.ncu-rep --page raw --csv > gpurun_out/tmem_bench_raw.csv
K="python tools/profile_k1.py --t 16 --reps 1"
$K > gpurun_out/plain_k1tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lgp_matvec_tc -c 1 \
    -o gpurun_out/k1tc $K > gpurun_out/ncu_k1tc.log 2>&1
ncu -i gpurun_out/k1tc.ncu-rep --page raw --csv > gpurun_out/k1tc_raw.csv
ncu -i gpurun_out/k1tc.ncu-rep --page source --csv > gpurun_out/k1tc_source.csv 2>/dev/null || true
cat gpurun_out/tmem_bench_plain.log gpurun_out/plain_k1tc.log
