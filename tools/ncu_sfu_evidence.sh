#!/bin/bash
# ncu evidence for the SFU (MUFU.EX2) roofline denominator: tools/alu_bench.cu's
# MUFU.EX2-only loop (8 warps per SM, 148 CTAs), --set full, raw CSV.
set -e
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o gpurun_out/alu_bench tools/alu_bench.cu
gpurun_out/alu_bench > gpurun_out/alu_bench_plain.log 2>&1
ncu --set full --clock-control none -k regex:bench -s 1 -c 1 -o gpurun_out/alu_mufu gpurun_out/alu_bench \
    > gpurun_out/ncu_alu.log 2>&1
ncu -i gpurun_out/alu_mufu.ncu-rep --page raw --csv > gpurun_out/alu_mufu_raw.csv
head -3 gpurun_out/alu_bench_plain.log
