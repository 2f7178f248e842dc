#!/bin/bash
# under gpurun: event-timed rates + ncu pipe counters of scripts/micro/pipehalf.cu
set -e
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/pipehalf scripts/micro/pipehalf.cu
./scripts/micro/pipehalf > gpurun_out/pipehalf.txt 2>&1
ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fp16.sum,sm__inst_executed_pipe_xu.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp16_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --csv ./scripts/micro/pipehalf > gpurun_out/pipehalf_ncu.csv 2>&1 || true
cat gpurun_out/pipehalf.txt
