#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + full-set capture of every kernel of one step
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 2 --no-cpu-baseline --no-dense > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|mask_tile|act_" -s 8 -c 8 \
    -o gpurun_out/prof_full python tools/prof_one_step.py 3 > gpurun_out/prof_full.log 2>&1
S24_CFG=c3 ncu --set full --clock-control none -k regex:"gemm_kernel|mask_tile|act_" -s 9 -c 9 \
    -o gpurun_out/prof_full_c3 python tools/prof_one_step.py 2 > gpurun_out/prof_full_c3.log 2>&1
ls -la gpurun_out
