#!/bin/bash
for x in 0 64; do
  S24_EXP=$x timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:gemm_kernel --csv python tools/experiments/exp_dw2.py > gpurun_out/exp_dw2_$x.csv 2>&1
done
S24_GROUP_M_DW=4 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel --csv python tools/experiments/exp_dw2.py 22016 > gpurun_out/exp_dw2_g4.csv 2>&1
S24_GROUP_M_DW=16 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,dram__bytes_read.sum --clock-control none -k regex:gemm_kernel --csv python tools/experiments/exp_dw2.py 22016 > gpurun_out/exp_dw2_g16.csv 2>&1
