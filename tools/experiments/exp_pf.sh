#!/bin/bash
for pf in ${PFS:-0 2 4 8}; do
  for cfg in c2 c3; do
    S24_PF=$pf S24_PF_DW=$pf S24_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum \
       --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/pf_${pf}_$cfg.csv 2>&1
  done
done
