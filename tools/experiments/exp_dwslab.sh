#!/bin/bash
for v in 0 1; do
  for cfg in c3 c4; do
    S24_DW_SLABS=$v S24_CFG=$cfg timeout 400 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum \
       --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/dws_${v}_$cfg.csv 2>&1
  done
  S24_DW_SLABS=$v timeout 300 python tools/experiments/exp_kernels.py c3 10
done
