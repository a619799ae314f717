#!/bin/bash
for v in 0 1; do
  for cfg in c2 c3; do
    S24_MC=$v S24_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,lts__t_sectors_srcunit_tex_op_read.sum,launch__grid_size \
       --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/mc_${v}_$cfg.csv 2>&1
  done
done
for v in 0 1 0 1; do for c in c2 c3; do S24_MC=$v timeout 300 python tools/experiments/exp_kernels.py $c 20; done; done
