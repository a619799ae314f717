#!/bin/bash
# per-GEMM cycles of one step for library variants in exp_libs/ (S24_LIB_PATH)
for v in ${VARIANTS:-e8 e12}; do
  for cfg in ${CFGS:-c2 c3}; do
    S24_LIB_PATH=$PWD/exp_libs/$v.so S24_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg \
       --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/var_${v}_$cfg.csv 2>&1
  done
done
