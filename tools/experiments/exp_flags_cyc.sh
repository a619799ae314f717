#!/bin/bash
# per-GEMM cycles of one C2 step under experiment flags
for x in ${EXPS:-0 16 1 17}; do
  S24_EXP=$x S24_CFG=${CFG:-c2} timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg \
     --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/fl_$x.csv 2>&1
done
