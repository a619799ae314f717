#!/bin/bash
mkdir -p gpurun_out
for x in ${EXPS:-0 1 2 3}; do
  S24_EXP=$x timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg,sm__cycles_elapsed.avg \
     --clock-control none -k regex:gemm_kernel -s 3 --csv python tools/experiments/exp_gemm_iso.py 4 > gpurun_out/exp_iso_$x.csv 2>&1
done
