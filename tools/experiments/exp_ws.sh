#!/bin/bash
for ws in 0 1; do
  for cfg in c2 c3; do
    S24_WAVESYNC=$ws S24_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum \
       --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/ws_${ws}_$cfg.csv 2>&1
  done
done
for ws in 0 1; do for c in c2 c3; do S24_WAVESYNC=$ws timeout 300 python tools/experiments/exp_kernels.py $c 20; done; done
