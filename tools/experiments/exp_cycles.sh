#!/bin/bash
# per-GEMM cycles + clock of one step (ncu, serialized), for configs c2 c3; tag = $1
mkdir -p gpurun_out
for cfg in ${CFGS:-c2 c3}; do
  S24_CFG=$cfg timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none -k regex:"gemm_kernel|prune" -s 8 -c 8 --csv python tools/prof_one_step.py 2 > gpurun_out/cyc_$1_$cfg.csv 2>&1
done
