#!/bin/bash
# raster-group experiment: per-kernel step times and HBM bytes for several group sizes
mkdir -p gpurun_out
for cfg in c3 c2; do
  for g in 8 0; do
    for gd in 8 4 16; do
      if [ "$g" = "0" ]; then unset S24_GROUP_M; else export S24_GROUP_M=$g; fi
      export S24_GROUP_M_DW=$gd
      timeout 300 python tools/experiments/exp_kernels.py $cfg 20
    done
  done
done > gpurun_out/exp_group.jsonl 2> gpurun_out/exp_group.err
unset S24_GROUP_M S24_GROUP_M_DW
for g in 8 0; do
  if [ "$g" = "0" ]; then unset S24_GROUP_M; else export S24_GROUP_M=$g; fi
  S24_CFG=c3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpc__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:gemm_kernel -s 6 -c 6 --csv python tools/prof_one_step.py 2 > gpurun_out/exp_group_ncu_$g.csv 2>&1
done
