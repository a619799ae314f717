#!/bin/bash
mkdir -p gpurun_out
for x in 0 32; do
  S24_EXP=$x S24_CFG=c3 timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum \
     --clock-control none -k regex:gemm_kernel -s 8 -c 4 --csv python tools/prof_one_step.py 2 > gpurun_out/exp_dw_$x.csv 2>&1
done
