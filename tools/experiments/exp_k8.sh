#!/bin/bash
for lib in exp_libs/k8old.so paper_2404_01847_b200/libs24b200.so; do
  S24_LIB_PATH=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,gpc__cycles_elapsed.avg.per_second,smsp__inst_executed.sum --clock-control none -k regex:mvue -s 1 -c 1 --csv python tools/prof_k8.py > gpurun_out/k8_$(basename $lib .so).csv 2>&1
done
