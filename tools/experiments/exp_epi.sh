#!/bin/bash
mkdir -p gpurun_out
for cfg in c2 c3; do
  for x in 0 16 32 48 1 17; do
    S24_EXP=$x timeout 300 python tools/experiments/exp_kernels.py $cfg 20
  done
done > gpurun_out/exp_epi.jsonl 2> gpurun_out/exp_epi.err
