#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + full-set capture of the six GEMMs
# of exactly one step (the second) and of the per-step prune kernel, for C2, C3 and one C5 block.
# usage: tools/gpu_profile_round.sh <tag>     (then: tools/ncu_traffic.py ... on the reports)
set -x
TAG=${1:-cur}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_c2.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/launches_run.log 2>&1
for cfg in c2 c3 c5; do
  S24_CFG=$cfg ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 6 \
      -o gpurun_out/prof_full_${TAG}_$cfg python tools/prof_one_step.py 2 > gpurun_out/prof_full_$cfg.log 2>&1
  S24_CFG=$cfg ncu --set full --clock-control none --import-source on -k regex:"prune|search" -s 0 -c 2 \
      -o gpurun_out/prof_mask_${TAG}_$cfg python tools/prof_one_step.py 2 > gpurun_out/prof_mask_$cfg.log 2>&1
done
ls -la gpurun_out
