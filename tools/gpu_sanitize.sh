#!/bin/bash
# compute-sanitizer over one C2 step (plain) and one MVUE step (K8 exact, transposes, two-slab 2:4 dW)
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py c2 > gpurun_out/san/${tool}_c2.log 2>&1
  S24_SDW_SLABS=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py mvue > gpurun_out/san/${tool}_mvue.log 2>&1
done
tail -n 3 gpurun_out/san/*.log
