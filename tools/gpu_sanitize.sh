#!/bin/bash
# compute-sanitizer over one C2 step (plain), one MVUE step (K8 exact, transposes, two-slab 2:4 dW),
# the gated (SwiGLU) epilogues at a small C3-shaped size, and the training-loop kernels
# (run_training + the autograd module on fp32 parameters).  usage: tools/gpu_sanitize.sh [tag]
TAG=${1:-san}
mkdir -p gpurun_out/$TAG
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py c2 > gpurun_out/$TAG/${tool}_c2.log 2>&1
  S24_SDW_SLABS=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py mvue > gpurun_out/$TAG/${tool}_mvue.log 2>&1
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py c3-small > gpurun_out/$TAG/${tool}_c3small.log 2>&1
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_step.py train > gpurun_out/$TAG/${tool}_train.log 2>&1
done
tail -n 3 gpurun_out/$TAG/*.log
