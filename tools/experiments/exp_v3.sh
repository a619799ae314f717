#!/bin/bash
# K1 persistent-kernel check + wave-sync / raster experiments on the sparse GEMMs (C4, C3)
mkdir -p gpurun_out/v3
timeout 900 python -m pytest tests/test_gpu_mask.py tests/test_gpu_packed.py tests/test_gpu_parity_configs.py -q -x -k "mask or interleave or search or compress or pack" 2>&1 | tail -3
timeout 300 python tools/time_k1.py
for c in c4 c3; do
  for env in "" "S24_WAVESYNC=1" "S24_WAVESYNC=1 S24_GROUP_M=4" "S24_WAVESYNC=1 S24_GROUP_M=16" ""; do
    echo "== $c $env"; env $env timeout 600 python tools/experiments/exp_kernels.py $c 40 2>/dev/null | tail -1
  done
done
