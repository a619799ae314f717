#!/bin/bash
# 2:4 vs dense speedup of the d=12288 d_ff=49152 GELU block over token counts.
# usage: tools/c4_sweep.sh [out_dir]   (one bench.py JSON line per token count)
out=${1:-gpurun_out}
mkdir -p "$out"
for n in 2048 4096 8192 16384 32768 65536; do
  timeout 900 python bench.py --config c4 --tokens $n --steps 20 --warmup 4 --no-cpu-baseline \
    > "$out/c4_sweep_$n.json" 2> "$out/c4_sweep_$n.err" || echo "N=$n failed rc=$?"
done
