#!/bin/bash
# One GPU call that regenerates the round's evidence: GPU tests, smoke, ncu captures (reduced to
# text / json summaries on the box: gpurun brings back at most 64 MiB) and the bench lines of
# every config (ours + the reference arm).  usage: tools/gpu_round_evidence.sh <tag>
TAG=${1:-cur}
mkdir -p gpurun_out/ev_$TAG
OUT=gpurun_out/ev_$TAG
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
# bench lines first (fresh box), then the profiles
timeout 1500 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in c2 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for f in $OUT/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().splitlines()[-1])
print('$f', d.get('config',{}).get('workload','')[:30], round(d['value']), d.get('ms_per_step'), d.get('speedup_vs_best_dense'), d.get('mvue_exact_speedup_vs_best_dense'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))
"; done
# ncu: launch list of the default command, GEMM + K1/K2 captures of one step (C2, C3, C4, C5), K1 / K8 alone
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_default.csv \
    python bench.py --no-cpu-baseline > $OUT/launches_run.log 2>&1
for cfg in c2 c3 c4 c5; do
  S24_CFG=$cfg timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 6 \
      -o gpurun_out/pf_${TAG}_$cfg python tools/prof_one_step.py 2 > $OUT/prof_full_$cfg.log 2>&1
  python tools/ncu_traffic.py gpurun_out/pf_${TAG}_$cfg.ncu-rep $cfg $OUT/ncu_traffic_$cfg.json > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/pf_${TAG}_$cfg.ncu-rep > $OUT/ncu_full_$cfg.txt 2>&1
  S24_CFG=$cfg timeout 600 ncu --set full --clock-control none -k regex:"prune|search" -s 0 -c 2 \
      -o gpurun_out/pm_${TAG}_$cfg python tools/prof_one_step.py 2 > $OUT/prof_mask_$cfg.log 2>&1
  python tools/ncu_summary.py gpurun_out/pm_${TAG}_$cfg.ncu-rep > $OUT/ncu_mask_$cfg.txt 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:search_bf16 -s 2 -c 1 -o gpurun_out/pk1_$TAG \
    python tools/prof_k1.py 49152 12288 pair > $OUT/prof_k1.log 2>&1
ncu -i gpurun_out/pk1_$TAG.ncu-rep --page raw --csv > $OUT/ncu_raw_k1_c4.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:mvue_tile_kernel -s 1 -c 1 -o gpurun_out/pk8_$TAG \
    python tools/time_k8.py > $OUT/prof_k8.log 2>&1
ncu -i gpurun_out/pk8_$TAG.ncu-rep --page raw --csv > $OUT/ncu_raw_k8_c2.csv 2>&1
python tools/time_k1.py > $OUT/time_k1.txt 2>&1
python tools/time_k8.py > $OUT/time_k8.txt 2>&1
# keep the C2 GEMM capture (source-level stall analysis); the rest are summarised above
mv gpurun_out/pf_${TAG}_c2.ncu-rep $OUT/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
