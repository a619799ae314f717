#!/bin/bash
# Trimmed end-of-round evidence after a GEMM-only change: GPU tests + smoke, the bench lines
# (default C4 + C3 sub-line, C2, C5, reference arm), and the C4 ncu captures (launch list of the
# default command, --set full of one step's six GEMMs, K1/K2).  usage: tools/gpu_final_evidence.sh <tag>
TAG=${1:-cur}
OUT=gpurun_out/ev_$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in c2 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for f in $OUT/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().splitlines()[-1])
print('$f', d.get('config',{}).get('workload','')[:30], round(d['value']), d.get('ms_per_step'), d.get('speedup_vs_best_dense'), d.get('mvue_exact_speedup_vs_best_dense'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))
"; done
timeout 1500 tools/gpu_c4_evidence.sh $TAG > /dev/null 2>&1
cat gpurun_out/c4_$TAG/ncu_full_c4.txt | cut -c1-200
du -sh gpurun_out
# C4 token sweep (BASELINE configs[3]) on the final code
timeout 2400 tools/c4_sweep.sh $OUT/sweep > /dev/null 2>&1
for f in $OUT/sweep/c4_sweep_*.json; do python -c "
import json
d=json.loads(open('$f').read().splitlines()[-1])
print('$f', round(d['value']), d.get('speedup_vs_best_dense'), d.get('mvue_exact_speedup_vs_best_dense'), d.get('clocks',{}).get('sm_mhz'))
"; done
