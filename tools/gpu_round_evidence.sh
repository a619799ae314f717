#!/bin/bash
# One GPU call that regenerates the round's evidence: GPU tests, smoke, ncu captures and the
# bench lines of every config (ours + the reference arm).  usage: tools/gpu_round_evidence.sh <tag>
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 bash tools/gpu_profile_round.sh $TAG > gpurun_out/profile_$TAG.log 2>&1
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_${TAG}_$c.json').read().splitlines()[-1])
print('$c', round(d['value']), round(d['ms_per_step'],4), d.get('speedup_vs_dense'), d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])
"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; cut -c1-200 gpurun_out/bench_${TAG}_ref.json
