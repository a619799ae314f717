#!/bin/bash
# One GPU call that regenerates the round's evidence: GPU tests, smoke, ncu captures (reduced to
# text / json summaries on the box: gpurun brings back at most 64 MiB) and the bench lines of
# every config (ours + the reference arm).  usage: tools/gpu_round_evidence.sh <tag>
TAG=${1:-cur}
mkdir -p gpurun_out/ev_$TAG
OUT=gpurun_out/ev_$TAG
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 bash tools/gpu_profile_round.sh $TAG > $OUT/profile.log 2>&1
for c in c2 c3 c5; do
  python tools/ncu_traffic.py gpurun_out/prof_full_${TAG}_$c.ncu-rep $c $OUT/ncu_traffic_$c.json > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/prof_full_${TAG}_$c.ncu-rep > $OUT/ncu_full_$c.txt 2>&1
  python tools/ncu_summary.py gpurun_out/prof_mask_${TAG}_$c.ncu-rep > $OUT/ncu_mask_$c.txt 2>&1
done
cp gpurun_out/launches_${TAG}_c2.csv $OUT/ 2>/dev/null
# keep only the C2 GEMM capture (source-level stall analysis); the rest are summarised above
mv gpurun_out/prof_full_${TAG}_c2.ncu-rep $OUT/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "
import json
d=json.loads(open('$OUT/bench_$c.json').read().splitlines()[-1])
print('$c', round(d['value']), round(d['ms_per_step'],4), d.get('speedup_vs_dense'), d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])
"
done
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-200 $OUT/bench_ref.json
du -sh gpurun_out
