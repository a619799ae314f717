#!/bin/bash
# bench.py JSON lines of every config (ours) + the reference arm, into gpurun_out/<dir>
OUT=gpurun_out/${1:-bench_all}
mkdir -p $OUT
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
