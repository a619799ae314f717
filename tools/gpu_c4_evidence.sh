#!/bin/bash
# C4 (the default headline) evidence: ncu launch list of the default bench command and a
# --set full capture of the six GEMMs of one C4 step (+ K1/K2), summarised on the box.
# usage: tools/gpu_c4_evidence.sh <tag>
TAG=${1:-cur}
OUT=gpurun_out/c4_$TAG
mkdir -p $OUT
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --no-cpu-baseline --no-sub > $OUT/launches_run.log 2>&1
S24_CFG=c4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 6 \
    -o $OUT/full_c4 python tools/prof_one_step.py 2 > $OUT/full_c4.log 2>&1
S24_CFG=c4 timeout 600 ncu --set full --clock-control none -k regex:"prune|search" -s 0 -c 2 \
    -o $OUT/mask_c4 python tools/prof_one_step.py 2 > $OUT/mask_c4.log 2>&1
python tools/ncu_traffic.py $OUT/full_c4.ncu-rep c4 $OUT/ncu_traffic_c4.json > /dev/null 2>&1
python tools/ncu_summary.py $OUT/full_c4.ncu-rep > $OUT/ncu_full_c4.txt 2>&1
python tools/ncu_summary.py $OUT/mask_c4.ncu-rep > $OUT/ncu_mask_c4.txt 2>&1
rm -f $OUT/*.ncu-rep
cat $OUT/ncu_full_c4.txt $OUT/ncu_mask_c4.txt $OUT/ncu_traffic_c4.json
