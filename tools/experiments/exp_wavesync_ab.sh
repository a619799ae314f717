cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
 for ws in d 1; do
  for c in c4 c3; do
   if [ $ws = d ]; then out=$(python tools/experiments/exp_kernels.py $c 10 2>&1 | tail -1); else out=$(S24_WAVESYNC=1 python tools/experiments/exp_kernels.py $c 10 2>&1 | tail -1); fi
   echo "$r ws=$ws $c $out"
  done
 done
done
