# raster group 8 vs 12 on the small configs (C2 step, C5 block), alternating
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
 for g in 8 12; do
  echo "$r g=$g c2 $(S24_GROUP_M=$g python tools/experiments/exp_kernels.py c2 200 2>&1 | tail -1)"
  echo "$r g=$g c5 $(S24_GROUP_M=$g python tools/experiments/exp_kernels.py c5 100 2>&1 | tail -1)"
 done
done
