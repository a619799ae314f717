# packed-f32x2 GELU epilogue A/B: in-tree library vs exp_libs/gelu2.so, alternating, C4 / C2 steps
cd $GRAFT_REPO_ROOT
S24_LIB_PATH=exp_libs/gelu2.so python -m pytest tests/test_gpu_ffn.py tests/test_gpu_gemm.py tests/test_gpu_parity_configs.py -q -x 2>&1 | tail -2
for r in 1 2 3; do
 for v in base gelu2; do
  for c in c4 c2; do
   if [ $v = base ]; then o=$(python tools/experiments/exp_kernels.py $c 10 2>&1 | tail -1); else o=$(S24_LIB_PATH=exp_libs/gelu2.so python tools/experiments/exp_kernels.py $c 10 2>&1 | tail -1); fi
   echo "$r $v $c $o"
  done
 done
done
