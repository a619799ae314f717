// Adam element update shared by the optimizer step (s24_optim.cu) and the fused
// optimizer + per-step compression kernel (s24_mask.cu): adam_step (optim.py:128-147) with
// the masked decay on the gradient (optim.py:105-114) or at the update site (optim.py:117-125),
// every operation in numpy's evaluation order with explicit round-to-nearest intrinsics.
#pragma once
#include "s24_common.cuh"

namespace s24 {

struct AdamScalars {
  double lr, b1, b2, eps, omb1, omb2, bc1, bc2, lam, lr_lam;
  int mode;  // S24_DECAY_NONE / ON_GRADIENTS / ON_WEIGHTS
};

__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double rsqrt_(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float rsqrt_(float a) { return __fsqrt_rn(a); }

// one element; `pruned` = (1 - m) as the reference's (uint8) factor
template <typename T>
__device__ __forceinline__ void adam_elem(T& w, T& u, T& v, T g, bool pruned, const AdamScalars& s) {
  const T w0 = w;
  // (1 - m) * w exactly as numpy forms it (0 * w keeps the sign of zero, 0 * inf is NaN)
  const T dw = rmul(static_cast<T>(pruned ? 1 : 0), w0);
  if (s.mode == S24_DECAY_ON_GRADIENTS) g = radd(g, rmul(static_cast<T>(s.lam), dw));
  u = radd(rmul(u, static_cast<T>(s.b1)), rmul(static_cast<T>(s.omb1), g));
  v = radd(rmul(v, static_cast<T>(s.b2)), rmul(static_cast<T>(s.omb2), rmul(g, g)));
  T denom = rsqrt_(rdiv(v, static_cast<T>(s.bc2)));
  denom = radd(denom, static_cast<T>(s.eps));
  denom = rmul(denom, static_cast<T>(s.bc1));
  w = rsub(w0, rdiv(rmul(static_cast<T>(s.lr), u), denom));
  if (s.mode == S24_DECAY_ON_WEIGHTS) w = rsub(w, rmul(static_cast<T>(s.lr_lam), dw));
}

}  // namespace s24
