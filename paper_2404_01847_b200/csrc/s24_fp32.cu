// fp32 mode of the FFN block (the reference computes on float32 / float64 fused types,
// _core.pyx:21-23; BASELINE configs[0] / C1 is fp32).  The 2:4 tensor cores take bf16 or tf32,
// and tf32 structured sparsity is 1:2 at 32-bit granularity (one of each adjacent pair), which
// cannot express a transposable 2:4 mask (a group may keep both elements of a pair).  So every
// fp32 product runs on the bf16 2:4 pipe as three split products:
//   x = x_hi + x_lo (x_hi = bf16(x), x_lo = bf16(x - x_hi)),  A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi
// accumulated in fp32 (relative error ~2^-16 per product, well inside the fp32 mode's 2e-3).
// This file holds the elementwise pieces: the split, and the (gated) activation forward /
// backward on FEATURE-major fp32 activations (features x tokens, the storage order of the
// reference's column-major FST outputs, gated_ffn.py:162), emitting the split operands of the
// next product and the bias gradients.  Exact erf GELU (gated_ffn.py:58-70) and exp SiLU.
#include "s24_common.cuh"

namespace s24 {

__device__ __forceinline__ void split2(float x, uint16_t& hi, uint16_t& lo) {
  hi = f32_to_bf16(x);
  lo = f32_to_bf16(x - bf16_to_f32(hi));
}

__global__ void split_kernel(const float* __restrict__ x, int64_t n, uint16_t* __restrict__ hi,
                             uint16_t* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    split2(x[i], hi[i], lo[i]);
}

// exact GELU and its derivative (gated_ffn.py:58-70: 0.5 x (1 + erf(x / sqrt 2)), and
// 0.5 (1 + erf(x / sqrt 2)) + x phi(x))
__device__ __forceinline__ void gelu_exact(float x, float& g, float& dg) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  g = x * cdf;
  dg = cdf + x * 0.39894228040143268f * expf(-0.5f * x * x);
}
__device__ __forceinline__ void silu_exact(float x, float& a, float& da) {
  const float sg = 1.0f / (1.0f + expf(-x));
  a = x * sg;
  da = sg * (1.0f + x * (1.0f - sg));
}
template <int kAct>
__device__ __forceinline__ void act_exact(float x, float& a, float& da) {
  if constexpr (kAct == S24_ACT_RELU) {
    a = fmaxf(x, 0.0f);
    da = x > 0.0f ? 1.0f : 0.0f;
  } else if constexpr (kAct == S24_ACT_SWIGLU) {
    silu_exact(x, a, da);
  } else {
    gelu_exact(x, a, da);
  }
}

// forward: one CTA row-strip per feature j (gated: rows j (u) and r + j (v) of Z), tokens along
// threads.  Z += bias in place (the backward's pre-activation), A = act(z) or act(z_u) z_v,
// A_hi / A_lo its split.
template <int kAct, bool kGated>
__global__ void __launch_bounds__(256) act_fwd_f32_kernel(float* __restrict__ z, int64_t ldz,
                                                          const float* __restrict__ bias, int64_t r, int64_t n,
                                                          float* __restrict__ a, int64_t lda,
                                                          uint16_t* __restrict__ a_hi, uint16_t* __restrict__ a_lo) {
  const int64_t j = blockIdx.x;
  float* zu = z + j * ldz;
  float* zv = kGated ? z + (r + j) * ldz : nullptr;
  const float bu = bias ? bias[j] : 0.0f;
  const float bv = (kGated && bias) ? bias[r + j] : 0.0f;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    const float u = zu[t] + bu;
    zu[t] = u;
    float av, dv;
    act_exact<kAct>(u, av, dv);
    if constexpr (kGated) {
      const float v = zv[t] + bv;
      zv[t] = v;
      av *= v;
    }
    a[j * lda + t] = av;
    split2(av, a_hi[j * lda + t], a_lo[j * lda + t]);
  }
}

// backward: dZ (fp32 and split) and the bias gradient dbias[f] = sum_t dZ[f, t], one CTA per
// feature row with a fixed-order block reduction (deterministic).
template <int kAct, bool kGated>
__global__ void __launch_bounds__(256) act_bwd_f32_kernel(const float* __restrict__ z, int64_t ldz,
                                                          const float* __restrict__ da, int64_t ldda, int64_t r,
                                                          int64_t n, float* __restrict__ dz, int64_t lddz,
                                                          uint16_t* __restrict__ dz_hi, uint16_t* __restrict__ dz_lo,
                                                          float* __restrict__ dbias) {
  const int64_t j = blockIdx.x;
  const float* zu = z + j * ldz;
  const float* zv = kGated ? z + (r + j) * ldz : nullptr;
  float su = 0.0f, sv = 0.0f;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    const float g = da[j * ldda + t];
    float av, dv;
    act_exact<kAct>(zu[t], av, dv);
    float du;
    if constexpr (kGated) {
      const float v = zv[t];
      du = g * v * dv;
      const float dvv = g * av;
      sv += dvv;
      if (dz) dz[(r + j) * lddz + t] = dvv;
      split2(dvv, dz_hi[(r + j) * lddz + t], dz_lo[(r + j) * lddz + t]);
    } else {
      du = g * dv;
    }
    su += du;
    if (dz) dz[j * lddz + t] = du;
    split2(du, dz_hi[j * lddz + t], dz_lo[j * lddz + t]);
  }
  __shared__ float red[2][8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    su += __shfl_xor_sync(0xffffffffu, su, o);
    sv += __shfl_xor_sync(0xffffffffu, sv, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = su;
    red[1][w] = sv;
  }
  __syncthreads();
  if (threadIdx.x == 0 && dbias != nullptr) {
    float a0 = 0.0f, a1 = 0.0f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
      a0 += red[0][i];
      a1 += red[1][i];
    }
    dbias[j] = a0;
    if constexpr (kGated) dbias[r + j] = a1;
  }
}

}  // namespace s24

using namespace s24;

extern "C" int s24_split_bf16(const float* x, int64_t n, uint16_t* hi, uint16_t* lo, void* stream) {
  S24_REQUIRE(x && hi && lo, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(n >= 0, S24_ERR_SHAPE, "negative size");
  if (n == 0) return S24_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  split_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, hi, lo);
  return s24_check_launch("split_bf16");
}

#define S24_ACT_DISPATCH(KERNEL, ...)                                                                    \
  switch (act) {                                                                                         \
    case S24_ACT_RELU: KERNEL<S24_ACT_RELU, false><<<grid, 256, 0, st>>>(__VA_ARGS__); break;           \
    case S24_ACT_GELU: KERNEL<S24_ACT_GELU, false><<<grid, 256, 0, st>>>(__VA_ARGS__); break;           \
    case S24_ACT_GEGLU: KERNEL<S24_ACT_GEGLU, true><<<grid, 256, 0, st>>>(__VA_ARGS__); break;          \
    default: KERNEL<S24_ACT_SWIGLU, true><<<grid, 256, 0, st>>>(__VA_ARGS__); break;                    \
  }

extern "C" int s24_act_fwd_f32(float* z, int64_t ldz, const float* bias, int64_t r, int64_t n, int act, float* a,
                               int64_t lda, uint16_t* a_hi, uint16_t* a_lo, void* stream) {
  S24_REQUIRE(z && a && a_hi && a_lo, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(act >= S24_ACT_RELU && act <= S24_ACT_SWIGLU, S24_ERR_ARG, "bad activation");
  S24_REQUIRE(r >= 0 && n >= 0 && ldz >= n && lda >= n, S24_ERR_SHAPE, "bad feature-major shape");
  if (r == 0 || n == 0) return S24_OK;
  S24_REQUIRE(r <= INT32_MAX, S24_ERR_SHAPE, "too many features");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(static_cast<unsigned>(r));
  S24_ACT_DISPATCH(act_fwd_f32_kernel, z, ldz, bias, r, n, a, lda, a_hi, a_lo)
  return s24_check_launch("act_fwd_f32");
}

extern "C" int s24_act_bwd_f32(const float* z, int64_t ldz, const float* da, int64_t ldda, int64_t r, int64_t n,
                               int act, float* dz, int64_t lddz, uint16_t* dz_hi, uint16_t* dz_lo, float* dbias,
                               void* stream) {
  S24_REQUIRE(z && da && dz_hi && dz_lo, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(act >= S24_ACT_RELU && act <= S24_ACT_SWIGLU, S24_ERR_ARG, "bad activation");
  S24_REQUIRE(r >= 0 && n >= 0 && ldz >= n && ldda >= n && lddz >= n, S24_ERR_SHAPE, "bad feature-major shape");
  if (r == 0 || n == 0) return S24_OK;
  S24_REQUIRE(r <= INT32_MAX, S24_ERR_SHAPE, "too many features");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(static_cast<unsigned>(r));
  S24_ACT_DISPATCH(act_bwd_f32_kernel, z, ldz, da, ldda, r, n, dz, lddz, dz_hi, dz_lo, dbias)
  return s24_check_launch("act_bwd_f32");
}
