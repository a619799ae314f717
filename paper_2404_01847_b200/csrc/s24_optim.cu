// the optimizer step either side of the hot path, fused into one
// HBM-bound pass per weight --
//   masked decay on the gradient (DecayMode.ON_GRADIENTS, optim.py:105-114, trainer.py:439-441)
//   -> Adam (optim.py:128-147)
//   -> SR-STE decay at the update site (DecayMode.ON_WEIGHTS, optim.py:117-125, trainer.py:442-447)
// and the mask flip statistics of a refresh (flip_rate optim.py:94-102, the per-block flip
// counts of block_flip_stats optim.py:164-192) computed from the pattern indices.
//
// double state reproduces the reference bit for bit: every operation is the reference's numpy
// expression in its evaluation order with explicit round-to-nearest intrinsics (no FMA
// contraction), and the scalar factors (1 - b1, 1 - b1^t, lr * lambda, ...) come from the
// host exactly as Python computes them.  float state is the production path (fp32 master
// weights and moments, 28 bytes of HBM traffic per weight).
#include "s24_common.cuh"
#include "s24_patterns.h"
#include "s24_adam.cuh"

namespace s24 {

__constant__ uint16_t c_opt_pat_bits[90] = S24_PATTERN_BITS;

// 16-byte vector access of 4 consecutive elements (float: one 16-byte access, double: two);
// every parameter tensor is allocated by torch (256-byte aligned) and e0 % 4 == 0
__device__ __forceinline__ void ld4(const float* p, float (&x)[4]) {
  const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
  x[0] = t.x, x[1] = t.y, x[2] = t.z, x[3] = t.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&x)[4]) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p)), b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  x[0] = a.x, x[1] = a.y, x[2] = b.x, x[3] = b.y;
}
__device__ __forceinline__ void st4(float* p, const float (&x)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(x[0], x[1], x[2], x[3]));
}
__device__ __forceinline__ void st4(double* p, const double (&x)[4]) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(x[0], x[1]));
  __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(x[2], x[3]));
}

// 4 consecutive columns of one row per thread (one mask block row); g may be fp32 or T
template <typename T, typename G>
__global__ void __launch_bounds__(256) adam_kernel(T* __restrict__ w, T* __restrict__ u, T* __restrict__ v,
                                                   const G* __restrict__ g, int64_t rows, int64_t cols,
                                                   const uint8_t* __restrict__ idx, const AdamScalars s) {
  const int64_t n4 = rows * cols / 4;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n4;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e0 = 4 * q;
    uint32_t keep = 0xF;  // mask bits of these 4 columns (1 = kept)
    if (idx != nullptr) {
      const int64_t r = e0 / cols, c = e0 - r * cols;
      const uint32_t p = idx[(r >> 2) * (cols >> 2) + (c >> 2)];
      keep = (c_opt_pat_bits[p < 90 ? p : 0] >> (4 * (r & 3))) & 0xF;
    }
    T wv[4], uv[4], vv[4];
    G gv[4];
    ld4(w + e0, wv);
    ld4(u + e0, uv);
    ld4(v + e0, vv);
    ld4(g + e0, gv);
#pragma unroll
    for (int i = 0; i < 4; ++i) adam_elem<T>(wv[i], uv[i], vv[i], static_cast<T>(gv[i]), !((keep >> i) & 1), s);
    st4(w + e0, wv);
    st4(u + e0, uv);
    st4(v + e0, vv);
  }
  // tail of a flat (unmasked) vector whose length is not a multiple of 4
  const int64_t n = rows * cols;
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t e = (n & ~int64_t(3)) + threadIdx.x;
    T wi = w[e], ui = u[e], vi = v[e];
    adam_elem<T>(wi, ui, vi, static_cast<T>(g[e]), false, s);
    w[e] = wi;
    u[e] = ui;
    v[e] = vi;
  }
}

// changed mask bits between two pattern-index maps (popcount of the xor of the 4x4 patterns)
__global__ void __launch_bounds__(256) mask_flips_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                         int64_t nb, unsigned long long* __restrict__ total,
                                                         int32_t* __restrict__ per_block) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nb;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t pa = a[i], pb = b[i];
    const int f = __popc(static_cast<uint32_t>(c_opt_pat_bits[pa < 90 ? pa : 0] ^ c_opt_pat_bits[pb < 90 ? pb : 0]));
    local += f;
    if (per_block != nullptr && f) per_block[i] += f;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ unsigned long long part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long sum = 0;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) sum += part[k];
    if (sum) atomicAdd(total, sum);
  }
}

static int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  return static_cast<int>(want < 1 ? 1 : want < cap ? want : cap);
}

}  // namespace s24

using namespace s24;

extern "C" int s24_adam_step(void* w, void* u, void* v, int state_dtype, const void* g, int g_dtype, int64_t rows,
                             int64_t cols, const uint8_t* idx, double lr, double beta1, double beta2, double eps,
                             double one_minus_beta1, double one_minus_beta2, double bias_corr1, double bias_corr2,
                             double lambda_w, double lr_lambda, int decay_mode, void* stream) {
  S24_REQUIRE(w && u && v && g, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(rows >= 0 && cols >= 0, S24_ERR_SHAPE, "negative shape");
  S24_REQUIRE(state_dtype == S24_F32 || state_dtype == S24_F64, S24_ERR_UNSUPPORTED,
              "Adam state must be fp32 or fp64");
  S24_REQUIRE(g_dtype == S24_F32 || g_dtype == state_dtype, S24_ERR_UNSUPPORTED,
              "gradient must be fp32 or the state's dtype");
  S24_REQUIRE(decay_mode >= S24_DECAY_NONE && decay_mode <= S24_DECAY_ON_WEIGHTS, S24_ERR_ARG, "bad decay mode");
  S24_REQUIRE(((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v) |
                reinterpret_cast<uintptr_t>(g)) & 15) == 0,
              S24_ERR_UNSUPPORTED, "w, u, v, g need 16-byte aligned base addresses");
  if (decay_mode != S24_DECAY_NONE || idx != nullptr) {
    S24_REQUIRE(idx != nullptr, S24_ERR_ARG, "masked decay needs the pattern indices");
    S24_REQUIRE(rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE, "masked weights need rows, cols %% 4 == 0");
  } else {
    // an unmasked parameter is a flat vector: view it as one row
    cols = rows * cols;
    rows = cols > 0 ? 1 : 0;
  }
  if (rows * cols == 0) return S24_OK;
  AdamScalars s{lr, beta1, beta2, eps, one_minus_beta1, one_minus_beta2, bias_corr1, bias_corr2, lambda_w, lr_lambda,
                decay_mode};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(rows * cols / 4 > 0 ? rows * cols / 4 : 1);
  if (state_dtype == S24_F64) {
    if (g_dtype == S24_F64)
      adam_kernel<double, double><<<grid, 256, 0, st>>>(static_cast<double*>(w), static_cast<double*>(u),
                                                        static_cast<double*>(v), static_cast<const double*>(g),
                                                        rows, cols, idx, s);
    else
      adam_kernel<double, float><<<grid, 256, 0, st>>>(static_cast<double*>(w), static_cast<double*>(u),
                                                       static_cast<double*>(v), static_cast<const float*>(g), rows,
                                                       cols, idx, s);
  } else {
    adam_kernel<float, float><<<grid, 256, 0, st>>>(static_cast<float*>(w), static_cast<float*>(u),
                                                    static_cast<float*>(v), static_cast<const float*>(g), rows, cols,
                                                    idx, s);
  }
  return s24_check_launch("adam_step");
}

extern "C" int s24_mask_flips(const uint8_t* idx_prev, const uint8_t* idx_curr, int64_t nblocks,
                              unsigned long long* changed_bits, int32_t* block_flips, void* stream) {
  S24_REQUIRE(idx_prev && idx_curr && changed_bits, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(nblocks >= 0, S24_ERR_SHAPE, "negative block count");
  if (nblocks == 0) return S24_OK;
  mask_flips_kernel<<<grid_for(nblocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(idx_prev, idx_curr, nblocks,
                                                                                       changed_bits, block_flips);
  return s24_check_launch("mask_flips");
}
