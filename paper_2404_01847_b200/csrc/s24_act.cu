// K6 / K7: fused (gated) activation forward and backward on feature-major
// activations (features x tokens, tokens contiguous).
//
// Reference: kernels.gate_gelu (_core.pyx:222-250) computes
// gelu(z1) * z2 with z1 = Z[:, :r], z2 = Z[:, r:] of the column-major Z; the
// paper's point is to walk that layout along its
// contiguous axis.  Here the contiguous axis is tokens: one 16-byte vector of
// z1 and of z2 (the same 8 tokens, rows j and r + j) produce one 16-byte
// vector of A, so every byte is read once and fully coalesced.
// The backward (gated_ffn.py:336-348) is one CTA per feature row: it streams
// dA, z1, z2 along tokens, writes dZ1 / dZ2 and reduces the bias gradients
// (d_b = sum_t dZ1, d_c = sum_t dZ2) in registers + shared memory, so the
// bias reduction costs no extra pass.
#include "s24_common.cuh"

namespace s24 {

// GELU / GELU' and SiLU / SiLU' with one MUFU op each (gelu_and_grad, sigmoid_fast in
// s24_common.cuh -- the same functions as the GEMM epilogues, so the fused and unfused
// paths agree); the backward of the gated forms needs act and act' of the same z1.
template <int kAct>
__device__ __forceinline__ void act_both(float x, float& a, float& da) {
  if constexpr (kAct == S24_ACT_RELU) {
    a = fmaxf(x, 0.0f);
    da = x > 0.0f ? 1.0f : 0.0f;
  } else if constexpr (kAct == S24_ACT_SWIGLU) {
    const float sg = sigmoid_fast(x);
    a = x * sg;
    da = sg * fmaf(x, 1.0f - sg, 1.0f);
  } else {
    gelu_and_grad(x, a, da);
  }
}
template <int kAct>
__device__ __forceinline__ float act_f(float x) {
  if constexpr (kAct == S24_ACT_RELU) return fmaxf(x, 0.0f);
  else if constexpr (kAct == S24_ACT_SWIGLU) return x * sigmoid_fast(x);
  else {
    float a, da;
    gelu_and_grad(x, a, da);
    return a;
  }
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                    pack_bf16x2(f[6], f[7]));
}

template <int kAct, bool kGated>
__global__ void __launch_bounds__(256) act_fwd_kernel(const uint16_t* __restrict__ z, int64_t ldz, int64_t r,
                                                      int64_t n, uint16_t* __restrict__ a, int64_t lda) {
  // token-major: z row t = [z1 (r) | z2 (r)] (gated) or [z (r)]; a row t = act(z1) * z2
  const int64_t vpr = r / 8;  // 16-byte vectors per output row
  const int64_t total = n * vpr;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = v / vpr, j = (v % vpr) * 8;
    float x[8], o[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(z + t * ldz + j)), x);
    if constexpr (kGated) {
      float g[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(z + t * ldz + r + j)), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = act_f<kAct>(x[i]) * g[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = act_f<kAct>(x[i]);
    }
    *reinterpret_cast<uint4*>(a + t * lda + j) = pack8(o);
  }
}

constexpr int kBwdTokens = 64;  // tokens per CTA in the backward (bias partials per CTA)

template <int kAct, bool kGated>
__global__ void __launch_bounds__(256) act_bwd_kernel(const uint16_t* __restrict__ z, int64_t ldz,
                                                      const uint16_t* __restrict__ da, int64_t ldda, int64_t r,
                                                      int64_t n, uint16_t* __restrict__ dz, int64_t lddz,
                                                      float* __restrict__ dbias) {
  // thread = 8 consecutive features, loops over kBwdTokens tokens; bias partial
  // sums stay in registers and land with one atomic per feature per CTA
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (j >= r) return;
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * kBwdTokens;
  const int64_t t1 = min(n, t0 + kBwdTokens);
  float s1[8], s2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s1[i] = s2[i] = 0.0f;
#pragma unroll 4
  for (int64_t t = t0; t < t1; ++t) {
    float x[8], d[8], o1[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(z + t * ldz + j)), x);
    unpack8(__ldg(reinterpret_cast<const uint4*>(da + t * ldda + j)), d);
    if constexpr (kGated) {
      float g[8], o2[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(z + t * ldz + r + j)), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float a, da_;
        act_both<kAct>(x[i], a, da_);
        o1[i] = d[i] * g[i] * da_;  // dZ1 = dA * z2 * act'(z1)
        o2[i] = d[i] * a;           // dZ2 = dA * act(z1)
        s1[i] += o1[i];
        s2[i] += o2[i];
      }
      *reinterpret_cast<uint4*>(dz + t * lddz + r + j) = pack8(o2);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float a, da_;
        act_both<kAct>(x[i], a, da_);
        o1[i] = d[i] * da_;
        s1[i] += o1[i];
      }
    }
    *reinterpret_cast<uint4*>(dz + t * lddz + j) = pack8(o1);
  }
  if (dbias == nullptr) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    atomicAdd(dbias + j + i, s1[i]);
    if (kGated) atomicAdd(dbias + r + j + i, s2[i]);
  }
}

}  // namespace s24

using namespace s24;

static int check_act(const void* z, int64_t ldz, const void* o, int64_t ldo, int64_t r, int64_t n, int act) {
  S24_REQUIRE(z && o, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(act >= S24_ACT_RELU && act <= S24_ACT_SWIGLU, S24_ERR_ARG, "unknown activation %d", act);
  const int64_t r_in = (act == S24_ACT_GEGLU || act == S24_ACT_SWIGLU) ? 2 * r : r;
  S24_REQUIRE(r >= 0 && n >= 0 && ldz >= r_in && ldo >= r, S24_ERR_SHAPE, "bad activation shape");
  S24_REQUIRE(r % 8 == 0 && ldz % 8 == 0 && ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(z) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(o) & 15) == 0,
              S24_ERR_UNSUPPORTED, "activation rows must be 16-byte aligned (features %% 8 == 0)");
  return S24_OK;
}

template <int kAct, bool kGated>
static void launch_fwd(const uint16_t* z, int64_t ldz, int64_t r, int64_t n, uint16_t* a, int64_t lda,
                       cudaStream_t st) {
  int64_t blocks = (n * (r / 8) + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  act_fwd_kernel<kAct, kGated><<<static_cast<unsigned>(blocks), 256, 0, st>>>(z, ldz, r, n, a, lda);
}

extern "C" int s24_act_fwd(const uint16_t* z, int64_t ldz, int64_t r, int64_t n, int act, uint16_t* a, int64_t lda,
                           void* stream) {
  if (int rc = check_act(z, ldz, a, lda, r, n, act)) return rc;
  if (r == 0 || n == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (act) {
    case S24_ACT_RELU: launch_fwd<S24_ACT_RELU, false>(z, ldz, r, n, a, lda, st); break;
    case S24_ACT_GELU: launch_fwd<S24_ACT_GELU, false>(z, ldz, r, n, a, lda, st); break;
    case S24_ACT_GEGLU: launch_fwd<S24_ACT_GEGLU, true>(z, ldz, r, n, a, lda, st); break;
    default: launch_fwd<S24_ACT_SWIGLU, true>(z, ldz, r, n, a, lda, st); break;
  }
  return s24_check_launch("act_fwd");
}

extern "C" int s24_act_bwd(const uint16_t* z, int64_t ldz, const uint16_t* da, int64_t ldda, int64_t r, int64_t n,
                           int act, uint16_t* dz, int64_t lddz, float* dbias, void* stream) {
  if (int rc = check_act(z, ldz, dz, lddz, r, n, act)) return rc;
  S24_REQUIRE(da != nullptr && ldda >= r && ldda % 8 == 0 && (reinterpret_cast<uintptr_t>(da) & 15) == 0,
              S24_ERR_UNSUPPORTED, "dA rows must be 16-byte aligned");
  if (r == 0 || n == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool gated = act == S24_ACT_GEGLU || act == S24_ACT_SWIGLU;
  if (dbias != nullptr) {
    cudaError_t e = cudaMemsetAsync(dbias, 0, sizeof(float) * (gated ? 2 * r : r), st);
    S24_REQUIRE(e == cudaSuccess, S24_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  const dim3 grid(static_cast<unsigned>((r / 8 + 255) / 256), static_cast<unsigned>((n + kBwdTokens - 1) / kBwdTokens));
  switch (act) {
    case S24_ACT_RELU:
      act_bwd_kernel<S24_ACT_RELU, false><<<grid, 256, 0, st>>>(z, ldz, da, ldda, r, n, dz, lddz, dbias);
      break;
    case S24_ACT_GELU:
      act_bwd_kernel<S24_ACT_GELU, false><<<grid, 256, 0, st>>>(z, ldz, da, ldda, r, n, dz, lddz, dbias);
      break;
    case S24_ACT_GEGLU:
      act_bwd_kernel<S24_ACT_GEGLU, true><<<grid, 256, 0, st>>>(z, ldz, da, ldda, r, n, dz, lddz, dbias);
      break;
    default:
      act_bwd_kernel<S24_ACT_SWIGLU, true><<<grid, 256, 0, st>>>(z, ldz, da, ldda, r, n, dz, lddz, dbias);
      break;
  }
  return s24_check_launch("act_bwd");
}

// ---------------------------------------------------------------------------
// bf16 transpose (dst = src^T): the K-major token operand of the two-slab MVUE weight-gradient
// GEMM (X^T for dW_in, A^T for dW2).  64 x 64 tiles through shared memory, 16-byte loads and
// stores on both sides; HBM-bound (2 bytes read + 2 written per element).
namespace s24 {
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const uint16_t* __restrict__ src, int64_t rows,
                                                             int64_t cols, int64_t lds, uint16_t* __restrict__ dst,
                                                             int64_t ldd) {
  // 64 x 64 tile as 32-bit words (bf16 pairs along a row), pitch 33 words.  Write-out: warp wp
  // owns word columns 4 wp .. 4 wp + 3 (output rows 8 wp .. 8 wp + 7); lane (wq, j) reads word
  // 4 wp + wq of rows 8 j .. 8 j + 7 and emits elements r0 + 8 j .. + 7 of output rows 2 w and
  // 2 w + 1 (low / high halves), so 8 lanes write one output row's 128 contiguous bytes: a store
  // instruction touches 4 cache lines, not 32 (the L1 store wavefronts were the limit)
  __shared__ uint32_t t[64][33];
  const int tid = threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 64;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = tid + 256 * q, rr = i >> 3, v = i & 7;  // 64 rows x 8 vectors of 8
    uint4 x = make_uint4(0, 0, 0, 0);
    if (r0 + rr < rows && c0 + 8 * v < cols) x = __ldg(reinterpret_cast<const uint4*>(src + (r0 + rr) * lds + c0 + 8 * v));
    t[rr][4 * v] = x.x;
    t[rr][4 * v + 1] = x.y;
    t[rr][4 * v + 2] = x.z;
    t[rr][4 * v + 3] = x.w;
  }
  __syncthreads();
  const int lane = tid & 31, wp = tid >> 5;
  const int w = 4 * wp + (lane >> 3), j = lane & 7;  // word column, 8-row group
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = t[8 * j + k][w];
  const uint4 lo = make_uint4(__byte_perm(x[0], x[1], 0x5410), __byte_perm(x[2], x[3], 0x5410),
                              __byte_perm(x[4], x[5], 0x5410), __byte_perm(x[6], x[7], 0x5410));
  const uint4 hi = make_uint4(__byte_perm(x[0], x[1], 0x7632), __byte_perm(x[2], x[3], 0x7632),
                              __byte_perm(x[4], x[5], 0x7632), __byte_perm(x[6], x[7], 0x7632));
  if (r0 + 8 * j < rows) {
    if (c0 + 2 * w < cols) *reinterpret_cast<uint4*>(dst + (c0 + 2 * w) * ldd + r0 + 8 * j) = lo;
    if (c0 + 2 * w + 1 < cols) *reinterpret_cast<uint4*>(dst + (c0 + 2 * w + 1) * ldd + r0 + 8 * j) = hi;
  }
}
}  // namespace s24

extern "C" int s24_transpose_bf16(const uint16_t* src, int64_t rows, int64_t cols, int64_t lds, uint16_t* dst,
                                  int64_t ldd, void* stream) {
  S24_REQUIRE(src != nullptr && dst != nullptr, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(rows % 8 == 0 && cols % 8 == 0 && lds >= cols && ldd >= rows && lds % 8 == 0 && ldd % 8 == 0 &&
                  (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
              S24_ERR_UNSUPPORTED, "transpose needs 16-byte aligned rows and dims divisible by 8");
  if (rows == 0 || cols == 0) return S24_OK;
  const dim3 grid(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
  s24::transpose_bf16_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, rows, cols, lds, dst, ldd);
  return s24_check_launch("transpose_bf16");
}
