// K1 (transposable mask search, optionally fused with compression) and
// K2 (per-step prune/compress from a cached mask), plus the small format
// conversion kernels.
//
// Reference: transposable_search_conv (sparsity.py:258-271) scores all 90
// canonical patterns per 4x4 block by summing |w| over the 8 kept positions in
// ascending order in float64 (_core.pyx:98-109) and keeps the first maximum.
// Bit-exactness on the GPU:
//   * fast path (bf16 input, block exponent span <= 13): every |w| becomes an
//     exact integer (mantissa << (exp - emin)); the reference's float64 sums
//     are then exact too (<= 24 significant bits), so integer sums give the
//     identical scores in any order.  The canonical index is packed into the
//     low 7 bits (score << 7 | 127 - t) so one integer max implements
//     "largest score, lowest index on ties".
//   * slow path (larger spans, fp32/fp64 inputs): float64 adds in exactly the
//     reference's order (row 0 pair, row 1 pair, ...), with the row-0/row-1
//     prefix shared across patterns; strict '>' in canonical order.
//
// One CTA = one 128 x 128 tile of W, 8 warps; lane t of warp w owns the four
// horizontally adjacent blocks of rows 16w + 4(t/8) .. +3, columns
// 16(t%8) .. +15.  Loads are 16-byte and coalesced (8 lanes cover a 256-byte
// row segment).  Outputs (fwd values: 16-byte stores; idx: 4-byte stores;
// fwd/bwd metadata tiles and the transposed kept values: staged in shared
// memory, then written as contiguous lines).
#include "s24_common.cuh"
#include "s24_patterns.h"
#include "s24_search_tree.h"
#include "s24_adam.cuh"

namespace s24 {

__constant__ uint16_t c_pat_bits[90] = S24_PATTERN_BITS;

// exactly-two-bit 4-bit mask -> nibble i0 | i1 << 2 (i0 < i1)
__device__ __forceinline__ uint32_t nib_of_mask(uint32_t m4) {
  const uint32_t i0 = __ffs(m4) - 1;
  const uint32_t i1 = 31 - __clz(m4);
  return i0 | (i1 << 2);
}

// transposed 4-bit column masks of a 16-bit pattern mask (bit r of col c)
__device__ __forceinline__ uint32_t col_mask(uint32_t bits16, int c) {
  return ((bits16 >> c) & 1u) | (((bits16 >> (4 + c)) & 1u) << 1) | (((bits16 >> (8 + c)) & 1u) << 2) |
         (((bits16 >> (12 + c)) & 1u) << 3);
}

// ---------------------------------------------------------------------------
// per-block search

// float64 path in the reference's exact accumulation order.  a: |w| row-major.
__device__ __noinline__ int search_block_f64(const double (&a)[16]) {
  constexpr uint16_t kRows[90] = S24_PATTERN_ROWS;
  constexpr int kLo[6] = S24_PAIR_LO;
  constexpr int kHi[6] = S24_PAIR_HI;
  double best = 0.0;
  int best_t = 0;
  double s01 = 0.0;
#pragma unroll
  for (int t = 0; t < 90; ++t) {
    const int p0 = kRows[t] & 15, p1 = (kRows[t] >> 4) & 15, p2 = (kRows[t] >> 8) & 15, p3 = kRows[t] >> 12;
    if (t == 0 || (kRows[t] & 0xFF) != (kRows[t - 1] & 0xFF)) {
      s01 = __dadd_rn(__dadd_rn(__dadd_rn(a[kLo[p0]], a[kHi[p0]]), a[4 + kLo[p1]]), a[4 + kHi[p1]]);
    }
    double s = __dadd_rn(__dadd_rn(s01, a[8 + kLo[p2]]), a[8 + kHi[p2]]);
    s = __dadd_rn(__dadd_rn(s, a[12 + kLo[p3]]), a[12 + kHi[p3]]);
    if (t == 0 || s > best) {
      best = s;
      best_t = t;
    }
  }
  return best_t;
}

// bf16 input: integer fast path with the float64 fallback.  h: raw bf16 bits.
__device__ __forceinline__ int search_block_bf16(const uint16_t (&h)[16]) {
  uint32_t man[16];
  int ee[16];
  int emin = 1 << 20, emax = -1;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t mag = h[i] & 0x7FFFu;
    const int e = static_cast<int>(mag >> 7);
    man[i] = (mag & 0x7Fu) | (e ? 0x80u : 0u);
    ee[i] = e ? e : 1;
    if (man[i]) {
      emin = min(emin, ee[i]);
      emax = max(emax, ee[i]);
    }
  }
  if (emax < 0) return 0;  // all-zero block: every score ties -> pattern 0
  if (emax - emin > 13 || emax == 0xFF) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = static_cast<double>(bf16_to_f32(h[i] & 0x7FFFu));
    return search_block_f64(a);
  }
  int v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = static_cast<int>(man[i] << (ee[i] - emin + 7));
  constexpr int kLo[6] = S24_PAIR_LO;
  constexpr int kHi[6] = S24_PAIR_HI;
  int rp[4][6];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int p = 0; p < 6; ++p) rp[r][p] = v[4 * r + kLo[p]] + v[4 * r + kHi[p]];
  return s24_search_tree(rp);
}

template <int kDType>
struct Elem;
template <>
struct Elem<S24_BF16> {
  using T = uint16_t;
  static constexpr int kVec = 8;  // elements per 16-byte load
};
template <>
struct Elem<S24_F32> {
  using T = float;
  static constexpr int kVec = 4;
};
template <>
struct Elem<S24_F64> {
  using T = double;
  static constexpr int kVec = 2;
};

template <typename T>
__device__ __forceinline__ uint16_t to_bf16_bits(T x);
template <>
__device__ __forceinline__ uint16_t to_bf16_bits<uint16_t>(uint16_t x) {
  return x;
}
template <>
__device__ __forceinline__ uint16_t to_bf16_bits<float>(float x) {
  return f32_to_bf16(x);
}
template <>
__device__ __forceinline__ uint16_t to_bf16_bits<double>(double x) {
  return __bfloat16_as_ushort(__double2bfloat16(x));
}

// ---------------------------------------------------------------------------
// K1 / K2 tile kernel

constexpr int kTile = 128;
constexpr int kThreads = 256;

struct MaskArgs {
  const void* w;
  int64_t rows, cols;
  uint8_t* idx_out;        // K1: written
  const uint8_t* idx_in;   // K2: read
  uint16_t* fwd_vals;      // rows x cols/2
  uint8_t* fwd_e;          // E tiles of W
  uint16_t* bwd_vals;      // cols x rows/2
  uint8_t* bwd_e;          // E tiles of W^T
  int64_t perm_ff;         // >0: gated u/v interleave (output row p reads input row gate_row(p))
};

// Gated first weight W_in = [u; v] (2 d_ff rows) is compressed in an interleaved
// row order: output rows 32g..32g+15 are u rows 16g.., rows 32g+16..32g+31 the
// matching v rows, so one 32-row epilogue warp of GEMM1 holds both halves of
// 16 gate features.  4-row blocks never straddle u/v (16 % 4 == 0), so the
// per-block masks are the reference's masks with block rows permuted.
__host__ __device__ __forceinline__ int64_t gate_row(int64_t p, int64_t perm_ff) {
  const int64_t g = p >> 5, t = p & 31;
  return t < 16 ? 16 * g + t : perm_ff + 16 * g + (t - 16);
}

// kNarrow: bf16 rows that are only 8-byte aligned (cols % 8 == 4) load 4 elements at a time
template <int kDType, bool kSearch, bool kNarrow>
__global__ void __launch_bounds__(kThreads, 2) mask_tile_kernel(MaskArgs p) {
  using T = typename Elem<kDType>::T;
  constexpr int kVec = kNarrow ? 4 : Elem<kDType>::kVec;

  __shared__ __align__(16) uint32_t s_fe[512];        // fwd E tile, 2048 B
  __shared__ __align__(16) uint32_t s_be[512];        // bwd E tile, 2048 B
  __shared__ __align__(16) uint32_t s_bv[128 * 32];   // bwd kept values, 128 x 64 bf16 (swizzled)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tr = blockIdx.y, tc = blockIdx.x;  // tile row / col
  const int br = 4 * warp + (lane >> 3);              // block-row within tile (0..31)
  const int c0 = 16 * (lane & 7);                     // first column within tile
  const int64_t grow0 = tr * kTile + 4 * br;
  const int64_t gcol0 = tc * kTile + c0;
  const bool want_fe = p.fwd_e != nullptr, want_be = p.bwd_e != nullptr, want_bv = p.bwd_vals != nullptr;

  if (want_fe || want_be) {
    for (int i = threadIdx.x; i < 512; i += kThreads) {
      s_fe[i] = 0;
      s_be[i] = 0;
    }
  }
  if (want_fe || want_be || want_bv) __syncthreads();

  const bool row_ok = grow0 < p.rows;
  // ---- load 4 rows x 16 columns ----
  T v[4][16];
  const T* w = static_cast<const T*>(p.w);
  const int64_t in_row0 = p.perm_ff > 0 ? gate_row(grow0, p.perm_ff) : grow0;  // 4-row block stays contiguous
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int q = 0; q < 16 / kVec; ++q) {
      const int64_t col = gcol0 + q * kVec;
      if (row_ok && col < p.cols) {
        if constexpr (kNarrow) {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(w + (in_row0 + i) * p.cols + col));
          const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
          for (int j = 0; j < kVec; ++j) v[i][q * kVec + j] = e[j];
        } else {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(w + (in_row0 + i) * p.cols + col));
          const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
          for (int j = 0; j < kVec; ++j) v[i][q * kVec + j] = e[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < kVec; ++j) v[i][q * kVec + j] = T(0);
      }
    }
  }

  // ---- per block: pattern ----
  int pat[4];
  uint32_t idx_word = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const bool ok = row_ok && (gcol0 + 4 * b) < p.cols;
    int t = 0;
    if constexpr (kSearch) {
      if (ok) {
        if constexpr (kDType == S24_BF16) {
          uint16_t h[16];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) h[4 * i + j] = v[i][4 * b + j];
          t = search_block_bf16(h);
        } else {
          double a[16];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[4 * i + j] = fabs(static_cast<double>(v[i][4 * b + j]));
          t = search_block_f64(a);
        }
      }
    } else {
      if (ok) t = p.idx_in[(grow0 / 4) * (p.cols / 4) + gcol0 / 4 + b];
      if (t > 89) t = 0;  // validated upstream; never index out of the table
    }
    pat[b] = t;
    idx_word |= static_cast<uint32_t>(t) << (8 * b);
  }

  // ---- idx ----
  if (kSearch && row_ok) {
    uint8_t* dst = p.idx_out + (grow0 / 4) * (p.cols / 4) + gcol0 / 4;
    if (gcol0 + 16 <= p.cols && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
      *reinterpret_cast<uint32_t*>(dst) = idx_word;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (gcol0 + 4 * b < p.cols) dst[b] = static_cast<uint8_t>(idx_word >> (8 * b));
    }
  }

  // ---- fwd orientation: kept values along rows + E halfwords ----
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t packed[4];
    uint32_t half = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t m4 = (c_pat_bits[pat[b]] >> (4 * i)) & 0xFu;
      const uint32_t nib = nib_of_mask(m4);
      const int i0 = nib & 3, i1 = nib >> 2;
      uint16_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint16_t bits = to_bf16_bits<T>(v[i][4 * b + j]);
        lo = (j == i0) ? bits : lo;
        hi = (j == i1) ? bits : hi;
      }
      packed[b] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
      half |= nib << (4 * b);
    }
    if (p.fwd_vals != nullptr && row_ok) {
      uint16_t* dst = p.fwd_vals + (grow0 + i) * (p.cols / 2) + gcol0 / 2;
      if (gcol0 + 16 <= p.cols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (gcol0 + 4 * b < p.cols) reinterpret_cast<uint32_t*>(dst)[b] = packed[b];
      }
    }
    if (want_fe) {
      const int m = 4 * br + i;  // tile-local row
      const int L = (m & 7) + 8 * ((c0 & 31) >> 4) + 16 * (m >> 4);
      const int c = c0 >> 5, h = (m >> 3) & 1;
      reinterpret_cast<uint16_t*>(s_fe)[L * 8 + c * 2 + h] = static_cast<uint16_t>(half);
    }
  }

  // ---- bwd orientation (W^T): kept values along columns + E nibbles ----
  if (want_bv || want_be) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t bits16 = c_pat_bits[pat[b]];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t nib = nib_of_mask(col_mask(bits16, j));
        const int i0 = nib & 3, i1 = nib >> 2;
        uint16_t lo = 0, hi = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint16_t bits = to_bf16_bits<T>(v[i][4 * b + j]);
          lo = (i == i0) ? bits : lo;
          hi = (i == i1) ? bits : hi;
        }
        const int mp = c0 + 4 * b + j;  // tile-local row of W^T
        if (want_bv) {
          s_bv[mp * 32 + ((br + 4 * (mp >> 4)) & 31)] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        if (want_be) {
          const int L = (mp & 7) + 16 * (mp >> 4) + 8 * (warp & 1);
          const int c = warp >> 1, h = (mp >> 3) & 1;
          atomicOr(&s_be[L * 4 + c], nib << (16 * h + 4 * (lane >> 3)));
        }
      }
    }
  }

  if (want_fe || want_be || want_bv) __syncthreads();
  const bool full_tile = (tr + 1) * kTile <= p.rows && (tc + 1) * kTile <= p.cols;
  if (want_fe && full_tile) {
    uint4* dst = reinterpret_cast<uint4*>(p.fwd_e + (tr * (p.cols / kTile) + tc) * 2048);
    if (threadIdx.x < 128) dst[threadIdx.x] = reinterpret_cast<const uint4*>(s_fe)[threadIdx.x];
  }
  if (want_be && full_tile) {
    uint4* dst = reinterpret_cast<uint4*>(p.bwd_e + (tc * (p.rows / kTile) + tr) * 2048);
    if (threadIdx.x >= 128) dst[threadIdx.x - 128] = reinterpret_cast<const uint4*>(s_be)[threadIdx.x - 128];
  }
  if (want_bv) {
    // W^T tile: 128 rows x 64 kept values; one warp streams one 128-byte row
    const int64_t kcol = tr * (kTile / 2) + 2 * lane;  // kept-value column
    for (int rr = warp; rr < kTile; rr += kThreads / 32) {
      const int64_t grow_t = tc * kTile + rr;  // row of W^T = column of W
      if (grow_t < p.cols && kcol < p.rows / 2) {
        const uint32_t val = s_bv[rr * 32 + ((lane + 4 * (rr >> 4)) & 31)];
        *reinterpret_cast<uint32_t*>(p.bwd_vals + grow_t * (p.rows / 2) + kcol) = val;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K9+K2 fused: the fp32 optimizer step (Adam + masked decay, optim.py:105-147) of a sparse
// weight with the NEXT step's per-step prune / compress (gated_ffn.py:159-162) in the same
// pass: each thread updates 4 rows x 16 columns (w, u, v in place, 16-byte streaming
// accesses) and compresses the updated values into both orientations exactly as
// mask_tile_kernel does with a cached mask (the E tiles only change at a refresh).  The
// step's K2 launch then disappears from the forward.  Mask / compressed outputs follow the
// operand's row order (perm_ff: the gated u/v interleave); w, u, v, g stay in [u; v] order.
struct AdamCompressArgs {
  float* w;
  float* u;
  float* v;
  const float* g;
  int64_t rows, cols;
  const uint8_t* idx;  // operand order
  uint16_t* fwd_vals;
  uint16_t* bwd_vals;
  int64_t perm_ff;
  AdamScalars s;
};

__global__ void __launch_bounds__(kThreads, 2) adam_compress_kernel(AdamCompressArgs p) {
  __shared__ __align__(16) uint32_t s_bv[128 * 32];  // bwd kept values, 128 x 64 bf16 (swizzled)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tr = blockIdx.y, tc = blockIdx.x;
  const int br = 4 * warp + (lane >> 3);
  const int c0 = 16 * (lane & 7);
  const int64_t grow0 = tr * kTile + 4 * br;  // operand row
  const int64_t gcol0 = tc * kTile + c0;
  const bool ok = grow0 < p.rows && gcol0 < p.cols;  // rows, cols % 128 == 0 (host check)
  int pat[4] = {0, 0, 0, 0};
  if (ok) {
    const uint32_t word = *reinterpret_cast<const uint32_t*>(p.idx + (grow0 / 4) * (p.cols / 4) + gcol0 / 4);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int t = (word >> (8 * b)) & 0xFF;
      pat[b] = t > 89 ? 0 : t;
    }
  }
  float val[4][16];
  const int64_t in_row0 = p.perm_ff > 0 ? gate_row(grow0, p.perm_ff) : grow0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (!ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) val[i][4 * b + j] = 0.0f;
        continue;
      }
      const int64_t e = (in_row0 + i) * p.cols + gcol0 + 4 * b;
      const float4 w4 = __ldcs(reinterpret_cast<const float4*>(p.w + e));
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(p.g + e));
      const float4 u4 = __ldcs(reinterpret_cast<const float4*>(p.u + e));
      const float4 v4 = __ldcs(reinterpret_cast<const float4*>(p.v + e));
      float wv[4] = {w4.x, w4.y, w4.z, w4.w}, gv[4] = {g4.x, g4.y, g4.z, g4.w};
      float uv[4] = {u4.x, u4.y, u4.z, u4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
      const uint32_t keep = (c_pat_bits[pat[b]] >> (4 * i)) & 0xFu;
#pragma unroll
      for (int j = 0; j < 4; ++j) adam_elem<float>(wv[j], uv[j], vv[j], gv[j], !((keep >> j) & 1), p.s);
      __stcs(reinterpret_cast<float4*>(p.w + e), make_float4(wv[0], wv[1], wv[2], wv[3]));
      __stcs(reinterpret_cast<float4*>(p.u + e), make_float4(uv[0], uv[1], uv[2], uv[3]));
      __stcs(reinterpret_cast<float4*>(p.v + e), make_float4(vv[0], vv[1], vv[2], vv[3]));
#pragma unroll
      for (int j = 0; j < 4; ++j) val[i][4 * b + j] = wv[j];
    }
  }
  // fwd orientation: kept values along rows
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t packed[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t nib = nib_of_mask((c_pat_bits[pat[b]] >> (4 * i)) & 0xFu);
      const int i0 = nib & 3, i1 = nib >> 2;
      uint16_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint16_t bits = f32_to_bf16(val[i][4 * b + j]);
        lo = (j == i0) ? bits : lo;
        hi = (j == i1) ? bits : hi;
      }
      packed[b] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    if (ok && p.fwd_vals != nullptr)
      *reinterpret_cast<uint4*>(p.fwd_vals + (grow0 + i) * (p.cols / 2) + gcol0 / 2) =
          make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
  if (p.bwd_vals == nullptr) return;
  // bwd orientation (W^T): kept values along columns, transposed through shared memory
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const uint32_t bits16 = c_pat_bits[pat[b]];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t nib = nib_of_mask(col_mask(bits16, j));
      const int i0 = nib & 3, i1 = nib >> 2;
      uint16_t lo = 0, hi = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint16_t bits = f32_to_bf16(val[i][4 * b + j]);
        lo = (i == i0) ? bits : lo;
        hi = (i == i1) ? bits : hi;
      }
      const int mp = c0 + 4 * b + j;
      s_bv[mp * 32 + ((br + 4 * (mp >> 4)) & 31)] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
  }
  __syncthreads();
  const int64_t kcol = tr * (kTile / 2) + 2 * lane;
  for (int rr = warp; rr < kTile; rr += kThreads / 32) {
    const int64_t grow_t = tc * kTile + rr;
    *reinterpret_cast<uint32_t*>(p.bwd_vals + grow_t * (p.rows / 2) + kcol) =
        s_bv[rr * 32 + ((lane + 4 * (rr >> 4)) & 31)];
  }
}

// ---------------------------------------------------------------------------
// K2 fast path: the per-step prune of bf16 weights into both value orientations
// (metadata cached from the last refresh).  Same outputs as mask_tile_kernel with
// fwd_e = bwd_e = NULL, restructured for bandwidth: 512 threads per 128 x 128
// tile, each owning 4 rows x 8 columns (two 4x4 blocks, one 16-byte load per
// row), so a thread holds 16 data registers and 2-3 CTAs fit per SM.

constexpr int kPruneThreads = 512;

// PRMT selector picking elements i0 < i1 of a 4 x bf16 group held in two words
__device__ __forceinline__ uint32_t pair_selector(uint32_t nib) {
  const uint32_t i0 = nib & 3u, i1 = nib >> 2;
  return (2 * i0) | ((2 * i0 + 1) << 4) | ((2 * i1) << 8) | ((2 * i1 + 1) << 12);
}

// one launch prunes one or two weights (the per-step K2 of W_in and W2): CTAs [0, tiles0) take
// p0's 128 x 128 tiles, the rest p1's
// T = uint16_t: bf16 weights; T = float: fp32 master weights, kept values rounded to bf16 on the
// way in (cvt.rn.bf16x2.f32, the rounding of f32_to_bf16) -- the module's per-step K2 on fp32
// parameters (module.py _prepare_sparse), one pass instead of the general tiled kernel
template <typename T>
__global__ void __launch_bounds__(kPruneThreads, 2) prune_bf16_kernel(MaskArgs p0, MaskArgs p1, int tiles0) {
  __shared__ uint32_t s_bv[128 * 32];  // W^T tile: 128 rows x 32 words (64 kept bf16)
  __shared__ uint4 s_sel[90];          // per pattern: row selectors (x, y), column selectors (z, w)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool second = static_cast<int>(blockIdx.x) >= tiles0;
  const MaskArgs& p = second ? p1 : p0;
  const int64_t bid = second ? blockIdx.x - tiles0 : blockIdx.x;
  const int64_t tiles_x = p.cols / kTile;
  const int64_t tr = bid / tiles_x, tc = bid - tr * tiles_x;
  const int br = 2 * warp + (lane >> 4);  // block row in tile, 0..31
  const int c0 = 8 * (lane & 15);         // first column in tile, 0..120
  const int64_t grow0 = tr * kTile + 4 * br, gcol0 = tc * kTile + c0;
  const int64_t in_row0 = p.perm_ff > 0 ? gate_row(grow0, p.perm_ff) : grow0;
  const T* w = static_cast<const T*>(p.w);
  uint4 v[4];
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __ldg(reinterpret_cast<const uint4*>(w + (in_row0 + i) * p.cols + gcol0));
  } else {
    float4 f[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4* src = reinterpret_cast<const float4*>(w + (in_row0 + i) * p.cols + gcol0);
      f[i][0] = __ldg(src);
      f[i][1] = __ldg(src + 1);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      v[i] = make_uint4(pack_bf16x2(f[i][0].x, f[i][0].y), pack_bf16x2(f[i][0].z, f[i][0].w),
                        pack_bf16x2(f[i][1].x, f[i][1].y), pack_bf16x2(f[i][1].z, f[i][1].w));
  }
  const uint32_t t2 = *reinterpret_cast<const uint16_t*>(p.idx_in + (grow0 / 4) * (p.cols / 4) + gcol0 / 4);
  if (threadIdx.x < 90) {
    const uint32_t bits16 = c_pat_bits[threadIdx.x];
    uint32_t r[4], c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      r[k] = pair_selector(nib_of_mask((bits16 >> (4 * k)) & 0xFu));
      c[k] = pair_selector(nib_of_mask(col_mask(bits16, k)));
    }
    s_sel[threadIdx.x] = make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), c[0] | (c[1] << 16), c[2] | (c[3] << 16));
  }
  __syncthreads();
  uint32_t fw[4][2];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    uint32_t t = (t2 >> (8 * b)) & 0xFFu;
    const uint4 sel = s_sel[t > 89 ? 0 : t];
    // fwd orientation: row i keeps 2 of its 4 elements (one byte permute)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t si = ((i < 2 ? sel.x : sel.y) >> (16 * (i & 1))) & 0xFFFFu;
      fw[i][b] = __byte_perm((&v[i].x)[2 * b], (&v[i].x)[2 * b + 1], si);
    }
    // bwd orientation (W^T): transpose column j into two words, then keep 2 of 4.
    // Word (mp, br) sits at mp * 32 + (br + 2 (mp / 8)) % 32: the 32 lanes of a
    // warp (16 column strips x 2 block rows) hit 32 distinct banks.
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int wj = 2 * b + (j >> 1);
      const uint32_t hsel = (j & 1) ? 0x7632u : 0x5410u;
      const uint32_t col01 = __byte_perm((&v[0].x)[wj], (&v[1].x)[wj], hsel);
      const uint32_t col23 = __byte_perm((&v[2].x)[wj], (&v[3].x)[wj], hsel);
      const uint32_t sj = ((j < 2 ? sel.z : sel.w) >> (16 * (j & 1))) & 0xFFFFu;
      const int mp = c0 + 4 * b + j;
      s_bv[mp * 32 + ((br + 2 * (mp >> 3)) & 31)] = __byte_perm(col01, col23, sj);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint2*>(p.fwd_vals + (grow0 + i) * (p.cols / 2) + gcol0 / 2) = make_uint2(fw[i][0], fw[i][1]);
  __syncthreads();
  const int64_t kcol = tr * (kTile / 2) + 2 * lane;
#pragma unroll 4
  for (int rr = warp; rr < kTile; rr += kPruneThreads / 32) {
    const uint32_t val = s_bv[rr * 32 + ((lane + 2 * (rr >> 3)) & 31)];
    *reinterpret_cast<uint32_t*>(p.bwd_vals + (tc * kTile + rr) * (p.rows / 2) + kcol) = val;
  }
}

// ---------------------------------------------------------------------------
// K1 fast path: bf16 search fused with compression for tile-aligned weights.
// Same thread map as prune_bf16_kernel (4 rows x 8 columns = two 4x4 blocks per
// thread); kept values via byte permutes, metadata nibbles from a per-pattern
// table, E-tile bytes assembled without shared-memory atomics.

// integer search on one block given as 4 rows x 2 words (bf16 pairs).  Returns the pattern, or
// -1 when the block needs the float64 reference-order path (exponent span > 13, tiny values) and
// -2 when it holds inf / nan (the owner lane then runs the sequential reference loop itself)
// one = 1 from a kernel argument (opaque to the compiler): the products by `one` / `128 one` below
// compile to IMAD, which issues on the FMA pipe, instead of IADD3 / LEA on the integer ALU pipe --
// the search is ALU-pipe bound and the FMA pipe is mostly idle
__device__ __forceinline__ int search_block_fast(const uint32_t (&wd)[8], int one) {
  uint32_t h[16];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k) h[4 * r + k] = (wd[2 * r + (k >> 1)] >> (16 * (k & 1))) & 0x7FFFu;
  // magnitudes as exact f32; positive float bits order like the values, so the
  // exponent range over nonzero entries comes from integer max / min(bits - 1)
  float f[16];
  uint32_t bmax = 0, bmin1 = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t fb = h[i] << 16;
    f[i] = __uint_as_float(fb);
    bmax = max(bmax, fb);
    bmin1 = min(bmin1, fb - 1u);
  }
  if (bmax == 0) return 0;  // all-zero block: every score ties -> pattern 0
  const int emax = static_cast<int>(bmax >> 23), emin = static_cast<int>((bmin1 + 1u) >> 23);
  if (emax == 0xFF) return -2;
  // span > 13 (sums need > 24 bits) or tiny values (scale not representable): float64 path
  if (emax - emin > 13 || emin < 8) return -1;
  // |w| * 2^(134 - emin) is an integer < 2^21 (8-bit significand, span <= 13);
  // adding 1.5 * 2^23 puts it in the low mantissa bits exactly, and the integer
  // is pre-scaled by 128 for the tie-break bits: v = (bits - 0x4B400000) << 7
  const float scale = __uint_as_float(static_cast<uint32_t>(261 - emin) << 23);
  int v[16];
  const int k128 = one << 7;
#pragma unroll
  for (int i = 0; i < 16; ++i)
    v[i] = static_cast<int>(__float_as_uint(__fmaf_rn(f[i], scale, 12582912.0f))) * k128 -
           static_cast<int>(0x4B400000u << 7);
  constexpr int kLo[6] = S24_PAIR_LO;
  constexpr int kHi[6] = S24_PAIR_HI;
  int rp[4][6];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < 6; ++q) rp[r][q] = v[4 * r + kLo[q]] * one + v[4 * r + kHi[q]];
  return s24_search_tree(rp);
}

__device__ __forceinline__ void block_abs_f64(const uint32_t (&wd)[8], double (&a)[16]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      a[4 * r + k] = static_cast<double>(__uint_as_float(((wd[2 * r + (k >> 1)] >> (16 * (k & 1))) & 0x7FFFu) << 16));
}

__constant__ uint16_t c_pat_rows[90] = S24_PATTERN_ROWS;

// The float64 reference-order search of one block with finite values, warp-cooperatively (the
// north-star's warp-shuffle argmax): lane l scores patterns l, l + 32, l + 64 with the
// reference's sequential adds over the 8 kept positions (_core.pyx:98-109), then a butterfly
// reduction keeps the largest score and, on equal scores, the lowest pattern index -- for
// finite scores exactly the reference's first strict maximum.  wd is warp-uniform.
__device__ __noinline__ int search_block_f64_warp(const uint32_t (&wd)[8], int lane) {
  double a[16];
  block_abs_f64(wd, a);
  double best = 0.0;
  int bt = 127;  // none
#pragma unroll
  for (int rr = 0; rr < 3; ++rr) {
    const int t = lane + 32 * rr;
    if (t < 90) {
      const uint32_t rows = c_pat_rows[t];
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t q = (rows >> (4 * r)) & 15u;
        const int lo = static_cast<int>((0x000112u >> (4 * q)) & 15u), hi = static_cast<int>((0x123233u >> (4 * q)) & 15u);
        s = r == 0 ? __dadd_rn(a[lo], a[hi]) : __dadd_rn(__dadd_rn(s, a[4 * r + lo]), a[4 * r + hi]);
      }
      if (bt == 127 || s > best) {
        best = s;
        bt = t;
      }
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
    const int ot = __shfl_xor_sync(0xFFFFFFFFu, bt, off);
    if (ot != 127 && (bt == 127 || ob > best || (ob == best && ot < bt))) {
      best = ob;
      bt = ot;
    }
  }
  return bt;
}

// Persistent K1 with warp-owned strips.  A CTA of 4 warps owns one SUPER-TILE at a time: two
// horizontally adjacent 128 x 128 tiles (one when the weight has an odd number of tile columns),
// super-tiles blockIdx.x, + gridDim.x, ... over p0's, then p1's.  Warp a owns rows 32 a .. 32 a
// + 31 and sweeps them in PASSES of 32 columns (4 per tile; lane = (block row lane / 4, column
// group lane % 4) holds two 4x4 blocks of a pass, 4 rows x 16 bytes).  Every lane streams its
// 4 x 16 bytes of the pass two ahead into its own shared-memory slots with cp.async while it
// searches the current one.  Every output leaves in whole 32-byte sectors (a partial-sector
// write that misses L2 costs a DRAM read to fill the sector):
//   fwd_vals  4 rows x 8 bytes per lane and pass (4 lanes = one row's 32-byte segment);
//   bwd_vals  8 W^T rows x 4 bytes per lane and pass (8 lanes = one W^T row's 32-byte segment);
//   fwd E     the warp's 32 rows are 32 whole metadata lines per tile: lane (m & 7, kpar, m >> 4)
//             gathers one 4-byte word of its line per pass (4 shuffles), stores the line once;
//   idx       8 bytes per lane per tile after a 4-lane exchange;
//   bwd E     a W^T metadata line spans all 128 rows (all four warps): per pass each lane's word
//             comes out of an 8 x 8 nibble transpose (one gather shuffle + three butterfly
//             stages), is staged in shared memory, and the tiles leave as 16-byte lines after the
//             super-tile's one 4-warp barrier (one barrier per 8 passes).
// Blocks whose exponent span needs the float64 reference-order path are searched after the fast
// path by the whole warp together (search_block_f64_warp, the north-star's warp-shuffle argmax).
constexpr int kK1Threads = 128;  // 4 warps per CTA
#ifndef S24_K1_MINB
#define S24_K1_MINB 6  // CTAs per SM (6: 80 registers per thread, no spills)
#endif
constexpr int kK1Depth = 3;      // input slots per lane: the current pass + two in flight
struct K1Smem {
  uint4 in[kK1Depth][4][kK1Threads];  // 24 KB: slot (buffer, row i, thread)
  uint32_t be[2][2][512];             // bwd E staging: [super-tile parity][tile of the pair]
  uint4 sel[90];                      // per pattern: row selectors (x, y), column selectors (z, w)
  uint2 nib[90];                      // per pattern: x = fwd row nibble i at bits 8 i, y = bwd column nibbles
};
constexpr int kK1SmemBytes = static_cast<int>(sizeof(K1Smem));

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait2() { asm volatile("cp.async.wait_group 2;" ::: "memory"); }

struct K1Pos {
  int which;         // 0: p0, 1: p1, -1: past the end
  int ntile;         // tiles in this super-tile (1 or 2)
  uint32_t tr, tc0;  // first tile of the super-tile
};

// super-tile t of the concatenated list; sx = super-tiles per tile row, pair = 2-tile super-tiles
__device__ __forceinline__ K1Pos k1_pos(uint32_t t, uint32_t st0, uint32_t total, uint32_t sx0, uint32_t sx1,
                                        int pair0, int pair1) {
  K1Pos q{-1, 1, 0, 0};
  if (t >= total) return q;
  const bool second = t >= st0;
  const uint32_t b = second ? t - st0 : t, sx = second ? sx1 : sx0;
  const int pr = second ? pair1 : pair0;
  q.which = second ? 1 : 0;
  q.ntile = pr ? 2 : 1;
  q.tr = b / sx;
  q.tc0 = (b - q.tr * sx) * (pr ? 2 : 1);
  return q;
}

// lane j of an 8-lane group holds row j of an 8 x 8 nibble matrix (nibble c at bits 4 c); after
// the three butterfly stages it holds column j (nibble c = row c's nibble j)
__device__ __forceinline__ uint32_t nibble_transpose8(uint32_t x, int j) {
#pragma unroll
  for (int sdist = 4; sdist >= 1; sdist >>= 1) {
    const uint32_t keep = sdist == 4 ? 0x0000FFFFu : sdist == 2 ? 0x00FF00FFu : 0x0F0F0F0Fu;
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, sdist);
    x = (j & sdist) ? ((x & ~keep) | ((y & ~keep) >> (4 * sdist))) : ((x & keep) | ((y & keep) << (4 * sdist)));
  }
  return x;
}

__global__ void __launch_bounds__(kK1Threads, S24_K1_MINB) search_bf16_kernel(MaskArgs p0, MaskArgs p1,
                                                                               uint32_t st0, uint32_t total,
                                                                               int pairs, int one) {
  extern __shared__ __align__(16) uint8_t k1_raw[];
  K1Smem& S = *reinterpret_cast<K1Smem*>(k1_raw);
  const int tid = threadIdx.x, lane = tid & 31, wa = tid >> 5;  // warp = row strip of the tile
  const int br = lane >> 2;  // block row in the strip, 0..7
  const int g = lane & 3;    // column group (8 columns = two blocks), 0..3
  if (tid < 90) {
    const uint32_t bits16 = c_pat_bits[tid];
    uint32_t r[4], c[4], nf = 0, nb = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t rn = nib_of_mask((bits16 >> (4 * k)) & 0xFu), cn = nib_of_mask(col_mask(bits16, k));
      r[k] = pair_selector(rn);
      c[k] = pair_selector(cn);
      nf |= rn << (8 * k);
      nb |= cn << (4 * k);
    }
    S.sel[tid] = make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), c[0] | (c[1] << 16), c[2] | (c[3] << 16));
    S.nib[tid] = make_uint2(nf, nb);
  }
  const int pair0 = pairs & 1, pair1 = (pairs >> 1) & 1;
  const uint32_t sx0 = static_cast<uint32_t>(p0.cols >> 7) / (pair0 ? 2 : 1);
  const uint32_t sx1 = static_cast<uint32_t>(p1.cols >> 7) / (pair1 ? 2 : 1);

  // pass sequence of this CTA: super-tile blockIdx.x + k gridDim.x, passes 0 .. 4 ntile - 1
  auto prefetch = [&](const K1Pos& q, int pp, int buf) {
    if (q.which >= 0) {
      const MaskArgs& a = q.which ? p1 : p0;
      const uint64_t cols = static_cast<uint64_t>(a.cols);
      const uint32_t grow0 = 128 * q.tr + 32 * wa + 4 * br;
      const uint32_t in_row0 = a.perm_ff > 0 ? static_cast<uint32_t>(gate_row(grow0, a.perm_ff)) : grow0;
      const uint16_t* src = static_cast<const uint16_t*>(a.w) + (in_row0 * cols + 128 * q.tc0 + 32 * pp + 8 * g);
#pragma unroll
      for (int i = 0; i < 4; ++i) cp_async16(&S.in[buf][i][tid], src + i * cols);
    }
    cp_async_commit();  // (possibly empty) group: wait_group 2 below always means "the current pass"
  };

  uint32_t t = blockIdx.x;
  K1Pos cur = k1_pos(t, st0, total, sx0, sx1, pair0, pair1);
  K1Pos nxt = k1_pos(t + gridDim.x, st0, total, sx0, sx1, pair0, pair1);
  prefetch(cur, 0, 0);
  prefetch(cur.ntile * 4 > 1 ? cur : nxt, 1, 1);
  __syncthreads();  // tables ready
  int buf = 0, sslot = 0;
  uint32_t f0 = 0, f1 = 0, f2 = 0, f3 = 0;  // fwd E line words of the tile's passes 0..3
  uint64_t idx_acc = 0;                      // the lane's 2-byte idx chunk of the tile's passes 0..3
  // bwd E transpose roles: lane = (q2, mhi, k) of its line word, gather source row k
  const int tk = lane & 7, tmhi = (lane >> 3) & 1, tq2 = lane >> 4;
  const int tsrc = 4 * (4 * tq2 + (tk & 3)) + 2 * tmhi + (tk >> 2);
  while (cur.which >= 0) {
    const MaskArgs& p = cur.which ? p1 : p0;
    const uint32_t rows = static_cast<uint32_t>(p.rows), cols = static_cast<uint32_t>(p.cols);
    const int npass = 4 * cur.ntile;
#pragma unroll 1
    for (int pp = 0; pp < npass; ++pp) {
      // prefetch pass pp + 2 (this super-tile's, or the next one's first passes)
      if (pp + 2 < npass) prefetch(cur, pp + 2, buf == 0 ? 2 : buf - 1);
      else prefetch(nxt, pp + 2 - npass, buf == 0 ? 2 : buf - 1);
      cp_async_wait2();  // this lane's slot of the current pass has landed
      uint4 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = S.in[buf][i][tid];

      // ---- search: integer fast path per lane, then the float64 blocks warp-cooperatively ----
      int pat[2];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        uint32_t wd[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          wd[2 * i] = (&v[i].x)[2 * b];
          wd[2 * i + 1] = (&v[i].x)[2 * b + 1];
        }
        pat[b] = search_block_fast(wd, one);
        if (pat[b] == -2) {  // inf / nan: the sequential reference loop (its own comparison semantics)
          double a[16];
          block_abs_f64(wd, a);
          pat[b] = search_block_f64(a);
        }
      }
      unsigned slow0 = __ballot_sync(0xFFFFFFFFu, pat[0] < 0), slow1 = __ballot_sync(0xFFFFFFFFu, pat[1] < 0);
      while (slow0 | slow1) {  // warp-uniform
        const int b = slow0 ? 0 : 1;
        const int owner = __ffs(b ? slow1 : slow0) - 1;
        if (b) slow1 &= slow1 - 1;
        else slow0 &= slow0 - 1;
        uint32_t wd[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          wd[2 * i] = __shfl_sync(0xFFFFFFFFu, b ? v[i].z : v[i].x, owner);
          wd[2 * i + 1] = __shfl_sync(0xFFFFFFFFu, b ? v[i].w : v[i].y, owner);
        }
        const int tt = search_block_f64_warp(wd, lane);
        if (lane == owner) {
          if (b) pat[1] = tt;
          else pat[0] = tt;
        }
      }

      const int tile = pp >> 2, pass = pp & 3;
      const uint32_t grow0 = 128 * cur.tr + 32 * wa + 4 * br, gcol0 = 128 * cur.tc0 + 32 * pp + 8 * g;
      idx_acc = (idx_acc >> 16) | (static_cast<uint64_t>(pat[0] | (pat[1] << 8)) << 48);
      const uint2 n0 = S.nib[pat[0]], n1 = S.nib[pat[1]];
      {  // fwd E: byte i of fb = row 4 br + i of the lane's 8 columns (block 0 | block 1 << 4)
        const uint32_t fb = n0.x | (n1.x << 4);
        // lane -> line (m & 7, kpar, m >> 4): rows m, m + 8 x column groups 2 kpar, 2 kpar + 1
        const int m7 = lane & 7, kp = (lane >> 3) & 1, mhi = lane >> 4;
        const int br0 = 4 * mhi + (m7 >> 2), i = m7 & 3;
        const int la = 4 * br0 + 2 * kp, lb = la + 8;  // block rows br0 and br0 + 2
        const uint32_t a0 = __shfl_sync(0xFFFFFFFFu, fb, la), a1 = __shfl_sync(0xFFFFFFFFu, fb, la + 1);
        const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, fb, lb), b1 = __shfl_sync(0xFFFFFFFFu, fb, lb + 1);
        const uint32_t lo = __byte_perm(a0, a1, i | ((i + 4) << 4)), hi = __byte_perm(b0, b1, i | ((i + 4) << 4));
        f0 = f1;
        f1 = f2;
        f2 = f3;
        f3 = (lo & 0xFFFFu) | (hi << 16);
      }
      if (p.bwd_e) {
        // the lane's 8 column nibbles (block 0: columns 0-3, block 1: 4-7) are one row of an 8 x 8
        // nibble matrix per (q2, mhi) group; lane (q2, mhi, k) needs column k: nibble 4 h + bb =
        // column nibble k of block row 4 q2 + bb, column group 2 mhi + h
        const uint32_t mine = n0.y | (n1.y << 16);
        const uint32_t word = nibble_transpose8(__shfl_sync(0xFFFFFFFFu, mine, tsrc), tk);
        // nibble j of word = source row j = (bb = j & 3, h = j >> 2) -> bits 16 h + 4 bb: as stored
        S.be[sslot][tile][(tk + 16 * (2 * pass + tmhi) + 8 * tq2) * 4 + wa] = word;
      }
      uint32_t fw[4][2];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const uint4 sel = S.sel[pat[b]];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t si = ((i < 2 ? sel.x : sel.y) >> (16 * (i & 1))) & 0xFFFFu;
          fw[i][b] = __byte_perm((&v[i].x)[2 * b], (&v[i].x)[2 * b + 1], si);
        }
        if (p.bwd_vals) {
          // W^T row = column gcol0 + 4 b + jj, the block row's two kept values at element grow0 / 2
          uint16_t* bv = p.bwd_vals + (static_cast<uint64_t>(gcol0 + 4 * b) * (rows >> 1) + (grow0 >> 1));
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int wj = 2 * b + (jj >> 1);
            const uint32_t hsel = (jj & 1) ? 0x7632u : 0x5410u;
            const uint32_t col01 = __byte_perm((&v[0].x)[wj], (&v[1].x)[wj], hsel);
            const uint32_t col23 = __byte_perm((&v[2].x)[wj], (&v[3].x)[wj], hsel);
            const uint32_t sj = ((jj < 2 ? sel.z : sel.w) >> (16 * (jj & 1))) & 0xFFFFu;
            *reinterpret_cast<uint32_t*>(bv + static_cast<uint64_t>(jj) * (rows >> 1)) = __byte_perm(col01, col23, sj);
          }
        }
      }
      if (p.fwd_vals) {
        uint16_t* fv = p.fwd_vals + (static_cast<uint64_t>(grow0) * (cols >> 1) + (gcol0 >> 1));
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint2*>(fv + static_cast<uint64_t>(i) * (cols >> 1)) = make_uint2(fw[i][0], fw[i][1]);
      }
      if (pass == 3) {  // ---- per tile: fwd E lines, idx ----
        const uint32_t tr = cur.tr, tc = cur.tc0 + tile;
        if (p.fwd_e) {
          const int L = (lane & 7) + 8 * ((lane >> 3) & 1) + 16 * (2 * wa + (lane >> 4));
          *reinterpret_cast<uint4*>(p.fwd_e + (static_cast<uint64_t>(tr) * (cols >> 7) + tc) * 2048 + L * 16) =
              make_uint4(f0, f1, f2, f3);
        }
        if (p.idx_out) {
          // lane (br, g) stores block columns 8 g .. 8 g + 7 of its block row: pass g's chunks of lanes (br, 0..3)
          uint32_t part[4];
#pragma unroll
          for (int gg = 0; gg < 4; ++gg) {
            const uint64_t x = __shfl_sync(0xFFFFFFFFu, idx_acc, 4 * br + gg);
            part[gg] = static_cast<uint32_t>(x >> (16 * g)) & 0xFFFFu;
          }
          const uint32_t brow = 32 * tr + 8 * wa + br;
          *reinterpret_cast<uint2*>(p.idx_out + static_cast<uint64_t>(brow) * (cols >> 2) + 32 * tc + 8 * g) =
              make_uint2(part[0] | (part[1] << 16), part[2] | (part[3] << 16));
        }
      }
      buf = buf == kK1Depth - 1 ? 0 : buf + 1;
    }
    // ---- per super-tile: the bwd E tiles ----
    __syncthreads();  // the super-tile's bwd E words from all four warps are staged
    if (p.bwd_e) {
      for (int tl = 0; tl < cur.ntile; ++tl)
        reinterpret_cast<uint4*>(p.bwd_e + (static_cast<uint64_t>(cur.tc0 + tl) * (rows >> 7) + cur.tr) * 2048)[tid] =
            reinterpret_cast<const uint4*>(S.be[sslot][tl])[tid];
    }
    sslot ^= 1;
    t += gridDim.x;
    cur = nxt;
    nxt = k1_pos(t + gridDim.x, st0, total, sx0, sx1, pair0, pair1);
  }
}

// persistent grid: S24_K1_MINB 4-warp CTAs per SM (the kernel's register footprint)
// super-tiles: pairs of horizontally adjacent 128 x 128 tiles (one barrier per 8 passes) when the
// launch has many tiles per CTA and the weight an even number of tile columns, else single tiles
// (small weights need every CTA: C2's 512 tiles run as 512 CTAs)
static int64_t k1_super_tiles(int64_t rows, int64_t cols, bool pair) {
  const int64_t tx = cols / kTile;
  return (rows / kTile) * (pair ? tx / 2 : tx);
}
static bool k1_pairable(int64_t cols, int64_t tiles_total) {
  return (cols / kTile) % 2 == 0 && tiles_total >= 4LL * S24_K1_MINB * 148;
}

static int k1_grid(long long tiles) {
  const long long total = tiles;  // one super-tile per CTA at a time
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(search_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kK1SmemBytes);
    sms[dev] = n > 0 ? n : 148;
  }
  return static_cast<int>(total < S24_K1_MINB * sms[dev] ? total : S24_K1_MINB * sms[dev]);
}

// ---------------------------------------------------------------------------
// small conversion kernels

__global__ void idx_to_bits_kernel(const uint8_t* __restrict__ idx, int64_t rows, int64_t cols,
                                   uint8_t* __restrict__ bits) {
  const int64_t nb = (rows / 4) * (cols / 4);
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bi = b / (cols / 4), bj = b % (cols / 4);
    const uint32_t pb = c_pat_bits[min(static_cast<int>(idx[b]), 89)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t m4 = (pb >> (4 * r)) & 0xF;
      const uint32_t word = (m4 & 1) | ((m4 & 2) << 7) | ((m4 & 4) << 14) | ((m4 & 8) << 21);
      *reinterpret_cast<uint32_t*>(bits + (4 * bi + r) * cols + 4 * bj) = word;
    }
  }
}

__global__ void bits_to_idx_kernel(const uint8_t* __restrict__ bits, int64_t rows, int64_t cols,
                                   uint8_t* __restrict__ idx, int32_t* bad) {
  const int64_t nb = (rows / 4) * (cols / 4);
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bi = b / (cols / 4), bj = b % (cols / 4);
    uint32_t m16 = 0;
    bool ok = true;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint8_t x = bits[(4 * bi + r) * cols + 4 * bj + c];
        ok = ok && x <= 1;
        m16 |= static_cast<uint32_t>(x & 1) << (4 * r + c);
      }
    int found = 255;
    if (ok) {
      for (int t = 0; t < 90; ++t)
        if (c_pat_bits[t] == m16) {
          found = t;
          break;
        }
    }
    idx[b] = static_cast<uint8_t>(found);
    if (found == 255) atomicAdd(bad, 1);
  }
}

__global__ void meta_flat_kernel(const uint8_t* __restrict__ idx, int64_t rows, int64_t cols,
                                 uint8_t* __restrict__ fwd, uint8_t* __restrict__ bwd) {
  const int64_t nb = (rows / 4) * (cols / 4);
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bi = b / (cols / 4), bj = b % (cols / 4);
    const uint32_t pb = c_pat_bits[min(static_cast<int>(idx[b]), 89)];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (fwd) fwd[(4 * bi + r) * (cols / 4) + bj] = static_cast<uint8_t>(nib_of_mask((pb >> (4 * r)) & 0xF));
      if (bwd) bwd[(4 * bj + r) * (rows / 4) + bi] = static_cast<uint8_t>(nib_of_mask(col_mask(pb, r)));
    }
  }
}

__global__ void e_to_flat_kernel(const uint8_t* __restrict__ e, int64_t m, int64_t k, uint8_t* __restrict__ meta) {
  const int64_t ng = m * (k / 4);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = g / (k / 4), grp = g % (k / 4);
    const int64_t tile = (row / 128) * (k / 128) + (grp * 4) / 128;
    const int mm = row % 128, kk = (grp * 4) % 128;
    const int L = (mm & 7) + 8 * ((kk & 31) >> 4) + 16 * (mm >> 4);
    const int c = kk >> 5, h = (mm >> 3) & 1, gsub = (kk & 15) >> 2;
    const uint16_t word = *reinterpret_cast<const uint16_t*>(e + tile * 2048 + L * 16 + c * 4 + h * 2);
    meta[g] = static_cast<uint8_t>((word >> (4 * gsub)) & 0xF);
  }
}

__global__ void masked_decay_kernel(float* __restrict__ g, const void* __restrict__ w, int w_dtype,
                                    const uint8_t* __restrict__ idx, int64_t rows, int64_t cols, float lam) {
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    const uint32_t pb = c_pat_bits[min(static_cast<int>(idx[(r / 4) * (cols / 4) + c / 4]), 89)];
    if ((pb >> (4 * (r & 3) + (c & 3))) & 1) continue;
    float wv;
    if (w_dtype == S24_BF16)
      wv = bf16_to_f32(static_cast<const uint16_t*>(w)[e]);
    else if (w_dtype == S24_F32)
      wv = static_cast<const float*>(w)[e];
    else
      wv = static_cast<float>(static_cast<const double*>(w)[e]);
    g[e] = g[e] + lam * wv;
  }
}

// the same decay under an arbitrary 0/1 mask of any shape (flat, element-aligned): the
// reference's masked_decay_gradient on a flat parameter vector (optim.py:105-114, trainer.py:441)
__global__ void masked_decay_bits_kernel(float* __restrict__ g, const void* __restrict__ w, int w_dtype,
                                         const uint8_t* __restrict__ bits, int64_t n, float lam) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    if (bits[e]) continue;
    float wv;
    if (w_dtype == S24_BF16)
      wv = bf16_to_f32(static_cast<const uint16_t*>(w)[e]);
    else if (w_dtype == S24_F32)
      wv = static_cast<const float*>(w)[e];
    else
      wv = static_cast<float>(static_cast<const double*>(w)[e]);
    g[e] = g[e] + lam * wv;
  }
}

}  // namespace s24

using namespace s24;

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

static int check_w(const void* w, int dtype, int64_t rows, int64_t cols) {
  S24_REQUIRE(w != nullptr, S24_ERR_ARG, "weight pointer is NULL");
  S24_REQUIRE(dtype == S24_BF16 || dtype == S24_F32 || dtype == S24_F64, S24_ERR_UNSUPPORTED,
              "unsupported weight dtype %d", dtype);
  S24_REQUIRE(rows >= 0 && cols >= 0 && rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE,
              "shape (%lld, %lld) not divisible into 4x4 blocks", (long long)rows, (long long)cols);
  S24_REQUIRE((reinterpret_cast<uintptr_t>(w) & 15) == 0, S24_ERR_UNSUPPORTED,
              "weight base pointer must be 16-byte aligned");
  return S24_OK;
}

static int launch_mask(const MaskArgs& a, int dtype, bool search, cudaStream_t st) {
  if (a.rows == 0 || a.cols == 0) return S24_OK;
  dim3 grid(static_cast<unsigned>((a.cols + kTile - 1) / kTile), static_cast<unsigned>((a.rows + kTile - 1) / kTile));
  const bool narrow = dtype == S24_BF16 && (a.cols % 8) != 0;
  const bool aligned = a.rows % kTile == 0 && a.cols % kTile == 0;
  if (search) {
    if (dtype == S24_BF16 && aligned) {
      if (a.rows * a.cols < (int64_t(1) << 32)) {
        const bool pr = k1_pairable(a.cols, (a.rows / kTile) * (a.cols / kTile));
        const uint32_t nst = static_cast<uint32_t>(k1_super_tiles(a.rows, a.cols, pr));
        search_bf16_kernel<<<k1_grid(nst), kK1Threads, kK1SmemBytes, st>>>(a, a, nst, nst, pr ? 3 : 0, 1);
        return s24_check_launch("mask_search");
      }
      mask_tile_kernel<S24_BF16, true, false><<<grid, kThreads, 0, st>>>(a);
      return s24_check_launch("mask_search");
    }
    if (narrow) mask_tile_kernel<S24_BF16, true, true><<<grid, kThreads, 0, st>>>(a);
    else if (dtype == S24_BF16) mask_tile_kernel<S24_BF16, true, false><<<grid, kThreads, 0, st>>>(a);
    else if (dtype == S24_F32) mask_tile_kernel<S24_F32, true, false><<<grid, kThreads, 0, st>>>(a);
    else mask_tile_kernel<S24_F64, true, false><<<grid, kThreads, 0, st>>>(a);
  } else {
    if ((dtype == S24_BF16 || dtype == S24_F32) && a.fwd_e == nullptr && a.bwd_e == nullptr &&
        a.fwd_vals != nullptr && a.bwd_vals != nullptr && aligned) {
      const int tiles = static_cast<int>(grid.x * grid.y);
      if (dtype == S24_BF16) prune_bf16_kernel<uint16_t><<<tiles, kPruneThreads, 0, st>>>(a, a, tiles);
      else prune_bf16_kernel<float><<<tiles, kPruneThreads, 0, st>>>(a, a, tiles);
      return s24_check_launch("prune_compress");
    }
    if (narrow) mask_tile_kernel<S24_BF16, false, true><<<grid, kThreads, 0, st>>>(a);
    else if (dtype == S24_BF16) mask_tile_kernel<S24_BF16, false, false><<<grid, kThreads, 0, st>>>(a);
    else if (dtype == S24_F32) mask_tile_kernel<S24_F32, false, false><<<grid, kThreads, 0, st>>>(a);
    else mask_tile_kernel<S24_F64, false, false><<<grid, kThreads, 0, st>>>(a);
  }
  return s24_check_launch(search ? "mask_search" : "prune_compress");
}

extern "C" int s24_transposable_search(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx,
                                       void* stream) {
  if (int rc = check_w(w, dtype, rows, cols)) return rc;
  S24_REQUIRE(idx != nullptr, S24_ERR_ARG, "idx pointer is NULL");
  MaskArgs a{w, rows, cols, idx, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return launch_mask(a, dtype, true, static_cast<cudaStream_t>(stream));
}

static int check_compress_outputs(int64_t rows, int64_t cols, const void* fwd_e, const void* bwd_e) {
  if (fwd_e != nullptr || bwd_e != nullptr)
    S24_REQUIRE(rows % 128 == 0 && cols % 128 == 0, S24_ERR_SHAPE,
                "tensor-core metadata tiles need rows and cols divisible by 128, got (%lld, %lld)",
                (long long)rows, (long long)cols);
  return S24_OK;
}

static int check_perm(int64_t rows, int64_t perm_ff) {
  if (perm_ff > 0)
    S24_REQUIRE(rows == 2 * perm_ff && perm_ff % 16 == 0, S24_ERR_SHAPE,
                "gated interleave needs rows == 2 * d_ff and d_ff %% 16 == 0 (rows=%lld d_ff=%lld)", (long long)rows,
                (long long)perm_ff);
  return S24_OK;
}

extern "C" int s24_search_compress(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx,
                                   uint16_t* fwd_vals, uint8_t* fwd_e, uint16_t* bwd_vals, uint8_t* bwd_e,
                                   int64_t perm_ff, void* stream) {
  if (int rc = check_perm(rows, perm_ff)) return rc;
  if (int rc = check_w(w, dtype, rows, cols)) return rc;
  S24_REQUIRE(idx != nullptr, S24_ERR_ARG, "idx pointer is NULL");
  if (int rc = check_compress_outputs(rows, cols, fwd_e, bwd_e)) return rc;
  MaskArgs a{w, rows, cols, idx, nullptr, fwd_vals, fwd_e, bwd_vals, bwd_e, perm_ff};
  return launch_mask(a, dtype, true, static_cast<cudaStream_t>(stream));
}

extern "C" int s24_prune_compress(const void* w, int dtype, int64_t rows, int64_t cols, const uint8_t* idx,
                                  uint16_t* fwd_vals, uint8_t* fwd_e, uint16_t* bwd_vals, uint8_t* bwd_e,
                                  int64_t perm_ff, void* stream) {
  if (int rc = check_perm(rows, perm_ff)) return rc;
  if (int rc = check_w(w, dtype, rows, cols)) return rc;
  S24_REQUIRE(idx != nullptr, S24_ERR_ARG, "idx pointer is NULL");
  if (int rc = check_compress_outputs(rows, cols, fwd_e, bwd_e)) return rc;
  MaskArgs a{w, rows, cols, nullptr, idx, fwd_vals, fwd_e, bwd_vals, bwd_e, perm_ff};
  return launch_mask(a, dtype, false, static_cast<cudaStream_t>(stream));
}

extern "C" int s24_prune_compress_pair(const void* w0, const void* w1, int dtype, int64_t rows0, int64_t cols0,
                                       int64_t rows1, int64_t cols1, const uint8_t* idx0, const uint8_t* idx1,
                                       uint16_t* fwd_vals0, uint16_t* bwd_vals0, uint16_t* fwd_vals1,
                                       uint16_t* bwd_vals1, int64_t perm_ff0, int64_t perm_ff1, void* stream) {
  if (int rc = check_w(w0, dtype, rows0, cols0)) return rc;
  if (int rc = check_w(w1, dtype, rows1, cols1)) return rc;
  S24_REQUIRE(idx0 && idx1 && fwd_vals0 && bwd_vals0 && fwd_vals1 && bwd_vals1, S24_ERR_ARG, "NULL operand");
  MaskArgs a0{w0, rows0, cols0, nullptr, idx0, fwd_vals0, nullptr, bwd_vals0, nullptr, perm_ff0};
  MaskArgs a1{w1, rows1, cols1, nullptr, idx1, fwd_vals1, nullptr, bwd_vals1, nullptr, perm_ff1};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool fast = (dtype == S24_BF16 || dtype == S24_F32) && rows0 % kTile == 0 && cols0 % kTile == 0 &&
                    rows1 % kTile == 0 && cols1 % kTile == 0;
  if (!fast) {  // general shapes / dtypes: two launches of the tiled kernel
    if (int rc = launch_mask(a0, dtype, false, st)) return rc;
    return launch_mask(a1, dtype, false, st);
  }
  const int t0 = static_cast<int>((rows0 / kTile) * (cols0 / kTile)), t1 = static_cast<int>((rows1 / kTile) * (cols1 / kTile));
  if (t0 + t1 == 0) return S24_OK;
  if (dtype == S24_BF16) prune_bf16_kernel<uint16_t><<<t0 + t1, kPruneThreads, 0, st>>>(a0, a1, t0);
  else prune_bf16_kernel<float><<<t0 + t1, kPruneThreads, 0, st>>>(a0, a1, t0);
  return s24_check_launch("prune_compress_pair");
}

extern "C" int s24_search_compress_pair(const void* w0, const void* w1, int dtype, int64_t rows0, int64_t cols0,
                                        int64_t rows1, int64_t cols1, uint8_t* idx0, uint8_t* idx1,
                                        uint16_t* fwd_vals0, uint8_t* fwd_e0, uint16_t* bwd_vals0, uint8_t* bwd_e0,
                                        uint16_t* fwd_vals1, uint8_t* fwd_e1, uint16_t* bwd_vals1, uint8_t* bwd_e1,
                                        int64_t perm_ff0, int64_t perm_ff1, void* stream) {
  if (int rc = check_perm(rows0, perm_ff0)) return rc;
  if (int rc = check_perm(rows1, perm_ff1)) return rc;
  if (int rc = check_w(w0, dtype, rows0, cols0)) return rc;
  if (int rc = check_w(w1, dtype, rows1, cols1)) return rc;
  S24_REQUIRE(idx0 != nullptr && idx1 != nullptr, S24_ERR_ARG, "idx pointer is NULL");
  if (int rc = check_compress_outputs(rows0, cols0, fwd_e0, bwd_e0)) return rc;
  if (int rc = check_compress_outputs(rows1, cols1, fwd_e1, bwd_e1)) return rc;
  MaskArgs a0{w0, rows0, cols0, idx0, nullptr, fwd_vals0, fwd_e0, bwd_vals0, bwd_e0, perm_ff0};
  MaskArgs a1{w1, rows1, cols1, idx1, nullptr, fwd_vals1, fwd_e1, bwd_vals1, bwd_e1, perm_ff1};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool fast = dtype == S24_BF16 && rows0 % kTile == 0 && cols0 % kTile == 0 && rows1 % kTile == 0 &&
                    cols1 % kTile == 0;
  if (!fast) {  // general shapes / dtypes: two launches of the tiled kernel
    if (int rc = launch_mask(a0, dtype, true, st)) return rc;
    return launch_mask(a1, dtype, true, st);
  }
  const int t0 = static_cast<int>((rows0 / kTile) * (cols0 / kTile)), t1 = static_cast<int>((rows1 / kTile) * (cols1 / kTile));
  if (t0 + t1 == 0) return S24_OK;
  if (rows0 * cols0 >= (int64_t(1) << 32) || rows1 * cols1 >= (int64_t(1) << 32)) {  // 32-bit strip indexing
    if (int rc = launch_mask(a0, dtype, true, st)) return rc;
    return launch_mask(a1, dtype, true, st);
  }
  const bool pr0 = k1_pairable(cols0, t0 + t1), pr1 = k1_pairable(cols1, t0 + t1);
  const uint32_t s0 = static_cast<uint32_t>(k1_super_tiles(rows0, cols0, pr0));
  const uint32_t s1 = static_cast<uint32_t>(k1_super_tiles(rows1, cols1, pr1));
  search_bf16_kernel<<<k1_grid(s0 + s1), kK1Threads, kK1SmemBytes, st>>>(a0, a1, s0, s0 + s1,
                                                                         (pr0 ? 1 : 0) | (pr1 ? 2 : 0), 1);
  return s24_check_launch("search_compress_pair");
}

extern "C" int s24_idx_to_bits(const uint8_t* idx, int64_t rows, int64_t cols, uint8_t* bits, void* stream) {
  S24_REQUIRE(idx && bits, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE, "shape (%lld, %lld) not divisible into 4x4 blocks",
              (long long)rows, (long long)cols);
  S24_REQUIRE((reinterpret_cast<uintptr_t>(bits) & 3) == 0, S24_ERR_UNSUPPORTED, "bits must be 4-byte aligned");
  const int64_t nb = (rows / 4) * (cols / 4);
  if (nb == 0) return S24_OK;
  idx_to_bits_kernel<<<grid_for(nb, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(idx, rows, cols, bits);
  return s24_check_launch("idx_to_bits");
}

extern "C" int s24_bits_to_idx(const uint8_t* bits, int64_t rows, int64_t cols, uint8_t* idx, int32_t* bad_count,
                               void* stream) {
  S24_REQUIRE(idx && bits && bad_count, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE, "shape (%lld, %lld) not divisible into 4x4 blocks",
              (long long)rows, (long long)cols);
  const int64_t nb = (rows / 4) * (cols / 4);
  if (nb == 0) return S24_OK;
  bits_to_idx_kernel<<<grid_for(nb, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(bits, rows, cols, idx,
                                                                                        bad_count);
  return s24_check_launch("bits_to_idx");
}

extern "C" int s24_meta_flat(const uint8_t* idx, int64_t rows, int64_t cols, uint8_t* fwd_meta, uint8_t* bwd_meta,
                             void* stream) {
  S24_REQUIRE(idx != nullptr, S24_ERR_ARG, "NULL idx");
  S24_REQUIRE(rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE, "shape (%lld, %lld) not divisible into 4x4 blocks",
              (long long)rows, (long long)cols);
  const int64_t nb = (rows / 4) * (cols / 4);
  if (nb == 0) return S24_OK;
  meta_flat_kernel<<<grid_for(nb, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(idx, rows, cols, fwd_meta,
                                                                                     bwd_meta);
  return s24_check_launch("meta_flat");
}

extern "C" int s24_e_to_flat(const uint8_t* e, int64_t m, int64_t k, uint8_t* meta, void* stream) {
  S24_REQUIRE(e && meta, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(m % 128 == 0 && k % 128 == 0, S24_ERR_SHAPE, "E tiles need m, k divisible by 128");
  const int64_t ng = m * (k / 4);
  if (ng == 0) return S24_OK;
  e_to_flat_kernel<<<grid_for(ng, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(e, m, k, meta);
  return s24_check_launch("e_to_flat");
}

extern "C" int s24_masked_decay(float* g, const void* w, int w_dtype, const uint8_t* idx, int64_t rows,
                                int64_t cols, float lambda_w, void* stream) {
  S24_REQUIRE(g && w && idx, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE, "shape (%lld, %lld) not divisible into 4x4 blocks",
              (long long)rows, (long long)cols);
  S24_REQUIRE(w_dtype == S24_BF16 || w_dtype == S24_F32 || w_dtype == S24_F64, S24_ERR_UNSUPPORTED, "bad dtype");
  const int64_t n = rows * cols;
  if (n == 0) return S24_OK;
  masked_decay_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(g, w, w_dtype, idx, rows, cols,
                                                                                       lambda_w);
  return s24_check_launch("masked_decay");
}

extern "C" int s24_masked_decay_bits(float* g, const void* w, int w_dtype, const uint8_t* bits, int64_t n,
                                     float lambda_w, void* stream) {
  S24_REQUIRE(g && w && bits, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(w_dtype == S24_BF16 || w_dtype == S24_F32 || w_dtype == S24_F64, S24_ERR_UNSUPPORTED, "bad dtype");
  if (n == 0) return S24_OK;
  masked_decay_bits_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(g, w, w_dtype, bits, n,
                                                                                            lambda_w);
  return s24_check_launch("masked_decay_bits");
}

extern "C" int s24_adam_compress(float* w, float* u, float* v, const float* g, int64_t rows, int64_t cols,
                                 const uint8_t* idx, double lr, double beta1, double beta2, double eps,
                                 double one_minus_beta1, double one_minus_beta2, double bias_corr1, double bias_corr2,
                                 double lambda_w, double lr_lambda, int decay_mode, uint16_t* fwd_vals,
                                 uint16_t* bwd_vals, int64_t perm_ff, void* stream) {
  S24_REQUIRE(w && u && v && g && idx, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(rows % 128 == 0 && cols % 128 == 0 && rows > 0 && cols > 0, S24_ERR_SHAPE,
              "the fused optimizer + compression needs rows, cols %% 128 == 0 (got %lld, %lld)", (long long)rows,
              (long long)cols);
  S24_REQUIRE(decay_mode >= S24_DECAY_NONE && decay_mode <= S24_DECAY_ON_WEIGHTS, S24_ERR_ARG, "bad decay mode");
  S24_REQUIRE(((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v) |
                reinterpret_cast<uintptr_t>(g)) & 15) == 0,
              S24_ERR_UNSUPPORTED, "w, u, v, g need 16-byte aligned base addresses");
  if (int rc = check_perm(rows, perm_ff)) return rc;
  AdamCompressArgs a{w, u, v, g, rows, cols, idx, fwd_vals, bwd_vals, perm_ff,
                     AdamScalars{lr, beta1, beta2, eps, one_minus_beta1, one_minus_beta2, bias_corr1, bias_corr2,
                                 lambda_w, lr_lambda, decay_mode}};
  const dim3 grid(static_cast<unsigned>(cols / kTile), static_cast<unsigned>(rows / kTile));
  adam_compress_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return s24_check_launch("adam_compress");
}
