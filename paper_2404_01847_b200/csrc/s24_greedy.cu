// the paper's comparators for the transposable mask search (and, for
// §8(f) #3, the per-block score gaps of block_flip_stats) --
//   transposable_search_greedy (sparsity.py:229-238 -> kernels.greedy_masks, _core.pyx:139-219):
//     per 4x4 block, scan cells by descending |w| (lowest flat index on ties), pick a cell while
//     its block row and column hold fewer than two picks; a stranded 7-pick block is completed
//     by the single swap with the largest net gain (first best on ties).
//   prune_2of4 (sparsity.py:274-279 -> kernels.prune_2of4_keep, _core.pyx:113-136): keep the two
//     largest |w| of every aligned group of four along rows or columns (ties -> lowest index).
// One thread per block / group; magnitudes in float64 as the reference casts them
// (as_array(w, np.float64)), the swap gain in the reference's (a + b) - c order, so both
// kernels are bit-exact for every input dtype.  The greedy result is emitted as the pattern
// index of the 90-pattern table, i.e. in the same form as the exhaustive search (K1), so the
// compress / prune kernels and the TransposableMask API take it unchanged.
#include "s24_common.cuh"
#include "s24_patterns.h"

namespace s24 {

__constant__ uint16_t c_gr_pat_bits[90] = S24_PATTERN_BITS;

template <typename T>
__device__ __forceinline__ double mag(T x);
template <>
__device__ __forceinline__ double mag<uint16_t>(uint16_t x) {
  return fabs(static_cast<double>(__uint_as_float(static_cast<uint32_t>(x) << 16)));
}
template <>
__device__ __forceinline__ double mag<float>(float x) { return fabs(static_cast<double>(x)); }
template <>
__device__ __forceinline__ double mag<double>(double x) { return fabs(x); }

template <typename T>
__global__ void __launch_bounds__(256) greedy_kernel(const T* __restrict__ w, int64_t rows, int64_t cols,
                                                     uint8_t* __restrict__ idx, int32_t* __restrict__ failures) {
  const int64_t bc = cols >> 2, nb = (rows >> 2) * bc;
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r0 = 4 * (b / bc), c0 = 4 * (b % bc);
    double a[16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) a[4 * r + c] = mag<T>(w[(r0 + r) * cols + c0 + c]);
    // descending scan with the reference's selection loop (first index wins ties)
    uint32_t used = 0, picked = 0;
    int rowc[4] = {0, 0, 0, 0}, colc[4] = {0, 0, 0, 0}, total = 0;
    for (int pos = 0; pos < 16; ++pos) {
      int best = -1;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (!((used >> i) & 1) && (best == -1 || a[i] > a[best])) best = i;
      used |= 1u << best;
      const int r = best >> 2, c = best & 3;
      if (rowc[r] < 2 && colc[c] < 2) {
        picked |= 1u << best;
        ++rowc[r];
        ++colc[c];
        ++total;
      }
    }
    if (total == 7) {
      int rdef = -1, cdef = -1;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rowc[i] < 2) rdef = i;
        if (colc[i] < 2) cdef = i;
      }
      double bestgain = 0.0;
      bool first = true;
      int br = -1, bcc = -1;
      for (int r2 = 0; r2 < 4; ++r2) {
        if (r2 == rdef) continue;
        for (int c2 = 0; c2 < 4; ++c2) {
          if (c2 == cdef) continue;
          if ((picked >> (4 * r2 + c2)) & 1) {
            const double gain = __dsub_rn(__dadd_rn(a[rdef * 4 + c2], a[r2 * 4 + cdef]), a[r2 * 4 + c2]);
            if (first || gain > bestgain) {
              bestgain = gain;
              br = r2;
              bcc = c2;
              first = false;
            }
          }
        }
      }
      if (br >= 0) {
        picked &= ~(1u << (4 * br + bcc));
        picked |= 1u << (4 * rdef + bcc);
        picked |= 1u << (4 * br + cdef);
        total = 8;
      }
    }
    int p = 255;
    if (total == 8)
      for (int k = 0; k < 90; ++k)
        if (c_gr_pat_bits[k] == picked) {
          p = k;
          break;
        }
    if (p == 255) atomicAdd(failures, 1);  // the reference raises RuntimeError
    idx[b] = static_cast<uint8_t>(p);
  }
}

// keep-bits of the two largest |w| per aligned group of four (row-wise: consecutive columns,
// col-wise: consecutive rows); bits is a rows x cols 0/1 uint8 matrix
template <typename T>
__global__ void __launch_bounds__(256) prune2of4_kernel(const T* __restrict__ w, int64_t rows, int64_t cols,
                                                        int colwise, uint8_t* __restrict__ bits) {
  const int64_t ng = rows * cols / 4;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < ng;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t e[4];
    if (colwise) {
      // group g covers rows 4 (g / cols) .. +3 of column g % cols (column-major group order)
      const int64_t c = g % cols, r0 = 4 * (g / cols);
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = (r0 + i) * cols + c;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = 4 * g + i;
    }
    double a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = mag<T>(w[e[i]]);
    int i1 = 0;
#pragma unroll
    for (int i = 1; i < 4; ++i)
      if (a[i] > a[i1]) i1 = i;
    int i2 = -1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i != i1 && (i2 == -1 || a[i] > a[i2])) i2 = i;
#pragma unroll
    for (int i = 0; i < 4; ++i) bits[e[i]] = (i == i1 || i == i2) ? 1 : 0;
  }
}

// retained-L1 gap per block: best - second best of the 90 float64 pattern scores, each the
// ascending-position sequential sum of kernels.pattern_scores (_core.pyx:102-105); the
// second best is taken over the multiset of scores (np.partition), so ties give 0
template <typename T>
__global__ void __launch_bounds__(256) gaps_kernel(const T* __restrict__ w, int64_t rows, int64_t cols,
                                                   double* __restrict__ gaps) {
  const int64_t bc = cols >> 2, nb = (rows >> 2) * bc;
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r0 = 4 * (b / bc), c0 = 4 * (b % bc);
    double a[16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) a[4 * r + c] = mag<T>(w[(r0 + r) * cols + c0 + c]);
    double b1 = -INFINITY, b2 = -INFINITY;
    for (int k = 0; k < 90; ++k) {
      const uint32_t bits = c_gr_pat_bits[k];
      double s = 0.0;
      bool first = true;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if ((bits >> i) & 1) {
          s = first ? a[i] : __dadd_rn(s, a[i]);
          first = false;
        }
      if (s > b1) {
        b2 = b1;
        b1 = s;
      } else if (s > b2) {
        b2 = s;
      }
    }
    gaps[b] = __dsub_rn(b1, b2);
  }
}

static int grid_for_work(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + 255) / 256, cap = static_cast<int64_t>(sms) * 16;
  return static_cast<int>(want < 1 ? 1 : want < cap ? want : cap);
}

}  // namespace s24

using namespace s24;

extern "C" int s24_greedy_search(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx,
                                 int32_t* failures, void* stream) {
  S24_REQUIRE(w && idx && failures, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(rows >= 0 && cols >= 0 && rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE,
              "shape (%lld, %lld) not divisible into 4x4 blocks", (long long)rows, (long long)cols);
  const int64_t nb = (rows / 4) * (cols / 4);
  if (nb == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for_work(nb);
  if (dtype == S24_BF16) greedy_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, idx, failures);
  else if (dtype == S24_F32) greedy_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, idx, failures);
  else if (dtype == S24_F64) greedy_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), rows, cols, idx, failures);
  else return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported weight dtype %d", dtype);
  return s24_check_launch("greedy_search");
}

extern "C" int s24_prune_2of4(const void* w, int dtype, int64_t rows, int64_t cols, int colwise, uint8_t* bits,
                              void* stream) {
  S24_REQUIRE(w && bits, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(rows >= 0 && cols >= 0, S24_ERR_SHAPE, "negative shape");
  S24_REQUIRE(colwise ? rows % 4 == 0 : cols % 4 == 0, S24_ERR_SHAPE,
              "groups of 4 along the %s need that dimension %% 4 == 0 (shape %lld x %lld)", colwise ? "rows" : "columns",
              (long long)rows, (long long)cols);
  const int64_t ng = rows * cols / 4;
  if (ng == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for_work(ng);
  if (dtype == S24_BF16) prune2of4_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, colwise, bits);
  else if (dtype == S24_F32) prune2of4_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, colwise, bits);
  else if (dtype == S24_F64) prune2of4_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), rows, cols, colwise, bits);
  else return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported weight dtype %d", dtype);
  return s24_check_launch("prune_2of4");
}

extern "C" int s24_block_gaps(const void* w, int dtype, int64_t rows, int64_t cols, double* gaps, void* stream) {
  S24_REQUIRE(w && gaps, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(rows >= 0 && cols >= 0 && rows % 4 == 0 && cols % 4 == 0, S24_ERR_SHAPE,
              "shape (%lld, %lld) not divisible into 4x4 blocks", (long long)rows, (long long)cols);
  const int64_t nb = (rows / 4) * (cols / 4);
  if (nb == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for_work(nb);
  if (dtype == S24_BF16) gaps_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, gaps);
  else if (dtype == S24_F32) gaps_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, gaps);
  else if (dtype == S24_F64) gaps_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), rows, cols, gaps);
  else return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported weight dtype %d", dtype);
  return s24_check_launch("block_gaps");
}
