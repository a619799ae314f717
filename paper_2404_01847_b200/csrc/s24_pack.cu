// the reference's packed 2:4 storage (Compressed24, spmm.py:38-147) on
// the GPU, so the packed-route API (compress / decompress / mask_of / spmm / spmm_right)
// drops in:
//   s24_pack24     compress (spmm.py:92-106) + Mask24.validate (sparsity.py:98-105): per
//                  group of four (row-wise: along a row, groups row-major; column-wise: down a
//                  column, groups column-major) i0 = first and i1 = last set mask bit, values
//                  copied verbatim, meta = i0 | i1 << 2; groups whose mask is not exactly two
//                  0/1 ones are counted (FormatError).
//   s24_unpack24   decompress / mask_of (spmm.py:109-135); groups with i0 >= i1 are counted
//                  (kept_indices' FormatError, spmm.py:61-67).
//   s24_flat_to_e  reference nibbles of a row-wise operand -> the tensor-core E tiles, the
//                  inverse of s24_e_to_flat, so a Compressed24 feeds s24_spmm directly (its
//                  value order is the kernel's).
// One thread per group; element-size generic copies (bf16 / f32 / f64).  Not on the training
// step: these are the API's packed route and its parity tools.
#include "s24_common.cuh"

namespace s24 {

__device__ __forceinline__ int64_t group_elem(int64_t g, int i, int64_t rows, int64_t cols, int colwise) {
  if (colwise) {
    const int64_t c = g / (rows >> 2), r0 = 4 * (g % (rows >> 2));
    return (r0 + i) * cols + c;
  }
  return 4 * g + i;
}

template <typename T>
__global__ void __launch_bounds__(256) pack_kernel(const T* __restrict__ w, const uint8_t* __restrict__ bits,
                                                   int64_t rows, int64_t cols, int colwise, T* __restrict__ vals,
                                                   uint8_t* __restrict__ meta, int32_t* __restrict__ bad) {
  const int64_t ng = rows * cols / 4;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < ng;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t e[4];
    uint32_t b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      e[i] = group_elem(g, i, rows, cols, colwise);
      b[i] = bits[e[i]];
    }
    const bool ok = b[0] <= 1 && b[1] <= 1 && b[2] <= 1 && b[3] <= 1 && b[0] + b[1] + b[2] + b[3] == 2;
    if (!ok) atomicAdd(bad, 1);
    // np.argmax(bits) / 3 - np.argmax(bits[::-1]): first and last maximal entry
    int i0 = 0, i1 = 3;
    uint32_t mx = b[0];
#pragma unroll
    for (int i = 1; i < 4; ++i)
      if (b[i] > mx) {
        mx = b[i];
        i0 = i;
      }
    uint32_t mr = b[3];
#pragma unroll
    for (int i = 2; i >= 0; --i)
      if (b[i] > mr) {
        mr = b[i];
        i1 = i;
      }
    if (meta) meta[g] = static_cast<uint8_t>(i0 | (i1 << 2));
    if (vals && w) {
      vals[2 * g] = w[e[i0]];
      vals[2 * g + 1] = w[e[i1]];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) unpack_kernel(const T* __restrict__ vals, const uint8_t* __restrict__ meta,
                                                     int64_t rows, int64_t cols, int colwise, T* __restrict__ out,
                                                     uint8_t* __restrict__ bits, int32_t* __restrict__ bad) {
  const int64_t ng = rows * cols / 4;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < ng;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i0 = meta[g] & 3, i1 = (meta[g] >> 2) & 3;
    if (i0 >= i1) atomicAdd(bad, 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t e = group_elem(g, i, rows, cols, colwise);
      if (out) out[e] = (i == i1) ? vals[2 * g + 1] : (i == i0) ? vals[2 * g] : T(0);
      if (bits) bits[e] = (i == i0 || i == i1) ? 1 : 0;
    }
  }
}

// one thread per 16-bit E word: (tile, lane L, column c, half h) holds the nibbles of row
// mm = (L%8) + 8h + 16(L/16) and groups kk/4 with kk = 32c + 16((L/8)%2) + 4 gsub, gsub = 0..3
__global__ void __launch_bounds__(256) flat_to_e_kernel(const uint8_t* __restrict__ meta, int64_t m, int64_t k,
                                                        uint8_t* __restrict__ e) {
  const int64_t kt = k / 128, nwords = (m / 128) * kt * 1024;
  for (int64_t wd = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; wd < nwords;
       wd += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t tile = wd >> 10;
    const int in = static_cast<int>(wd & 1023);  // byte offset / 2 inside the tile
    const int L = in >> 3, c = (in >> 1) & 3, h = in & 1;
    const int64_t row = (tile / kt) * 128 + (L & 7) + 8 * h + 16 * (L >> 4);
    const int64_t kbase = (tile % kt) * 128 + 32 * c + 16 * ((L >> 3) & 1);
    uint32_t word = 0;
#pragma unroll
    for (int gs = 0; gs < 4; ++gs) word |= static_cast<uint32_t>(meta[row * (k / 4) + (kbase >> 2) + gs] & 0xF) << (4 * gs);
    reinterpret_cast<uint16_t*>(e)[wd] = static_cast<uint16_t>(word);
  }
}

static int grid_for_groups(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + 255) / 256, cap = static_cast<int64_t>(sms) * 16;
  return static_cast<int>(want < 1 ? 1 : want < cap ? want : cap);
}

static int check_groups(int64_t rows, int64_t cols, int colwise) {
  S24_REQUIRE(rows >= 0 && cols >= 0, S24_ERR_SHAPE, "negative shape");
  if (colwise)
    S24_REQUIRE(rows % 4 == 0, S24_ERR_SHAPE, "rows=%lld not divisible by 4 for column-wise groups", (long long)rows);
  else
    S24_REQUIRE(cols % 4 == 0, S24_ERR_SHAPE, "cols=%lld not divisible by 4 for row-wise groups", (long long)cols);
  return S24_OK;
}

}  // namespace s24

using namespace s24;

extern "C" int s24_pack24(const void* w, int dtype, const uint8_t* bits, int64_t rows, int64_t cols, int colwise,
                          void* vals, uint8_t* meta, int32_t* bad, void* stream) {
  S24_REQUIRE(bits && bad, S24_ERR_ARG, "NULL mask / counter");
  S24_REQUIRE(!vals || w, S24_ERR_ARG, "values requested without a source matrix");
  if (int rc = check_groups(rows, cols, colwise)) return rc;
  const int64_t ng = rows * cols / 4;
  if (ng == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for_groups(ng);
  if (dtype == S24_BF16)
    pack_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(w), bits, rows, cols, colwise,
                                                static_cast<uint16_t*>(vals), meta, bad);
  else if (dtype == S24_F32)
    pack_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), bits, rows, cols, colwise,
                                             static_cast<float*>(vals), meta, bad);
  else if (dtype == S24_F64)
    pack_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w), bits, rows, cols, colwise,
                                              static_cast<double*>(vals), meta, bad);
  else
    return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  return s24_check_launch("pack24");
}

extern "C" int s24_unpack24(const void* vals, int dtype, const uint8_t* meta, int64_t rows, int64_t cols, int colwise,
                            void* out, uint8_t* bits, int32_t* bad, void* stream) {
  S24_REQUIRE(meta && bad, S24_ERR_ARG, "NULL metadata / counter");
  S24_REQUIRE(!out || vals, S24_ERR_ARG, "dense output requested without values");
  if (int rc = check_groups(rows, cols, colwise)) return rc;
  const int64_t ng = rows * cols / 4;
  if (ng == 0) return S24_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for_groups(ng);
  if (dtype == S24_BF16)
    unpack_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(vals), meta, rows, cols, colwise,
                                                  static_cast<uint16_t*>(out), bits, bad);
  else if (dtype == S24_F32)
    unpack_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(vals), meta, rows, cols, colwise,
                                               static_cast<float*>(out), bits, bad);
  else if (dtype == S24_F64)
    unpack_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(vals), meta, rows, cols, colwise,
                                                static_cast<double*>(out), bits, bad);
  else
    return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  return s24_check_launch("unpack24");
}

extern "C" int s24_flat_to_e(const uint8_t* meta, int64_t m, int64_t k, uint8_t* e, void* stream) {
  S24_REQUIRE(meta && e, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(m >= 0 && k >= 0 && m % 128 == 0 && k % 128 == 0, S24_ERR_SHAPE,
              "E tiles need m, k %% 128 == 0 (got %lld x %lld)", (long long)m, (long long)k);
  const int64_t nwords = (m / 128) * (k / 128) * 1024;
  if (nwords == 0) return S24_OK;
  flat_to_e_kernel<<<grid_for_groups(nwords), 256, 0, static_cast<cudaStream_t>(stream)>>>(meta, m, k, e);
  return s24_check_launch("flat_to_e");
}
