// K8: MVUE (minimum-variance unbiased) 2:4 sparsification of an upstream
// gradient along tokens, emitted directly as the sparse tensor-core operand of
// the weight-gradient GEMM (kept values + E tiles).
//
// Reference: _grad_weight(mvue=True) (gated_ffn.py:367-373) ->
// mvue_slots_rowwise(dz^T) (sparsity.py:401-413) -> _mvue_kept (:358-376):
//   pi   = mvue_inclusion_probs(group)   (:290-324, water-filled, sum 2)
//   p    = mvue_pair_probs(pi)           (:327-355, greedy transportation fill)
//   u    = default_rng(seed).random(n)   (one draw per group, group order)
//   pick = min(#{cumsum(p) <= u * sum(p)}, 5); kept values g / pi
// Bit-exact reproduction: every float64 operation is issued explicitly in the
// reference's order (sequential 4-term sums, mul-then-div, no FMA
// contraction), and numpy's PCG64 (XSL-RR 128/64) stream is regenerated on the
// device with O(log n) jump-ahead to each thread's first group.
//
// Layout: input G is token-major (n tokens x f features); the sparsified
// matrix is G^T (f x n), groups of 4 consecutive tokens per feature, group
// index i = row * (n / 4) + token / 4 (row = feature in the reference's order;
// gate_ff > 0 maps the u/v-interleaved feature p back to its [u; v] row).
// One CTA = 128 features x 128 tokens = one E tile; the tile is staged in smem
// so each lane streams one feature column conflict-free.
#include "s24_common.cuh"

namespace s24 {

struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

struct MvueRng {
  U128 state;       // PCG64 state after seeding (numpy bit_generator.state)
  U128 inc;         // increment (odd)
  U128 mult[40];    // MULT^(2^i)
  U128 plus[40];    // additive term of 2^i steps
  U128 rowm[7];     // multiplier of (groups per feature row) * 2^i steps (K8 tile kernel)
  U128 rowp[7];     // additive term of the same
};

constexpr uint64_t kPcgMultHi = 0x2360ED051FC65DA4ull, kPcgMultLo = 0x4385DF649FCCF645ull;

__device__ __forceinline__ U128 pcg_advance(const MvueRng& rng, uint64_t delta) {
  U128 am{0, 1}, ap{0, 0};
  for (int i = 0; delta; ++i, delta >>= 1) {
    if (delta & 1) {
      am = mul128(am, rng.mult[i]);
      ap = add128(mul128(ap, rng.mult[i]), rng.plus[i]);
    }
  }
  return add128(mul128(am, rng.state), ap);
}
// the LCG's k-step maps x -> M x + P all commute; composition and application
__device__ __forceinline__ void affine_compose(U128& m, U128& p, const U128& m2, const U128& p2) {
  p = add128(mul128(p, m2), p2);
  m = mul128(m, m2);
}
__device__ __forceinline__ U128 affine_apply(const U128& m, const U128& p, const U128& x) {
  return add128(mul128(m, x), p);
}
__device__ __forceinline__ U128 shfl_xor128(const U128& v, int off) {
  U128 r;
  r.hi = __shfl_xor_sync(0xFFFFFFFFu, v.hi, off);
  r.lo = __shfl_xor_sync(0xFFFFFFFFu, v.lo, off);
  return r;
}
// PCG64 state `delta` steps after rng.state, computed by a whole warp (delta < 2^40): lane l
// holds the maps of bits l and l + 32, a butterfly composes them (every lane ends with the map)
__device__ __forceinline__ U128 pcg_advance_warp(const MvueRng& rng, uint64_t delta, int lane) {
  U128 m{0, 1}, p{0, 0};
  if ((delta >> lane) & 1) {
    m = rng.mult[lane];
    p = rng.plus[lane];
  }
  if (lane < 8 && ((delta >> (lane + 32)) & 1)) affine_compose(m, p, rng.mult[lane + 32], rng.plus[lane + 32]);
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const U128 m2 = shfl_xor128(m, off), p2 = shfl_xor128(p, off);
    affine_compose(m, p, m2, p2);
  }
  return affine_apply(m, p, rng.state);
}

// one PCG64 step and its XSL-RR 64-bit output
__device__ __forceinline__ uint64_t pcg_next64(U128& st, const U128& inc) {
  st = add128(mul128(st, U128{kPcgMultHi, kPcgMultLo}), inc);
  const uint64_t x = st.hi ^ st.lo;
  const unsigned rot = static_cast<unsigned>(st.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
// numpy Generator.random() of that output: (out >> 11) * 2^-53, exactly
__device__ __forceinline__ double pcg_double(uint64_t out) {
  return __dmul_rn(static_cast<double>(out >> 11), 1.0 / 9007199254740992.0);
}
// one numpy Generator.random(): step, XSL-RR output, 53-bit double
__device__ __forceinline__ double pcg_uniform(U128& st, const U128& inc) { return pcg_double(pcg_next64(st, inc)); }

// exact reference arithmetic helpers (no contraction)
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// MVUE selection for one group: returns the pair index (0..5) and the two kept values
__device__ __forceinline__ int mvue_group(const double (&g)[4], double u, double& v0, double& v1) {
  double a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = fabs(g[k]);
  const double total = dadd(dadd(dadd(a[0], a[1]), a[2]), a[3]);
  int fm = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (a[k] > a[fm]) fm = k;
  const double amax = a[fm];
  double b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = k == fm ? 0.0 : a[k];
  const double rest = dadd(dadd(dadd(b[0], b[1]), b[2]), b[3]);
  const bool clamp = amax > rest;
  int nnz = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) nnz += a[k] != 0.0;
  double pi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double plain = ddiv(dmul(2.0, a[k]), total);
    const double capped = k == fm ? 1.0 : ddiv(a[k], rest);
    pi[k] = clamp ? capped : plain;
    if (nnz == 1) pi[k] = a[k] > 0.0 ? 1.0 : 1.0 / 3.0;
    if (nnz == 0) pi[k] = 0.5;
  }
  // greedy pair fill (sparsity.py:334-355)
  double r0 = pi[0], r1 = pi[1], r2 = pi[2], r3 = pi[3];
  double s = dmul(0.5, dadd(dadd(dadd(pi[0], pi[1]), pi[2]), pi[3]));
  const double p01 = fmax(fmin(fmin(fmin(r0, r1), dsub(s, r2)), dsub(s, r3)), 0.0);
  r0 = dsub(r0, p01);
  r1 = dsub(r1, p01);
  s = dsub(s, p01);
  const double p02 = fmax(fmin(fmin(r0, r2), dsub(s, r3)), 0.0);
  r0 = dsub(r0, p02);
  r2 = dsub(r2, p02);
  s = dsub(s, p02);
  const double p03 = fmax(fmin(r0, r3), 0.0);
  r3 = dsub(r3, p03);
  s = dsub(s, p03);
  const double p12 = fmax(fmin(fmin(r1, r2), dsub(s, r3)), 0.0);
  r1 = dsub(r1, p12);
  r2 = dsub(r2, p12);
  const double p13 = fmax(fmin(r1, r3), 0.0);
  r3 = dsub(r3, p13);
  const double p23 = fmax(fmin(r2, r3), 0.0);
  double c[6];
  c[0] = p01;
  c[1] = dadd(c[0], p02);
  c[2] = dadd(c[1], p03);
  c[3] = dadd(c[2], p12);
  c[4] = dadd(c[3], p13);
  c[5] = dadd(c[4], p23);
  const double draw = dmul(u, c[5]);
  int idx = 0;
#pragma unroll
  for (int j = 0; j < 6; ++j) idx += c[j] <= draw;
  idx = min(idx, 5);
  // register selects, not indexed arrays (dynamic indexing would go to local memory)
  const double g0 = idx < 3 ? g[0] : (idx < 5 ? g[1] : g[2]);
  const double q0 = idx < 3 ? pi[0] : (idx < 5 ? pi[1] : pi[2]);
  const bool s1 = idx == 0, s2 = idx == 1 || idx == 3;
  const double g1 = s1 ? g[1] : (s2 ? g[2] : g[3]);
  const double q1 = s1 ? pi[1] : (s2 ? pi[2] : pi[3]);
  v0 = ddiv(g0, q0);
  v1 = ddiv(g1, q1);
  return idx;
}

// The exact estimator's common case in fp32 with a certificate.  When the group's nonzero
// magnitudes span at most 14 binades, every sum of them (total, rest) is exact in fp32 (bf16
// significands: the sum is an integer < 2^24 times the smallest binade's unit), so the clamp test
// amax > rest is the reference's.  The inclusion probabilities n / d (n = 2 a or a) are then
// within 2 ulp(1) of the reference's float64 quotients (reciprocal and product roundings), and
// the greedy pair fill and cumulative sums add their operands' bounds step by step -- at most
// 968 ulp(1) between c_j and the draw (tools/mvue_bound.py), so a decision
// c_j <= draw whose fp32 margin exceeds 2^-14 (1024 ulp(1)) is the reference's decision.  The
// kept VALUES need no division: pi_k is proportional to |g_k| (2 |g_k| / total, or |g_k| / rest
// when clamped), so the reference's g_k / pi_k is sign(g_k) total / 2 (resp. sign(g_k) rest) up
// to two float64 roundings (2^-52 relative), which its f32 conversion removes because that
// magnitude is an (exact) f32 number; the clamped maximum (pi = 1) and the single nonzero of a
// group keep g itself, zeros keep +-0.  Anything uncertain (span, margins, extreme magnitudes)
// sets ok = false and the caller reruns the group in float64 (mvue_group_slow): bit-exact by
// construction.
__device__ __forceinline__ int mvue_group_cert(const float (&g)[4], uint64_t out, uint32_t& packed, bool& ok) {
  // written as selects throughout: `if` forms compiled to branches with reconvergence
  // bookkeeping (BSSY / BSYNC) in every group
  const float a0 = fabsf(g[0]), a1 = fabsf(g[1]), a2 = fabsf(g[2]), a3 = fabsf(g[3]);
  const float total = __fadd_rn(__fadd_rn(__fadd_rn(a0, a1), a2), a3);
  // first maximum (strict >, the reference's scan)
  const bool s1 = a1 > a0;
  float amax = s1 ? a1 : a0;
  int fm = s1 ? 1 : 0;
  const bool s2 = a2 > amax;
  amax = s2 ? a2 : amax;
  fm = s2 ? 2 : fm;
  const bool s3 = a3 > amax;
  amax = s3 ? a3 : amax;
  fm = s3 ? 3 : fm;
  const float b0 = fm == 0 ? 0.0f : a0, b1 = fm == 1 ? 0.0f : a1, b2 = fm == 2 ? 0.0f : a2, b3 = fm == 3 ? 0.0f : a3;
  const float rest = __fadd_rn(__fadd_rn(__fadd_rn(b0, b1), b2), b3);
  const int nnz = (a0 != 0.0f) + (a1 != 0.0f) + (a2 != 0.0f) + (a3 != 0.0f);
  const float amin = fminf(fminf(a0 == 0.0f ? amax : a0, a1 == 0.0f ? amax : a1),
                           fminf(a2 == 0.0f ? amax : a2, a3 == 0.0f ? amax : a3));
  // exact sums: binade span <= 14 over the nonzero magnitudes, all normal and far from overflow
  const int span = static_cast<int>(__float_as_uint(amax) >> 23) - static_cast<int>(__float_as_uint(amin) >> 23);
  bool good = nnz == 0 || (span <= 14 && amin >= 1.0e-30f && total <= 1.0e30f);  // total: also NaN / inf
  const bool clamp = amax > rest;
  const float inv = __frcp_rn(clamp ? rest : total);
  const float ak[4] = {a0, a1, a2, a3};
  float pi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float pg = clamp ? (k == fm ? 1.0f : __fmul_rn(ak[k], inv)) : __fmul_rn(2.0f * ak[k], inv);
    const float p1 = ak[k] > 0.0f ? 1.0f : (1.0f / 3.0f);
    pi[k] = nnz >= 2 ? pg : (nnz == 1 ? p1 : 0.5f);
  }
  float r0 = pi[0], r1 = pi[1], r2 = pi[2], r3 = pi[3];
  float s = 0.5f * __fadd_rn(__fadd_rn(__fadd_rn(pi[0], pi[1]), pi[2]), pi[3]);
  const float p01 = fmaxf(fminf(fminf(fminf(r0, r1), __fsub_rn(s, r2)), __fsub_rn(s, r3)), 0.0f);
  r0 = __fsub_rn(r0, p01);
  r1 = __fsub_rn(r1, p01);
  s = __fsub_rn(s, p01);
  const float p02 = fmaxf(fminf(fminf(r0, r2), __fsub_rn(s, r3)), 0.0f);
  r0 = __fsub_rn(r0, p02);
  r2 = __fsub_rn(r2, p02);
  s = __fsub_rn(s, p02);
  const float p03 = fmaxf(fminf(r0, r3), 0.0f);
  r3 = __fsub_rn(r3, p03);
  s = __fsub_rn(s, p03);
  const float p12 = fmaxf(fminf(fminf(r1, r2), __fsub_rn(s, r3)), 0.0f);
  r1 = __fsub_rn(r1, p12);
  r2 = __fsub_rn(r2, p12);
  const float p13 = fmaxf(fminf(r1, r3), 0.0f);
  r3 = __fsub_rn(r3, p13);
  const float p23 = fmaxf(fminf(r2, r3), 0.0f);
  const float c0 = p01, c1 = __fadd_rn(c0, p02), c2 = __fadd_rn(c1, p03), c3 = __fadd_rn(c2, p12),
              c4 = __fadd_rn(c3, p13), c5 = __fadd_rn(c4, p23);
  // the uniform's top 24 bits: within 2^-24 of the reference's 53-bit double (no float64 ops)
  const float uf = __uint2float_rn(static_cast<uint32_t>(out >> 40)) * 5.9604644775390625e-8f;  // 2^-24
  const float draw = __fmul_rn(uf, c5);
  constexpr float kMargin = 6.103515625e-5f;  // 2^-14 = 1024 ulp(1) > the 968 ulp(1) bound
  const float dmin = fminf(fminf(fminf(fabsf(c0 - draw), fabsf(c1 - draw)), fminf(fabsf(c2 - draw), fabsf(c3 - draw))),
                           fminf(fabsf(c4 - draw), fabsf(c5 - draw)));
  good = good && dmin > kMargin;
  const int idx = min((c0 <= draw) + (c1 <= draw) + (c2 <= draw) + (c3 <= draw) + (c4 <= draw) + (c5 <= draw), 5);
  const int i0 = idx < 3 ? 0 : (idx < 5 ? 1 : 2);
  const int i1 = idx == 0 ? 1 : (idx == 1 || idx == 3) ? 2 : 3;
  const float g0 = i0 == 0 ? g[0] : (i0 == 1 ? g[1] : g[2]);
  const float g1 = i1 == 1 ? g[1] : (i1 == 2 ? g[2] : g[3]);
  // nnz >= 2: a kept element has pi > 0 (its pair probability is positive), so a != 0
  good = good && (nnz < 2 || (g0 != 0.0f && g1 != 0.0f));
  ok = good;
  const float m = clamp ? rest : 0.5f * total;  // kept magnitude when pi = 2 a / total or a / rest
  // nnz == 1: the nonzero keeps g (pi = 1), zeros keep +-0; nnz == 0: +-0
  const float v0 = (nnz < 2 || (clamp && i0 == fm)) ? g0 : copysignf(m, g0);
  const float v1 = (nnz < 2 || (clamp && i1 == fm)) ? g1 : copysignf(m, g1);
  packed = static_cast<uint32_t>(f32_to_bf16(v0)) | (static_cast<uint32_t>(f32_to_bf16(v1)) << 16);
  return idx;
}

// the float64 reference computation of one group, out of line (the rare uncertain groups)
__device__ __noinline__ int mvue_group_slow(const float (&g)[4], uint64_t out, uint32_t& packed) {
  const double u = pcg_double(out);
  double gv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) gv[k] = static_cast<double>(g[k]);
  double v0, v1;
  const int idx = mvue_group(gv, u, v0, v1);
  // f64 -> f32 -> bf16 (the rounding of the reference-side bf16 operand)
  packed = static_cast<uint32_t>(f32_to_bf16(__double2float_rn(v0))) |
           (static_cast<uint32_t>(f32_to_bf16(__double2float_rn(v1))) << 16);
  return idx;
}

// Throughput mode: the same estimator in fp32 (inclusion probabilities, greedy
// pair fill, cumulative draw, g / pi) with a counter-based uniform per group.
// Unbiased like the reference (E[value] = g) but not bit-identical to numpy's
// stream; selected with exact=0.  Branch-free: pi_k = min(a_k * inv, 1) covers
// both the plain (2 a / total) and the clamped (1 for the max, a / rest) case.
__device__ __forceinline__ uint32_t mvue_nibble_f32(const float (&g)[4], float u, float& v0, float& v1) {
  const float a0 = fabsf(g[0]), a1 = fabsf(g[1]), a2 = fabsf(g[2]), a3 = fabsf(g[3]);
  const float total = ((a0 + a1) + a2) + a3;
  const float amax = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
  const float rest = total - amax;
  const bool clamp = amax > rest;
  const float inv = __frcp_rn(clamp ? rest : 0.5f * total);
  float pi[4] = {fminf(a0 * inv, 1.0f), fminf(a1 * inv, 1.0f), fminf(a2 * inv, 1.0f), fminf(a3 * inv, 1.0f)};
  if (rest == 0.0f) {  // at most one nonzero: it is kept, the zeros share 1 (or all 0.5)
    const float z = total > 0.0f ? (1.0f / 3.0f) : 0.5f;
#pragma unroll
    for (int k = 0; k < 4; ++k) pi[k] = (k == 0 ? a0 : k == 1 ? a1 : k == 2 ? a2 : a3) > 0.0f ? 1.0f : z;
  }
  float r0 = pi[0], r1 = pi[1], r2 = pi[2], r3 = pi[3];
  float s = 0.5f * (((pi[0] + pi[1]) + pi[2]) + pi[3]);
  const float p01 = fmaxf(fminf(fminf(fminf(r0, r1), s - r2), s - r3), 0.0f);
  r0 -= p01; r1 -= p01; s -= p01;
  const float p02 = fmaxf(fminf(fminf(r0, r2), s - r3), 0.0f);
  r0 -= p02; r2 -= p02; s -= p02;
  const float p03 = fmaxf(fminf(r0, r3), 0.0f);
  r3 -= p03; s -= p03;
  const float p12 = fmaxf(fminf(fminf(r1, r2), s - r3), 0.0f);
  r1 -= p12; r2 -= p12;
  const float p13 = fmaxf(fminf(r1, r3), 0.0f);
  r3 -= p13;
  const float p23 = fmaxf(fminf(r2, r3), 0.0f);
  const float c0 = p01, c1 = c0 + p02, c2 = c1 + p03, c3 = c2 + p12, c4 = c3 + p13, c5 = c4 + p23;
  const float draw = u * c5;
  const int idx = min((c0 <= draw) + (c1 <= draw) + (c2 <= draw) + (c3 <= draw) + (c4 <= draw) + (c5 <= draw), 5);
  const float g0 = idx < 3 ? g[0] : (idx < 5 ? g[1] : g[2]);
  const float q0 = idx < 3 ? pi[0] : (idx < 5 ? pi[1] : pi[2]);
  const bool s1 = idx == 0, s2 = idx == 1 || idx == 3;
  const float g1 = s1 ? g[1] : (s2 ? g[2] : g[3]);
  const float q1 = s1 ? pi[1] : (s2 ? pi[2] : pi[3]);
  v0 = __fdividef(g0, q0);
  v1 = __fdividef(g1, q1);
  return static_cast<uint32_t>(idx);
}

// murmur3 finaliser: a bijection on 32 bits, so distinct group counters under
// one key never share a uniform
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
__device__ __forceinline__ float counter_uniform(uint32_t k1, uint32_t k2, uint32_t ctr) {
  const uint32_t h = fmix32(fmix32(ctr ^ k1) + k2);
  return static_cast<float>(h >> 8) * (1.0f / 16777216.0f);  // [0, 1) with 24 bits
}

struct MvueArgs {
  const uint16_t* g;  // n x f token-major (ldg)
  int64_t ldg, n, f, gate_ff;
  uint16_t* vals;     // f x n/2
  uint8_t* e;         // E tiles [f/128][n/128]
  uint8_t* pairs;     // optional f x n/4 pair indices (tests)
  int force_f64;      // exact mode 2 (tests): every group through the float64 path, no certificate
  int64_t n_valid;    // tokens that exist (<= n, % 4 == 0): rows >= n_valid read as zeros, and the random
                      // stream's row stride is n_valid / 4 groups (the reference's index for its n)
};

template <bool kExact>
__global__ void __launch_bounds__(256) mvue_tile_kernel(MvueArgs p, const __grid_constant__ MvueRng rng) {
  __shared__ __align__(16) uint16_t s_g[128 * 136];  // [token][feature], row pitch 136 (272 B)
  __shared__ __align__(16) uint32_t s_e[512];
  const int tid = threadIdx.x;
  const int64_t f0 = static_cast<int64_t>(blockIdx.y) * 128, t0 = static_cast<int64_t>(blockIdx.x) * 128;
  for (int i = tid; i < 512; i += 256) s_e[i] = 0;
  // coalesced tile load: 128 token rows x 256 bytes; all 8 loads of a thread are in
  // flight before the first smem store (one DRAM latency per CTA, not eight)
  {
    uint4 buf[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = tid + 256 * q, tr = i >> 4, ch = i & 15;
      buf[q] = t0 + tr < p.n_valid ? __ldg(reinterpret_cast<const uint4*>(p.g + (t0 + tr) * p.ldg + f0 + ch * 8))
                                   : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = tid + 256 * q, tr = i >> 4, ch = i & 15;
      *reinterpret_cast<uint4*>(&s_g[tr * 136 + ch * 8]) = buf[q];
    }
  }
  __syncthreads();
  const int ml = tid & 127, half = tid >> 7;  // feature in tile, token half (64 tokens = 16 groups)
  const int64_t feat = f0 + ml;
  const int64_t row = p.gate_ff > 0 ? ((feat & 31) < 16 ? 16 * (feat >> 5) + (feat & 31)
                                                         : p.gate_ff + 16 * (feat >> 5) + (feat & 31) - 16)
                                    : feat;
  const int64_t grp0 = t0 / 4 + 16 * half;
  const uint64_t stream0 = static_cast<uint64_t>(row * (p.n_valid / 4) + grp0);
  U128 st{0, 0};
  if constexpr (kExact) {
    // stream index of this thread = base(u / v rows) + roff * (n / 4) + 16 half: the CTA's one or
    // two base states by a warp each (pcg_advance_warp), then at most 7 + 1 table steps per thread
    // instead of a full 40-bit jump-ahead
    __shared__ U128 s_base[2];
    const int w = tid >> 5, lane = tid & 31;
    const int nbase = p.gate_ff > 0 ? 2 : 1;
    const int64_t rbase0 = p.gate_ff > 0 ? f0 / 2 : f0;
    if (w < nbase) {
      const int64_t rb = rbase0 + (w ? p.gate_ff : 0);
      const U128 b = pcg_advance_warp(rng, static_cast<uint64_t>(rb * (p.n_valid / 4) + t0 / 4), lane);
      if (lane == 0) s_base[w] = b;
    }
    __syncthreads();
    const int sel = p.gate_ff > 0 ? ((ml >> 4) & 1) : 0;
    const int roff = p.gate_ff > 0 ? 16 * (ml >> 5) + (ml & 15) : ml;
    st = s_base[sel];
#pragma unroll
    for (int i = 0; i < 7; ++i)
      if ((roff >> i) & 1) st = affine_apply(rng.rowm[i], rng.rowp[i], st);
    if (half) st = affine_apply(rng.mult[4], rng.plus[4], st);  // 16 groups
  }
  uint32_t halfwords[4] = {0, 0, 0, 0};
  uint32_t pidx[4] = {0, 0, 0, 0};
  const uint32_t* s_out;  // [feature][32 words + 1 pad] kept-value pairs of the tile
  if constexpr (kExact) {
    // four passes of four groups: a fully unrolled 16-group body with the certificate and the
    // float64 fallback call overflows the instruction cache (measured: "no instruction" stalls
    // dominated); values go straight to their own staging area
    extern __shared__ uint32_t s_pk[];  // 128 x 33 words (dynamic: the static tile already uses 36 KB)
#pragma unroll 1
    for (int jj = 0; jj < 4; ++jj) {
      uint32_t hw = 0, pw = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 4 * jj + q;
        float gv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) gv[k] = bf16_to_f32(s_g[(64 * half + 4 * j + k) * 136 + ml]);
        const uint64_t out = pcg_next64(st, rng.inc);
        bool ok;
        uint32_t pk;
        int idx = mvue_group_cert(gv, out, pk, ok);
        if (!ok || p.force_f64) idx = mvue_group_slow(gv, out, pk);
        s_pk[ml * 33 + 16 * half + j] = pk;
        // nibble i0 | i1 << 2 of pair idx = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE}[idx]
        hw |= ((0xED9C84u >> (4 * idx)) & 0xFu) << (4 * q);
        pw |= static_cast<uint32_t>(idx) << (8 * q);
      }
      halfwords[0] = halfwords[1];
      halfwords[1] = halfwords[2];
      halfwords[2] = halfwords[3];
      halfwords[3] = hw;
      pidx[0] = pidx[1];
      pidx[1] = pidx[2];
      pidx[2] = pidx[3];
      pidx[3] = pw;
    }
    __syncthreads();
    s_out = s_pk;
  } else {
    uint32_t packed[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float gv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) gv[k] = bf16_to_f32(s_g[(64 * half + 4 * j + k) * 136 + ml]);
      float f0, f1;
      const uint32_t k1 = static_cast<uint32_t>(rng.state.lo ^ (rng.state.lo >> 32)),
                     k2 = static_cast<uint32_t>(rng.inc.hi ^ (rng.inc.hi >> 32));
      const int idx =
          static_cast<int>(mvue_nibble_f32(gv, counter_uniform(k1, k2, static_cast<uint32_t>(stream0 + j)), f0, f1));
      packed[j] = pack_bf16x2(f0, f1);
      // nibble i0 | i1 << 2 of pair idx = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE}[idx]
      const uint32_t nib = (0xED9C84u >> (4 * idx)) & 0xFu;
      halfwords[j >> 2] |= nib << (4 * (j & 3));
      pidx[j >> 2] |= static_cast<uint32_t>(idx) << (8 * (j & 3));
    }
    // kept values staged in the (now free) input tile, then streamed as whole 128-byte rows
    __syncthreads();
    uint32_t* s_v = reinterpret_cast<uint32_t*>(s_g);
#pragma unroll
    for (int j = 0; j < 16; ++j) s_v[ml * 33 + 16 * half + j] = packed[j];
    __syncthreads();
    s_out = s_v;
  }
  if (p.pairs) {
    uint4* dp = reinterpret_cast<uint4*>(p.pairs + feat * (p.n / 4) + grp0);
    *dp = make_uint4(pidx[0], pidx[1], pidx[2], pidx[3]);
  }
  for (int rr = tid >> 5; rr < 128; rr += 8) {
    const int lane = tid & 31;
    reinterpret_cast<uint32_t*>(p.vals + (f0 + rr) * (p.n / 2) + t0 / 2)[lane] = s_out[rr * 33 + lane];
  }
  // metadata: halfword w covers tokens 64 half + 16 w .. +15 of row ml
  if (p.e) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int kk = 64 * half + 16 * w;
      const int L = (ml & 7) + 8 * ((kk & 31) >> 4) + 16 * (ml >> 4);
      const int c = kk >> 5, h = (ml >> 3) & 1;
      reinterpret_cast<uint16_t*>(s_e)[L * 8 + c * 2 + h] = static_cast<uint16_t>(halfwords[w]);
    }
    __syncthreads();
    uint4* de = reinterpret_cast<uint4*>(p.e + (static_cast<int64_t>(blockIdx.y) * (p.n / 128) + blockIdx.x) * 2048);
    if (tid < 128) de[tid] = reinterpret_cast<const uint4*>(s_e)[tid];
  }
}

// mvue_prune (sparsity.py:379-398) of any (rows x cols) matrix along `colwise`: the same exact
// float64 estimator and PCG64 stream as the K8 tile kernel, with the reference's group order
// (to_groups: row-wise groups row-major, column-wise groups column-major) as the stream index.
// Output: the dense float64 estimate (kept g / pi, zeros elsewhere) and its 0/1 mask.  Each
// thread jumps ahead once and walks kMvueRun consecutive groups.
constexpr int kMvueRun = 16;

template <typename T>
__device__ __forceinline__ double as_f64(T x);
template <>
__device__ __forceinline__ double as_f64<uint16_t>(uint16_t x) {
  return static_cast<double>(bf16_to_f32(x));
}
template <>
__device__ __forceinline__ double as_f64<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double as_f64<double>(double x) { return x; }

template <typename T>
__global__ void __launch_bounds__(256) mvue_prune_kernel(const T* __restrict__ g, int64_t rows, int64_t cols,
                                                         int colwise, const __grid_constant__ MvueRng rng,
                                                         double* __restrict__ out, uint8_t* __restrict__ bits) {
  const int64_t ng = rows * cols / 4;
  const int64_t first = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * kMvueRun;
  if (first >= ng) return;
  U128 st = pcg_advance(rng, static_cast<uint64_t>(first));
  const int64_t last = min(first + kMvueRun, ng);
  for (int64_t gi = first; gi < last; ++gi) {
    int64_t e[4];
    if (colwise) {
      const int64_t c = gi / (rows >> 2), r0 = 4 * (gi % (rows >> 2));
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = (r0 + k) * cols + c;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = 4 * gi + k;
    }
    double gv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) gv[k] = as_f64<T>(g[e[k]]);
    const double u = pcg_uniform(st, rng.inc);
    double v0, v1;
    const int idx = mvue_group(gv, u, v0, v1);
    const int i0 = idx < 3 ? 0 : (idx < 5 ? 1 : 2);
    const int i1 = idx == 0 ? 1 : (idx == 1 || idx == 3) ? 2 : 3;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      out[e[k]] = k == i0 ? v0 : (k == i1 ? v1 : 0.0);
      if (bits) bits[e[k]] = (k == i0 || k == i1) ? 1 : 0;
    }
  }
}

static void mvue_rng_tables(MvueRng& rng, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                            uint64_t row_groups = 0) {
  rng.state = U128{state_hi, state_lo};
  rng.inc = U128{inc_hi, inc_lo};
  unsigned __int128 m = (static_cast<unsigned __int128>(kPcgMultHi) << 64) | kPcgMultLo;
  unsigned __int128 pl = (static_cast<unsigned __int128>(inc_hi) << 64) | inc_lo;
  for (int i = 0; i < 40; ++i) {
    rng.mult[i] = U128{static_cast<uint64_t>(m >> 64), static_cast<uint64_t>(m)};
    rng.plus[i] = U128{static_cast<uint64_t>(pl >> 64), static_cast<uint64_t>(pl)};
    pl = (m + 1) * pl;
    m = m * m;
  }
  // (row_groups * 2^i)-step maps: x -> M x + P composed from the 2^i tables, then squared
  unsigned __int128 rm = 1, rp = 0;
  for (int i = 0; i < 40; ++i)
    if ((row_groups >> i) & 1) {
      const unsigned __int128 mi = (static_cast<unsigned __int128>(rng.mult[i].hi) << 64) | rng.mult[i].lo;
      const unsigned __int128 pi = (static_cast<unsigned __int128>(rng.plus[i].hi) << 64) | rng.plus[i].lo;
      rp = rp * mi + pi;
      rm = rm * mi;
    }
  for (int i = 0; i < 7; ++i) {
    rng.rowm[i] = U128{static_cast<uint64_t>(rm >> 64), static_cast<uint64_t>(rm)};
    rng.rowp[i] = U128{static_cast<uint64_t>(rp >> 64), static_cast<uint64_t>(rp)};
    rp = rm * rp + rp;
    rm = rm * rm;
  }
}

}  // namespace s24

using namespace s24;

extern "C" int s24_mvue_prune(const void* g, int dtype, int64_t rows, int64_t cols, int colwise, uint64_t state_hi,
                              uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double* out, uint8_t* bits,
                              void* stream) {
  S24_REQUIRE(g && out, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(rows >= 0 && cols >= 0, S24_ERR_SHAPE, "negative shape");
  if (colwise)
    S24_REQUIRE(rows % 4 == 0, S24_ERR_SHAPE, "rows=%lld not divisible by 4 for column-wise groups", (long long)rows);
  else
    S24_REQUIRE(cols % 4 == 0, S24_ERR_SHAPE, "cols=%lld not divisible by 4 for row-wise groups", (long long)cols);
  const int64_t ng = rows * cols / 4;
  if (ng == 0) return S24_OK;
  S24_REQUIRE(static_cast<double>(ng) < 1099511627776.0, S24_ERR_SHAPE, "MVUE stream index exceeds the 2^40 jump table");
  MvueRng rng;
  mvue_rng_tables(rng, state_hi, state_lo, inc_hi, inc_lo);
  const int64_t threads = (ng + kMvueRun - 1) / kMvueRun;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == S24_BF16)
    mvue_prune_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(g), rows, cols, colwise, rng, out, bits);
  else if (dtype == S24_F32)
    mvue_prune_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(g), rows, cols, colwise, rng, out, bits);
  else if (dtype == S24_F64)
    mvue_prune_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(g), rows, cols, colwise, rng, out, bits);
  else
    return s24_set_error(S24_ERR_UNSUPPORTED, "unsupported dtype %d", dtype);
  return s24_check_launch("mvue_prune");
}

extern "C" int s24_mvue_compress(const uint16_t* g, int64_t ldg, int64_t n, int64_t f, uint64_t state_hi,
                                 uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t gate_ff,
                                 uint16_t* vals, uint8_t* e, uint8_t* pairs, int exact, void* stream) {
  return s24_mvue_compress_ragged(g, ldg, n, n, f, state_hi, state_lo, inc_hi, inc_lo, gate_ff, vals, e, pairs, exact,
                                  stream);
}

extern "C" int s24_mvue_compress_ragged(const uint16_t* g, int64_t ldg, int64_t n, int64_t n_valid, int64_t f,
                                        uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                        int64_t gate_ff, uint16_t* vals, uint8_t* e, uint8_t* pairs, int exact,
                                        void* stream) {
  S24_REQUIRE(g && vals, S24_ERR_ARG, "NULL pointer");
  S24_REQUIRE(n_valid > 0 && n_valid <= n && n_valid % 4 == 0 && n - n_valid < 128, S24_ERR_SHAPE,
              "MVUE: valid tokens must be a positive multiple of 4 in (n - 128, n] (got %lld of %lld)",
              (long long)n_valid, (long long)n);
  S24_REQUIRE(n % 128 == 0 && f % 128 == 0 && n > 0 && f > 0, S24_ERR_SHAPE,
              "MVUE operand needs tokens and features divisible by 128 (got n=%lld f=%lld)", (long long)n,
              (long long)f);
  S24_REQUIRE(ldg >= f && ldg % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0, S24_ERR_UNSUPPORTED,
              "gradient rows must be 16-byte aligned");
  if (gate_ff > 0) S24_REQUIRE(f == 2 * gate_ff && gate_ff % 16 == 0, S24_ERR_SHAPE, "gated MVUE: f must be 2 d_ff");
  MvueRng rng;
  mvue_rng_tables(rng, state_hi, state_lo, inc_hi, inc_lo, static_cast<uint64_t>(n_valid / 4));
  S24_REQUIRE(static_cast<double>(f) * static_cast<double>(n / 4) < 1099511627776.0, S24_ERR_SHAPE,
              "MVUE stream index exceeds the 2^40 jump table");
  S24_REQUIRE(exact || static_cast<double>(f) * static_cast<double>(n / 4) < 4294967296.0, S24_ERR_SHAPE,
              "fast MVUE: group counter exceeds 2^32 (use exact mode or split the call)");
  MvueArgs a{g, ldg, n, f, gate_ff, vals, e, pairs, exact == 2 ? 1 : 0, n_valid};
  dim3 grid(static_cast<unsigned>(n / 128), static_cast<unsigned>(f / 128));
  if (exact) {
    constexpr int kPkBytes = 128 * 33 * 4;
    static bool attr[64] = {false};  // per device: the opt-in belongs to the kernel, not to the call
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
      cudaFuncSetAttribute(mvue_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPkBytes);
      if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    mvue_tile_kernel<true><<<grid, 256, kPkBytes, static_cast<cudaStream_t>(stream)>>>(a, rng);
  }
  else mvue_tile_kernel<false><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, rng);
  return s24_check_launch("mvue_compress");
}
