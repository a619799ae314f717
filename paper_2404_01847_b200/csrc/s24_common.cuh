// Shared device helpers for the sm_100a kernels: status plumbing, mbarrier,
// TMA (cp.async.bulk[.tensor]), and tcgen05 (TMEM alloc / MMA / ld / cp)
// wrappers written directly in PTX.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/sparse24_b200.h"

// ---------------------------------------------------------------------------
// host-side status helpers (defined in s24_capi.cu)

int s24_set_error(int code, const char* fmt, ...);
int s24_check_launch(const char* what);

#define S24_REQUIRE(cond, code, ...)                     \
  do {                                                   \
    if (!(cond)) return s24_set_error((code), __VA_ARGS__); \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers

namespace s24 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "S24_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra S24_DONE_%=;\n\t"
      "bra S24_WAIT_%=;\n"
      "S24_DONE_%=:\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---- TMA ---------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                            int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(gmem_src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---- tcgen05 -----------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]   (kind::f16, bf16 in, fp32 accumulate)
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// sparse A (2:4, metadata in TMEM at e_tmem)
__device__ __forceinline__ void mma_sp_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t e_tmem,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// smem (128 rows x 16 B) -> TMEM (128 lanes x 4 columns)
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

// 16 lanes x 256 bit, 4 repetitions along columns -> 16 registers per thread in the m16n8
// accumulator-fragment layout: thread t holds, for column group c (8 columns each),
// r[4c + 0, 1] = (lane t/4,     columns 8c + 2(t%4) + {0, 1})
// r[4c + 2, 3] = (lane t/4 + 8, columns 8c + 2(t%4) + {0, 1})
__device__ __forceinline__ void tmem_ld16x256b_x4(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// four 8x8 bf16 matrices (fragment layout) stored transposed: matrix j's row i goes to the
// 16-byte smem row whose address thread 8j + i supplies
__device__ __forceinline__ void stmatrix_x4_trans(uint32_t saddr, uint32_t r0, uint32_t r1, uint32_t r2,
                                                  uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(r0),
               "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}

// ---- cta_group::2 (CTA pair) variants -------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// TMA load whose completion bytes land on the leader CTA's mbarrier (peer bit cleared)
__device__ __forceinline__ void tma_load_2d_cg2(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                                int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
// CTA-pair TMA load multicast to the CTAs in `mask` (same smem offset in each); each
// destination's completion bytes land on the same-offset mbarrier of its pair's leader CTA
__device__ __forceinline__ void tma_load_mc_cg2(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                                int32_t y, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                         int32_t y) {
  if constexpr (CG == 1) tma_load_2d(smem_dst, map, bar, x, y);
  else tma_load_2d_cg2(smem_dst, map, bar, x, y);
}
// 4-D box load (coordinates x, 0, 0, w): the u/v row interleave of a gated dense weight
// (dims: inner, 16 rows, 2 halves, row groups -- see make_map_gate in s24_gemm.cu)
template <int CG>
__device__ __forceinline__ void tma_load4(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t x,
                                          int32_t w) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %4, %5}], "
        "[%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(0), "r"(w)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%3, %4, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(0), "r"(w)
        : "memory");
  }
}
// arrive on the same-offset mbarrier of CTA `cta` in the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* smem_result, uint32_t ncols) {
  if constexpr (CG == 1) {
    tmem_alloc(smem_result, ncols);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 1) tmem_dealloc(taddr, ncols);
  else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_bf16_cg(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  if constexpr (CG == 1) {
    mma_bf16(d_tmem, adesc, bdesc, idesc, accumulate);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void mma_sp_bf16_cg(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t e_tmem,
                                               uint32_t idesc, uint32_t accumulate) {
  if constexpr (CG == 1) {
    mma_sp_bf16(d_tmem, adesc, bdesc, e_tmem, idesc, accumulate);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// commit all prior tcgen05 ops of this thread to the mbarrier at the same smem
// offset in every CTA of the pair (CG=2) or in this CTA (CG=1)
template <int CG>
__device__ __forceinline__ void mma_commit_cg(uint64_t* bar, uint16_t mask = 0x3) {
  if constexpr (CG == 1) {
    mma_commit(bar);
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_cp_128x128b_cg(uint32_t taddr, uint64_t sdesc) {
  if constexpr (CG == 1) tmem_cp_128x128b(taddr, sdesc);
  else asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// ---- TMA store (smem -> global), bulk-group completion ----------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(x), "r"(y)
               : "memory");
}
// element-wise add-reduce of the smem tile into global (type from the tensor map)
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* smem_src, int32_t x, int32_t y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Fast erf for |error| < 2e-7 (Abramowitz & Stegun 7.1.26), returning also
// exp(-x^2) so GELU' can reuse it for the Gaussian density.
__device__ __forceinline__ float erf_fast(float x, float& e_mx2) {
  const float ax = fabsf(x);
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, ax, 1.0f)));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  e_mx2 = __expf(-ax * ax);
  const float r = fmaf(-p, e_mx2, 1.0f);
  return copysignf(r, x);
}
// exact-erf GELU 0.5 x (1 + erf(x / sqrt 2)) with the fast erf
__device__ __forceinline__ float gelu_fast(float x) {
  float e;
  return 0.5f * x * (1.0f + erf_fast(x * 0.70710678118654752f, e));
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// GELU(x) = x Phi(x) and GELU'(x) = Phi(x) + x phi(x) with ONE MUFU op (GEMM epilogues, where
// the MUFU pipe is the limit): Phi(x) ~ 0.5 (1 + tanh(x (a + b x^2 + c x^4))) with a, b, c
// minimax-fitted to the exact-erf GELU on [0, 9] (|err| < 4e-5 for GELU, < 1e-4 for GELU' with
// an exact tanh; tanh.approx adds <= 2.5e-4 |x|, a twentieth of a bf16 ulp of the stored value).
// |x| > 9 saturates exactly (Phi = 0 or 1).
__device__ __forceinline__ void gelu_and_grad(float x, float& g, float& dg) {
  constexpr float kA = 0.797422874f, kB = 0.0370039386f, kC = -3.47603262e-4f;
  const float xc = fminf(fmaxf(x, -9.0f), 9.0f);
  const float x2 = xc * xc;
  const float t = tanh_approx(xc * fmaf(fmaf(kC, x2, kB), x2, kA));
  const float cdf = fmaf(0.5f, t, 0.5f);
  g = x * cdf;
  const float hdp = fmaf(fmaf(2.5f * kC, x2, 1.5f * kB), x2, 0.5f * kA);  // half the derivative of the tanh argument
  dg = fmaf(xc * fmaf(-t, t, 1.0f), hdp, cdf);
}
// Two elements of gelu_and_grad with the packed f32x2 FFMA2 / FMUL2 of sm_100 (half the FP
// instructions: the two-slab GEMM epilogue is not overlapped with the main loop, so its drain is
// issue-bound).  The clamp moves to x^2 <= 81: for |x| > 9 the tanh argument x * p(81) (p(81) > 1.5)
// saturates tanh to +-1 exactly as the clamped argument does, so g = x Phi and the derivative term
// x (1 - t^2) = 0 come out the same.
__device__ __forceinline__ void gelu_and_grad2(float x0, float x1, float& g0, float& g1, float& d0, float& d1) {
  constexpr float kA = 0.797422874f, kB = 0.0370039386f, kC = -3.47603262e-4f;
  const float2 x = make_float2(x0, x1);
  float2 x2 = __fmul2_rn(x, x);
  x2 = make_float2(fminf(x2.x, 81.0f), fminf(x2.y, 81.0f));
  const float2 p = __ffma2_rn(__ffma2_rn(make_float2(kC, kC), x2, make_float2(kB, kB)), x2, make_float2(kA, kA));
  const float2 u = __fmul2_rn(x, p);
  const float2 t = make_float2(tanh_approx(u.x), tanh_approx(u.y));
  const float2 cdf = __ffma2_rn(make_float2(0.5f, 0.5f), t, make_float2(0.5f, 0.5f));
  const float2 g = __fmul2_rn(x, cdf);
  // x (1 - t^2) = 4 g (1 - Phi): the factor 4 goes into the derivative polynomial, and 1 - Phi
  // needs no negated operand (a negated register costs an extra FADD per element)
  const float2 hdp4 = __ffma2_rn(__ffma2_rn(make_float2(10.0f * kC, 10.0f * kC), x2, make_float2(6.0f * kB, 6.0f * kB)),
                                 x2, make_float2(2.0f * kA, 2.0f * kA));
  const float2 omc = __ffma2_rn(make_float2(-0.5f, -0.5f), t, make_float2(0.5f, 0.5f));
  const float2 d = __ffma2_rn(__fmul2_rn(g, omc), hdp4, cdf);
  g0 = g.x;
  g1 = g.y;
  d0 = d.x;
  d1 = d.y;
}
// sigmoid(u) = 0.5 + 0.5 tanh(u / 2): one MUFU op
__device__ __forceinline__ float sigmoid_fast(float u) { return fmaf(0.5f, tanh_approx(0.5f * u), 0.5f); }

// UMMA shared-memory matrix descriptor (sm_100 "version 1" format):
//   [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 |
//   [49,52) base offset | [52] lbo mode | [61,64) layout (0 none, 2 = 128B swizzle)
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                               uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout & 7) << 61;
  return d;
}

// Instruction descriptor for kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool a_mn, bool b_mn, bool sparse) {
  return (sparse ? (1u << 2) : 0u) | (1u << 4) /*D f32*/ | (1u << 7) /*A bf16*/ | (1u << 10) /*B bf16*/ |
         ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((static_cast<uint32_t>(N) >> 3) << 17) |
         ((static_cast<uint32_t>(M) >> 4) << 24);
}

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}
// one F2FP.BF16.F32.PACK_AB (an ALU op) instead of two F2F conversions on the XU pipe
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

}  // namespace s24
