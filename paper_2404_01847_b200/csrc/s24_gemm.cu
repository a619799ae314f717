// K3/K4 (2:4-sparse) and K5 (dense dW) GEMMs on the 5th-generation tensor
// cores: tcgen05.mma[.sp] issued by one thread, operands staged in shared
// memory by TMA (128-byte swizzle), fp32 accumulators in TMEM, metadata for the
// sparse A operand copied smem -> TMEM with tcgen05.cp.
//
// D[m, n] = sum_k A[m, k] * B[n, k]
//   sparse (K3/K4): A = compressed W (m x k/2 bf16, K-major) + E tiles,
//                   B = activations (n tokens), D bf16 (+bias, +fused GELU).
//                   Replaces kernels.spmm_colwise (_core.pyx:63-80) as used by
//                   _GatherPlan.product (gated_ffn.py:159-162).
//   dense  (K5):    A, B = activation / gradient panels (K = tokens),
//                   D fp32 = dW + lambda (1 - M) W  (masked decay epilogue).
//                   Replaces _grad_weight(mvue=False) (gated_ffn.py:367-371)
//                   + masked_decay_gradient (optim.py:105-114).
//
// CTA layout (384 threads, one CTA per SM, CTA pairs (cta_group::2) sharing one MMA,
// persistent over output tiles):
//   warp 0       TMA producer (one elected lane; wave-synchronised for the dW GEMMs)
//   warp 1       MMA issuer (one elected lane of the pair's even CTA) + tcgen05.cp of
//                the sparse metadata
//   warp 2       TMEM allocator
//   warps 4..11  epilogue (lane quarter = warp % 4, two warps per quarter alternating
//                32-column chunks): token-major outputs on the fragment path
//                (tcgen05.ld 16x256b -> bf16x2 -> stmatrix.trans -> TMA store),
//                dW / feature-major outputs on the row path (tcgen05.ld 32x32b)
// Pipelines: kStages smem slots (full/empty mbarriers) and, for one-slab tiles, two
// TMEM accumulators (tmem_full/tmem_empty) so the epilogue of tile i overlaps the main
// loop of tile i+1; two-slab tiles (kSlabs = 2) trade that overlap for 512-row tiles.
// GemmShape::exp holds experiment flags for attribution studies (results invalid when
// set; 0 in production).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "s24_common.cuh"
#include "s24_patterns.h"

namespace s24 {

constexpr int kGemmThreads = 384;  // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;

// epilogues: plain store (+bias); Z and GELU(Z); GELU(Z) and GELU'(Z) (training forward);
// dZ = acc * GELU'(Z) with bias-gradient row sums (training backward); dW fp32 + masked decay
// gated (GEGLU / SwiGLU) training epilogues on the u/v-interleaved first weight:
// kEpiGatedGrad: A = act(u) * v (token-major) + AUX = v * act'(u), AUX2 = act(u) (feature-major)
// kEpiDGated:    dZ_u = dA * AUX, dZ_v = dA * AUX2 into the interleaved token-major dZ, bias grads
enum Epi : int {
  kEpiStore = 0, kEpiGeluAux = 1, kEpiDw = 2, kEpiGeluGrad = 3, kEpiDAct = 4, kEpiGatedGrad = 5, kEpiDGated = 6
};

struct EpiParams {
  void* d;
  int64_t ldd;
  const uint16_t* bias;
  uint16_t* aux;     // second output (kEpiGeluAux, kEpiGeluGrad) or GELU'(Z) input (kEpiDAct)
  int64_t ldaux;
  float* dbias;      // kEpiDAct / kEpiDGated: bias-gradient accumulator (zeroed by the caller)
  uint16_t* aux2;    // kEpiGatedGrad output / kEpiDGated input (same pitch as aux)
  int act;           // S24_ACT_GEGLU or S24_ACT_SWIGLU for the gated epilogues
  int64_t gate_ff;   // d_ff of the u/v interleave (gated epilogues, dW row remap); 0 = none
  const void* w;
  int w_dtype;
  const uint8_t* idx;
  float lam;
  int accumulate;    // kEpiStore, token-major: D += acc via TMA bf16 add-reduce (S24_EPI_STORE_ADD)
};

struct GemmShape {
  int m, n, k;  // k logical
  int streamk;  // 1: stream-K -- every cluster owns an equal run of (tile, k-block) iterations and
                //    partial tiles are summed with TMA add-reduce stores into the zeroed output;
                // S >= 2: lockstep split-K (WorkIter), partial tiles add-reduced the same way
  int group_m;  // M tiles per raster group: each group sweeps all N with its A panels L2-resident
  unsigned int* ws;  // caller's GEMM workspace (S24 ABI: zeroed once, left zeroed by every launch), or NULL
  int wave_sync;     // wave-synchronised schedule on ws[kWsWave] (see below; needs ws)
  int exp;      // experiment flags (timing studies only, results invalid): 1 skip B loads, 2 skip metadata cp, 4 every tile loads the B tile of n = 0,
                //  16 no activation math in the epilogue, 32 no epilogue global loads,
                //  128 no GELU'(z) AUX stores, 256 no D stores (fragment epilogue)
  int a_gate;   // dense A through the 4-D u/v interleave map (gated first weight in [u; v] order)
};

// Experiment flags exist only in builds with -DS24_EXPERIMENTS (attribution studies); in the
// production library every S24_EXP(f) is a compile-time false and the flag code is gone.
#ifdef S24_EXPERIMENTS
#define S24_EXP(f) ((shp.exp & (f)) != 0)
#else
#define S24_EXP(f) (false)
#endif

__constant__ uint16_t c_gemm_pat_bits[90] = S24_PATTERN_BITS;

// interleaved row p of the gated first weight -> row of [u; v] (see s24_mask.cu)
__device__ __forceinline__ int gate_row_dev(int p, int64_t ff) {
  return (p & 31) < 16 ? 16 * (p >> 5) + (p & 31) : static_cast<int>(ff) + 16 * (p >> 5) + (p & 31) - 16;
}

template <bool kSilu>
__device__ __forceinline__ void gate_act(float u, float& a, float& da) {
  if constexpr (kSilu) {
    const float sg = sigmoid_fast(u);
    a = u * sg;
    da = sg * fmaf(u, 1.0f - sg, 1.0f);
  } else {
    gelu_and_grad(u, a, da);
  }
}

// AUX layout exchanged between GEMM1's and GEMM3's fragment epilogues (GELU'(z), v act'(u),
// act(u); an F x n bf16 matrix, F rounded up to 16): 16-feature x 32-token sub-blocks of 1 KB,
// sub-block (f / 16, t / 32) at element ((f / 16) (n / 32) + t / 32) * 512.  Inside, 16-byte unit
// 32 s + 4 r + p holds feature 8 s + r (s = (f % 16) / 8, r = f % 8) at tokens 8 c + 2 p + k
// (c = 0..3, k = 0, 1, element 2 c + k): exactly what thread 4 r + p of a 16x256b TMEM load
// holds, so each warp reads or writes a sub-block as two coalesced 512-byte accesses.
__device__ __forceinline__ uint4* aux_frag(uint16_t* base, int f16blk, int n, int n0) {
  return reinterpret_cast<uint4*>(base + (static_cast<int64_t>(f16blk) * (n >> 5) + (n0 >> 5)) * 512);
}

// kCG = CTAs per MMA (1: M = 128, 2: CTA pair, M = 256, B split along N).
// Pipeline depth that fits next to the epilogue staging area.
template <int kStageBytes>
constexpr int stages_for() {
  constexpr int budget = 232448 - 1024 - 256 - kEpiWarps * 4096;
  return budget / kStageBytes > 6 ? 6 : budget / kStageBytes;
}

// kSlabs = 2 (sparse, plain-store epilogue, long K): every CTA holds TWO 128-row A slabs
// against one B tile -- a 512 x kBN pair tile in one TMEM accumulator (2 x kBN columns), so
// each B byte delivered from L2 feeds twice the MACs (operand bytes per MAC -30 %) at the
// price of an epilogue that no longer overlaps the main loop (a few % at K >= 8192).
template <bool kSparse, bool kAMN, bool kBMN, int kBN, int kStages, int kCG, int kAcc = 2, int kSlabs = 1>
struct Cfg {
  static constexpr int BK = kSparse ? 128 : 64;  // logical K per stage
  static constexpr int kMmaK = kSparse ? 32 : 16;
  static constexpr int kMmasPerStage = BK / kMmaK;  // 4
  static constexpr int BN_CTA = kBN / kCG;          // B rows held by one CTA
  static constexpr int B_CHUNKS = (BN_CTA + 63) / 64;  // MN-major 64-wide swizzle chunks
  static constexpr int A_BYTES = kSlabs * 128 * 64 * 2;  // 16 KB per slab, either major
  static constexpr int B_BOX_BYTES = kBMN ? BK * 128 : BN_CTA * 128;
  static constexpr int B_BOXES = kBMN ? B_CHUNKS : BK / 64;
  static constexpr int B_BYTES = B_BOXES * B_BOX_BYTES;
  static constexpr int E_BYTES = kSparse ? kSlabs * 2048 : 0;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + E_BYTES;
  static constexpr int TX_BYTES = A_BYTES + (kBMN ? B_BYTES : BN_CTA * BK * 2) + E_BYTES;  // per CTA
  static constexpr int ACC_COLS = kSlabs * kBN;
  static constexpr int E_COL = kAcc * ACC_COLS;  // kAcc TMEM accumulators (2: epilogue overlaps the next tile)
  static constexpr int USED_COLS = kAcc * ACC_COLS + (kSparse ? 4 * kSlabs : 0);
  static constexpr int TILE_M = 128 * kCG * kSlabs;  // output rows per (pair) tile
  static constexpr int TMEM_COLS = USED_COLS <= 32 ? 32 : USED_COLS <= 64 ? 64 : USED_COLS <= 128 ? 128
                                 : USED_COLS <= 256 ? 256 : 512;
  static constexpr int EPI_OFF = kStages * STAGE_BYTES;          // per-warp 4 KB output staging
  static constexpr int BAR_OFF = EPI_OFF + kEpiWarps * 4096;
  static constexpr int SMEM_BYTES = BAR_OFF + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t IDESC = make_idesc_bf16(128 * kCG, kBN, kAMN, kBMN, kSparse);
  static_assert(USED_COLS <= 512, "TMEM overflow");
  static_assert(kBN % 32 == 0 && kBN >= 32 && kBN <= 256, "bad BN");
  static_assert(B_BOX_BYTES % 1024 == 0, "B boxes must stay 1024-byte aligned for the 128B swizzle");
  static_assert(SMEM_BYTES <= 232448, "shared memory overflow");
};

// Work walk shared by the producer, MMA and epilogue roles: static round-robin over whole
// tiles, or stream-K (cluster c owns linear k-block iterations [c T / C, (c + 1) T / C) of
// T = tiles x k-blocks, so every cluster does the same work whatever the tile count).
// Wave synchronisation.  A persistent kernel's CTAs drift apart over many waves (a few percent
// speed difference per SM accumulates), so CTAs that should share A / B panels in L2 end up
// a wave apart and every panel streams from HBM several times (measured on B200: dW_in at C3
// read 15.3 GB with drift, 7.0 GB wave-synchronised, and ran 10% faster at the higher clock
// the lower HBM power allowed).  Each producer counts the tiles whose loads it has issued and,
// before the first load of wave w, waits until all CTAs have issued wave w - 1.  Purely a
// locality hint: the wait is bounded (~20 us), so CTAs that are not co-resident (an SM taken
// by another kernel) only cost time, never a hang -- and a wait that gives up is counted in
// ws[kWsTimeouts], so the caller can see that the locality (or, below, ordering) guarantee was
// dropped.  The last CTA to exit resets the counters, so every launch (and every CUDA-graph
// replay) starts from zero.  The counters live in the CALLER's workspace (one per stream), not
// in library globals: concurrent launches on different streams never share them.
constexpr int kWsWave = 0, kWsExit = 1, kWsTimeouts = 2, kWsSplit = 16;

// Ordered split-K (WorkIter mode S >= 3): the S partial tiles of one output tile are add-reduced
// in split order, so the fp32 sums are run-to-run identical.  Every storer (epilogue warp of
// either CTA of the pair) of split s waits until all storers of split s - 1 have completed their
// bulk reduce-adds (per-tile counter, bounded spin: the order is a determinism guarantee, the sum
// is correct either way), and the storer that completes the last split resets the counter.
constexpr int kSplitTiles = 2048;
static_assert((kWsSplit + kSplitTiles) * 4 <= S24_GEMM_WORKSPACE_BYTES, "GEMM workspace too small");

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct WorkIter {
  long long it, end, total;
  int tile, stride, split, ncl, head_tile = 0, head_kb1 = 0;
  bool sk;
  // mode 0: one full-K tile per step; S >= 2: lockstep split-K -- every tile is cut into S equal
  // K ranges, unit u = s * num_tiles + tile, so the clusters of one wave all sit at the same
  // relative K offset of their range and keep sharing operand panels in L2.
  // mode 1: K-aligned stream-K -- cluster c owns the run [T c / ncl, T (c + 1) / ncl) of the
  // (tile, k-block) space (T = tiles * num_kb) and processes the run's LAST segment first: that
  // segment starts at k-block 0 of its tile, like every other cluster's first segment, so all
  // clusters sweep K together; the remaining tail of the previous tile follows, at most
  // (1 - tiles / ncl) * num_kb k-blocks ahead of the others when the run is shorter than a tile
  __device__ __forceinline__ WorkIter(int mode, int num_tiles, int num_kb, int cid, int ncl_)
      : split(mode >= 2 ? mode : 1), ncl(ncl_), sk(mode == 1) {
    total = static_cast<long long>(num_tiles) * num_kb;
    it = sk ? total * cid / ncl : 0;
    end = sk ? total * (cid + 1) / ncl : 0;
    if (sk) {
      const long long b = end / num_kb;
      const int ke = static_cast<int>(end - b * num_kb);
      if (ke > 0 && b * num_kb > it) {  // the run ends inside tile b and starts before it
        head_tile = static_cast<int>(b);
        head_kb1 = ke;
        end = b * num_kb;
      }
    }
    tile = cid;
    stride = ncl;
  }
  // stream-K: how many runs start at or before linear k-block x (run starts floor(T c / ncl))
  __device__ __forceinline__ long long runs_upto(long long x) const {
    const long long c = ((x + 1) * ncl + total - 1) / total;
    return c < ncl ? c : ncl;
  }
  // next segment: output tile and its k-block range [kb0, kb1)
  int last_split = 0;   // index of the returned segment among its tile's K segments (K order)
  int last_nsplit = 1;  // number of K segments of that tile
  __device__ __forceinline__ bool next(int num_tiles, int num_kb, int& t, int& kb0, int& kb1) {
    if (sk) {
      if (head_kb1 > 0) {
        t = head_tile;
        kb0 = 0;
        kb1 = head_kb1;
        head_kb1 = 0;
      } else {
        if (it >= end) return false;
        t = static_cast<int>(it / num_kb);
        kb0 = static_cast<int>(it - static_cast<long long>(t) * num_kb);
        kb1 = static_cast<int>(min(static_cast<long long>(num_kb), kb0 + (end - it)));
        it += kb1 - kb0;
      }
      const long long base = static_cast<long long>(t) * num_kb;
      const long long r0 = runs_upto(base);
      last_split = static_cast<int>(runs_upto(base + kb0) - r0);
      last_nsplit = static_cast<int>(runs_upto(base + num_kb - 1) - r0) + 1;
      return true;
    }
    if (tile >= num_tiles * split) return false;
    const int s = tile / num_tiles;
    last_split = s;
    last_nsplit = split;
    t = tile - s * num_tiles;
    kb0 = static_cast<int>(static_cast<long long>(num_kb) * s / split);
    kb1 = static_cast<int>(static_cast<long long>(num_kb) * (s + 1) / split);
    tile += stride;
    return true;
  }
};

__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * num_n;
  const int group = tile / per_group;
  const int first_m = group * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int in_group = tile % per_group;
  mb = first_m + in_group % gm;
  nb = in_group / gm;
}

// kMC = CTA pairs per cluster.  kMC = 2: the two pairs of a 4-CTA cluster compute vertically
// adjacent tiles (m-tiles 2 i and 2 i + 1, same n-tile) and share the B (token) tile: each CTA
// TMA-loads half of its 112-row B half and multicasts it to the CTA at the same position in the
// other pair, halving the L2 reads of B.  A stage is reused only after both pairs' MMAs have
// released it (empty barriers count kMC arrivals, MMA commits multicast to all four CTAs).
template <bool kSparse, bool kAMN, bool kBMN, int kBN, int kStages, int kCG, int kEpi, bool kOutT, int kAcc,
          int kSlabs, int kMC>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmD,
                const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY, GemmShape shp,
                EpiParams ep) {
  using C = Cfg<kSparse, kAMN, kBMN, kBN, kStages, kCG, kAcc, kSlabs>;
  // token-major training / plain-store epilogues run on the fragment path (tcgen05.ld 16x256b +
  // stmatrix); the masked-decay dW epilogue and the API's z / GELU(z) epilogue on the row path
  constexpr bool kFrag = kOutT && (kEpi == kEpiStore || kEpi == kEpiGeluGrad || kEpi == kEpiDAct ||
                                   kEpi == kEpiGatedGrad || kEpi == kEpiDGated);
  static_assert(kOutT || !(kEpi == kEpiGeluGrad || kEpi == kEpiDAct || kEpi == kEpiGatedGrad || kEpi == kEpiDGated),
                "training epilogues store token-major outputs");
  static_assert(kSlabs == 1 || (kAcc == 1 && ((kSparse && kFrag) || kEpi == kEpiDw)),
                "slabs: sparse fragment epilogues or the dW epilogue only");
  static_assert(kMC == 1 || (kMC == 2 && kSparse && kCG == 2 && !kBMN && kSlabs == 1), "multicast: sparse pairs only");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = kCG == 2 ? cluster_rank() : 0;  // rank in the cluster
  const uint32_t rank = crank & (kCG - 1);                 // rank in the CTA pair
  const int pr = static_cast<int>(crank) / kCG;            // pair in the cluster (kMC = 2)
  // a two-slab tile may hang half over the last rows (m % 256 == 0): its second slab reads
  // zero-filled TMA boxes and its epilogue is skipped
  const int num_m = (shp.m + C::TILE_M - 1) / C::TILE_M;
  const int num_n = (shp.n + kBN - 1) / kBN;
  const int num_kb = shp.k / C::BK;  // k-blocks per output tile
  const int cluster_id = blockIdx.x / (kCG * kMC), num_clusters = gridDim.x / (kCG * kMC);
  // work tiles of the cluster: kMC vertically adjacent pair tiles (num_m % kMC == 0)
  const int num_mc = num_m / kMC;
  const int num_work = num_mc * num_n;
  auto coords = [&](int tile, int& mb, int& nb) {
    tile_coords(tile, num_mc, num_n, shp.group_m, mb, nb);
    mb = mb * kMC + pr;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmD);
    if constexpr (kSparse) tma_prefetch(&tmE);
    if constexpr (kEpi == kEpiGeluAux) tma_prefetch(&tmX);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kMC);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kEpiWarps * kCG);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_cg<kCG>(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  if constexpr (kCG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (every CTA of the pair) =====================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      WorkIter wk(shp.streamk, num_work, num_kb, cluster_id, num_clusters);
      int tile, kb0, kb1, wave = 0;
      unsigned int* wctr = (shp.ws != nullptr && shp.wave_sync && shp.streamk != 1) ? shp.ws + kWsWave : nullptr;
      while (wk.next(num_work, num_kb, tile, kb0, kb1)) {
        if (wctr != nullptr && wave > 0) {
          // every producer has issued the previous wave's loads (bounded wait)
          const unsigned int target = gridDim.x * wave;
          const long long t0 = clock64();
          bool late = false;
          while (static_cast<int>(ld_acquire_gpu(wctr) - target) < 0) {
            if (clock64() - t0 >= 40000) {
              late = true;
              break;
            }
            __nanosleep(32);
          }
          if (late) atomicAdd(shp.ws + kWsTimeouts, 1u);
        }
        int mb, nb;
        coords(tile, mb, nb);
        const int m0 = mb * C::TILE_M + 128 * rank;      // this CTA's A rows (slab s: + 128 kCG s)
        const int nb0 = (S24_EXP(4) ? 0 : nb * kBN) + C::BN_CTA * rank;  // this CTA's B rows (N split)
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + C::A_BYTES;
          const bool skip_b = S24_EXP(1);
          if (rank == 0)
            mbar_expect_tx(&full_bar[stage], (C::TX_BYTES - (skip_b ? C::TX_BYTES - C::A_BYTES - C::E_BYTES : 0)) * kCG);
          if constexpr (kSparse) {
#pragma unroll
            for (int sl = 0; sl < kSlabs; ++sl) {
              const int ms = m0 + 128 * kCG * sl;
              tma_load<kCG>(sA + sl * 16384, &tmA, &full_bar[stage], kb * 64, ms);  // 64 physical = 128 logical
              tma_load<kCG>(sB + C::B_BYTES + sl * 2048, &tmE, &full_bar[stage], 0, (ms / 128) * (shp.k / 128) + kb);
            }
          } else {
#pragma unroll
            for (int sl = 0; sl < kSlabs; ++sl) {
              const int ms = m0 + 128 * kCG * sl;
              if constexpr (kAMN) {
                if (shp.a_gate) {  // K runs over the interleaved rows: 64 of them = 2 row groups
                  tma_load4<kCG>(sA + sl * 16384, &tmA, &full_bar[stage], ms, 2 * kb);
                  tma_load4<kCG>(sA + sl * 16384 + 8192, &tmA, &full_bar[stage], ms + 64, 2 * kb);
                } else {
                  tma_load<kCG>(sA + sl * 16384, &tmA, &full_bar[stage], ms, kb * 64);
                  tma_load<kCG>(sA + sl * 16384 + 8192, &tmA, &full_bar[stage], ms + 64, kb * 64);
                }
              } else {
                if (shp.a_gate) tma_load4<kCG>(sA + sl * 16384, &tmA, &full_bar[stage], kb * 64, ms / 32);
                else tma_load<kCG>(sA + sl * 16384, &tmA, &full_bar[stage], kb * 64, ms);
              }
            }
          }
          if (skip_b) {
          } else if constexpr (kBMN) {
#pragma unroll
            for (int i = 0; i < C::B_CHUNKS; ++i)
              tma_load<kCG>(sB + i * C::B_BOX_BYTES, &tmB, &full_bar[stage], nb0 + 64 * i, kb * C::BK);
          } else if constexpr (kMC == 2) {
            // my half of this CTA's B rows, multicast to the same-position CTA of both pairs
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (kCG + rank)));
#pragma unroll
            for (int i = 0; i < C::BK / 64; ++i)
              tma_load_mc_cg2(sB + i * C::B_BOX_BYTES + pr * (C::BN_CTA / 2) * 128, &tmB, &full_bar[stage],
                              kb * C::BK + 64 * i, nb0 + pr * (C::BN_CTA / 2), mask);
          } else {
#pragma unroll
            for (int i = 0; i < C::BK / 64; ++i)
              tma_load<kCG>(sB + i * C::B_BOX_BYTES, &tmB, &full_bar[stage], kb * C::BK + 64 * i, nb0);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (wctr != nullptr) atomicAdd(wctr, 1u);
        ++wave;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (rank == 0 && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      WorkIter wk(shp.streamk, num_work, num_kb, cluster_id, num_clusters);
      int tile, kb0, kb1;
      while (wk.next(num_work, num_kb, tile, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b_addr = a_addr + C::A_BYTES;
          if (kSparse && !S24_EXP(2)) {
            // metadata: 128 rows x 16 B (no swizzle, 8-row core matrices 128 B apart) -> 4 TMEM columns
#pragma unroll
            for (int sl = 0; sl < kSlabs; ++sl)
              tmem_cp_128x128b_cg<kCG>(tmem_base + C::E_COL + 4 * sl,
                                       make_sdesc(b_addr + C::B_BYTES + sl * 2048, 2048, 128, 0));
          }
#pragma unroll
          for (int j = 0; j < C::kMmasPerStage; ++j) {
            uint64_t adesc, bdesc;
            if constexpr (kAMN) {
              adesc = make_sdesc(a_addr + j * (C::kMmaK * 128), 8192, 1024, 2);
            } else {
              adesc = make_sdesc(a_addr + j * 32, 16, 1024, 2);
            }
            if constexpr (kBMN) {
              bdesc = make_sdesc(b_addr + j * (C::kMmaK * 128), C::B_BOX_BYTES, 1024, 2);
            } else if constexpr (kSparse) {
              bdesc = make_sdesc(b_addr + (j >> 1) * C::B_BOX_BYTES + (j & 1) * 64, 16, 1024, 2);
            } else {
              bdesc = make_sdesc(b_addr + j * 32, 16, 1024, 2);
            }
            const uint32_t accum = (kb != kb0 || j != 0) ? 1u : 0u;
            if constexpr (kSparse) {
              // MMA j's metadata sits in TMEM column E_COL + 4 slab + j; the instruction takes a
              // 2-column-aligned address and selects the column with sparse_id2 (idesc[0:2))
#pragma unroll
              for (int sl = 0; sl < kSlabs; ++sl)
                mma_sp_bf16_cg<kCG>(d_tmem + sl * kBN, adesc + static_cast<uint64_t>((sl * 16384) >> 4), bdesc,
                                    tmem_base + C::E_COL + 4 * sl + (j & ~1), C::IDESC | static_cast<uint32_t>(j & 1),
                                    accum);
            } else {
#pragma unroll
              for (int sl = 0; sl < kSlabs; ++sl)
                mma_bf16_cg<kCG>(d_tmem + sl * kBN, adesc + static_cast<uint64_t>((sl * 16384) >> 4), bdesc, C::IDESC,
                                 accum);
            }
          }
          // release the stage in every CTA that reads it (both pairs when B is multicast)
          mma_commit_cg<kCG>(&empty_bar[stage], kMC == 2 ? 0xF : 0x3);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_cg<kCG>(&tfull_bar[acc], static_cast<uint16_t>(0x3u << (kCG * pr)));
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    if constexpr (kFrag) {
      // ============ fragment epilogue (token-major outputs, training epilogues) ============
      // tcgen05.ld 16x256b puts each thread on 4 rows (features m_w + 8j + t4, j = 2h + s) x 8
      // tokens (n0 + 8c + 2p + k, c = 0..3, p = lane % 4, k = 0, 1) of a 32 x 32 chunk: token
      // pairs pack into one bf16x2 register, stmatrix.trans writes the token-major tile into the
      // swizzled TMA staging (4 instructions per chunk), and the AUX exchange with the other
      // GEMM's epilogue is one 16-byte unit per (thread, row pair) -- see aux_frag.
      const int e = warp - 4, q = e & 3, cw = e >> 2;
      const int t4 = lane >> 2;
      uint8_t* stg = smem + C::EPI_OFF + e * 4096;
      // stmatrix row addresses: thread 8j + i addresses row i of matrix j
      const int mj = lane >> 3, mi = lane & 7;
      int acc = 0, sbuf = 0, par = 0;
      uint32_t acc_phase = 0;
      WorkIter wk(false, num_work, num_kb, cluster_id, num_clusters);
      int tile, kb0, kb1;
      for (; wk.next(num_work, num_kb, tile, kb0, kb1); par ^= 1) {
        int mb, nb;
        coords(tile, mb, nb);
        const int n_base = nb * kBN;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int slab = 0; slab < kSlabs; ++slab) {
        const int m_w = mb * C::TILE_M + 128 * kCG * slab + 128 * rank + 32 * q;  // first TMEM row of this warp
        if (kSlabs > 1 && m_w >= shp.m) continue;  // slab beyond the last row
        float bias4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // bias of row m_w + 8j + t4 (forward)
        float bs1[4] = {0.0f, 0.0f, 0.0f, 0.0f};    // bias-gradient partials (backward), u / plain
        float bs2[4] = {0.0f, 0.0f, 0.0f, 0.0f};    // v half (kEpiDGated)
        if constexpr (kEpi == kEpiStore || kEpi == kEpiGeluGrad || kEpi == kEpiGatedGrad) {
          if (ep.bias != nullptr) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int row = m_w + 8 * j + t4;
              bias4[j] = bf16_to_f32(ep.bias[kEpi == kEpiGatedGrad ? gate_row_dev(row, ep.gate_ff) : row]);
            }
          }
        }
        // AUX inputs of the backward epilogues, prefetched one chunk ahead (coalesced 512 B)
        constexpr bool kPre = kEpi == kEpiDAct || kEpi == kEpiDGated;
        uint4 pre[8];
        auto prefetch = [&](int cc) {
          const int n0p = n_base + 32 * cc;
          if (cc >= kBN / 32 || n0p >= shp.n) return;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4* gp = aux_frag(ep.aux, (m_w >> 4) + h, shp.n, n0p) + lane;
            pre[2 * h] = __ldg(gp);
            pre[2 * h + 1] = __ldg(gp + 32);
            if constexpr (kEpi == kEpiDGated) {
              const uint4* gp2 = aux_frag(ep.aux2, (m_w >> 4) + h, shp.n, n0p) + lane;
              pre[4 + 2 * h] = __ldg(gp2);
              pre[4 + 2 * h + 1] = __ldg(gp2 + 32);
            }
          }
        };
        // the two warps of a lane quarter take alternate chunks; the one starting flips per tile
        const int first = cw ^ par;
        if constexpr (kPre) prefetch(first);
        // TMEM loads run one chunk ahead: chunk cc + 2's tcgen05.ld is issued right after chunk
        // cc's data arrived, so its latency hides behind chunk cc's math and stores (the wait at
        // the top of the next iteration then finds it complete)
        uint32_t r[32];
        auto tmem_chunk = [&](int cc) {
          const uint32_t ta =
              tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * C::ACC_COLS + slab * kBN + 32 * cc;
          tmem_ld16x256b_x4(ta, r);
          tmem_ld16x256b_x4(ta + (16u << 16), r + 16);
        };
        if (first < kBN / 32) tmem_chunk(first);
#pragma unroll 1
        for (int cc = first; cc < kBN / 32; cc += 2) {
          uint4 cur[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cur[u] = pre[u];
          tmem_ld_wait();
          // v[16 h + 4 c + 2 s + k]: row m_w + 16 h + 8 s + t4, token n0 + 8 c + 2 p + k
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (cc + 2 < kBN / 32) tmem_chunk(cc + 2);
          const int n0 = n_base + 32 * cc;
          if (n0 >= shp.n) continue;
          if constexpr (kEpi == kEpiGatedGrad) {
            // h = 0: u rows, h = 1: the matching v rows of gate features fg + 8 s + t4
            const int fg = m_w >> 1;
            uint32_t pa[8], g1[8], g2[8];  // bf16x2 of (c, s): A = act(u) v, AUX = v act'(u), AUX2 = act(u)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
#pragma unroll
              for (int sl = 0; sl < 2; ++sl) {
                float a2[2], d2[2], o2[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                  const float u = v[4 * c + 2 * sl + k] + bias4[sl];
                  const float w = v[16 + 4 * c + 2 * sl + k] + bias4[2 + sl];
                  float a, da;
                  if S24_EXP(16) { a = u; da = u; }
                  else if (ep.act == S24_ACT_SWIGLU) gate_act<true>(u, a, da);
                  else gate_act<false>(u, a, da);
                  a2[k] = a * w;
                  d2[k] = w * da;
                  o2[k] = a;
                }
                pa[2 * c + sl] = pack_bf16x2(a2[0], a2[1]);
                g1[2 * c + sl] = pack_bf16x2(d2[0], d2[1]);
                g2[2 * c + sl] = pack_bf16x2(o2[0], o2[1]);
              }
            }
            // A: [32 tokens][16 features], 32-byte rows, 32B swizzle; matrices (c, s); two 1 KB
            // staging buffers, so the stmatrix of this chunk overlaps the previous chunk's store
            uint8_t* ab = stg + sbuf * 1024;
            const uint32_t ab_a = smem_u32(ab);
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int hc = 0; hc < 2; ++hc) {
              const int tok = 8 * (2 * hc + (mj >> 1)) + mi, sl = mj & 1;
              stmatrix_x4_trans(ab_a + tok * 32 + ((sl ^ ((tok >> 2) & 1)) << 4), pa[4 * hc], pa[4 * hc + 1],
                                pa[4 * hc + 2], pa[4 * hc + 3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmD, ab, fg, n0);
              bulk_commit();
            }
            sbuf ^= 1;
            uint4* p1 = aux_frag(ep.aux, fg >> 4, shp.n, n0) + lane;
            uint4* p2 = aux_frag(ep.aux2, fg >> 4, shp.n, n0) + lane;
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              p1[32 * sl] = make_uint4(g1[sl], g1[2 + sl], g1[4 + sl], g1[6 + sl]);
              p2[32 * sl] = make_uint4(g2[sl], g2[2 + sl], g2[4 + sl], g2[6 + sl]);
            }
          } else if constexpr (kEpi == kEpiDGated) {
            // dZ_u = dA AUX, dZ_v = dA AUX2 -> interleaved token-major dZ: this warp's 32 gate
            // features own the 64 columns [2 m_w, 2 m_w + 64): 32 h + 16 (v) + 8 s + row
            uint32_t pz[2][2][2][4];  // [h][u/v][s][c]
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int sl = 0; sl < 2; ++sl) {
                const uint4 x1 = cur[2 * h + sl], x2 = cur[4 + 2 * h + sl];
                const uint32_t a1[4] = {x1.x, x1.y, x1.z, x1.w}, a2[4] = {x2.x, x2.y, x2.z, x2.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const float da0 = v[16 * h + 4 * c + 2 * sl], da1 = v[16 * h + 4 * c + 2 * sl + 1];
                  const float z10 = da0 * __uint_as_float(a1[c] << 16), z11 = da1 * __uint_as_float(a1[c] & 0xFFFF0000u);
                  const float z20 = da0 * __uint_as_float(a2[c] << 16), z21 = da1 * __uint_as_float(a2[c] & 0xFFFF0000u);
                  bs1[2 * h + sl] += z10 + z11;
                  bs2[2 * h + sl] += z20 + z21;
                  pz[h][0][sl][c] = pack_bf16x2(z10, z11);
                  pz[h][1][sl][c] = pack_bf16x2(z20, z21);
                }
              }
            }
            // [32 tokens][64 columns] as two [32 tokens][32 columns] halves h (64-byte rows, 64B
            // swizzle, double-buffered 2 KB staging, one TMA store each); one stmatrix per c:
            // matrices j = (u/v, s) -> 16-byte column chunk j of half h
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint8_t* zb = stg + sbuf * 2048;
              const uint32_t zb_a = smem_u32(zb);
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int tok = 8 * c + mi;
                stmatrix_x4_trans(zb_a + tok * 64 + ((mj ^ ((tok >> 1) & 3)) << 4), pz[h][0][0][c], pz[h][0][1][c],
                                  pz[h][1][0][c], pz[h][1][1][c]);
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&tmD, zb, 2 * m_w + 32 * h, n0);
                bulk_commit();
              }
              sbuf ^= 1;
            }
          } else {
            // kEpiStore (+bias), kEpiGeluGrad (GELU(z) out, GELU'(z) to AUX), kEpiDAct (acc * AUX)
            uint32_t pd[16];  // bf16x2 of (h, c, s) at 8 h + 2 c + s ... stored as [c][j], j = 2 h + s
            if constexpr (kEpi == kEpiDAct) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 x = cur[j];
                const uint32_t a[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  float& v0 = v[16 * (j >> 1) + 4 * c + 2 * (j & 1)];
                  float& v1 = v[16 * (j >> 1) + 4 * c + 2 * (j & 1) + 1];
                  v0 *= __uint_as_float(a[c] << 16);
                  v1 *= __uint_as_float(a[c] & 0xFFFF0000u);
                  bs1[j] += v0 + v1;
                }
              }
            }
            uint4 gaux[4];  // GELU'(z) units, stored after the TMA store is issued (see below)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t gq[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                float x0 = v[16 * (j >> 1) + 4 * c + 2 * (j & 1)];
                float x1 = v[16 * (j >> 1) + 4 * c + 2 * (j & 1) + 1];
                if constexpr (kEpi == kEpiStore) {
                  x0 += bias4[j];
                  x1 += bias4[j];
                } else if constexpr (kEpi == kEpiGeluGrad) {
                  const float2 xb = __fadd2_rn(make_float2(x0, x1), make_float2(bias4[j], bias4[j]));
                  x0 = xb.x;
                  x1 = xb.y;
                }
                if constexpr (kEpi == kEpiGeluGrad) {
                  float g0, g1, d0, d1;
                  if S24_EXP(16) { g0 = d0 = x0; g1 = d1 = x1; }
                  else gelu_and_grad2(x0, x1, g0, g1, d0, d1);
                  x0 = g0;
                  x1 = g1;
                  gq[c] = pack_bf16x2(d0, d1);
                }
                pd[4 * c + j] = pack_bf16x2(x0, x1);
              }
              gaux[j] = make_uint4(gq[0], gq[1], gq[2], gq[3]);
            }
            // [32 tokens][32 features], 64-byte rows, 64B swizzle, double-buffered; one stmatrix per c
            if S24_EXP(256) continue;
            uint8_t* zb = stg + sbuf * 2048;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            const uint32_t zb_a = smem_u32(zb);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int tok = 8 * c + mi;
              stmatrix_x4_trans(zb_a + tok * 64 + ((mj ^ ((tok >> 1) & 3)) << 4), pd[4 * c], pd[4 * c + 1],
                                pd[4 * c + 2], pd[4 * c + 3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (kEpi == kEpiStore && ep.accumulate) tma_reduce_add_2d(&tmD, zb, m_w, n0);
              else tma_store_2d(&tmD, zb, m_w, n0);
              bulk_commit();
            }
            sbuf ^= 1;
            if (kEpi == kEpiGeluGrad && !S24_EXP(128)) {
              // GELU'(z) -> AUX units (rows m_w + 8 j + t4, this chunk).  Issued after the proxy
              // fence: the fence (MEMBAR + FENCE.VIEW.ASYNC) waits for every outstanding global
              // access of the thread, so stores issued before it stalled each chunk ~1 round trip
#pragma unroll
              for (int j = 0; j < 4; ++j)
                aux_frag(ep.aux, (m_w >> 4) + (j >> 1), shp.n, n0)[32 * (j & 1) + lane] = gaux[j];
            }
          }
          // next-but-one chunk's AUX inputs, likewise issued after this chunk's fence
          if constexpr (kPre) prefetch(cc + 2);
        }
        if constexpr (kEpi == kEpiDAct || kEpi == kEpiDGated) {
          // reduce the partials of the 4 threads sharing a row (lanes 4 t4 .. 4 t4 + 3)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            bs1[j] += __shfl_xor_sync(0xffffffffu, bs1[j], 1);
            bs1[j] += __shfl_xor_sync(0xffffffffu, bs1[j], 2);
            if constexpr (kEpi == kEpiDGated) {
              bs2[j] += __shfl_xor_sync(0xffffffffu, bs2[j], 1);
              bs2[j] += __shfl_xor_sync(0xffffffffu, bs2[j], 2);
            }
          }
          if (ep.dbias != nullptr && (lane & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              atomicAdd(ep.dbias + m_w + 8 * j + t4, bs1[j]);  // [b; c] order for gated: u half at j
              if constexpr (kEpi == kEpiDGated) atomicAdd(ep.dbias + ep.gate_ff + m_w + 8 * j + t4, bs2[j]);
            }
          }
        }
        }  // slab
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCG == 2) mbar_arrive_cluster(&tempty_bar[acc], crank & ~1u);  // pair leader
          else mbar_arrive(&tempty_bar[acc]);
        }
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (lane == 0) bulk_wait0();
    } else {
      // ============ row epilogue (8 warps: lane quarter q, column half h) ============
      // masked-decay dW (fp32), feature-major plain store, and the API's z / GELU(z) pair:
      // tcgen05.ld 32x32b (thread = row, 32 consecutive columns) -> registers -> swizzled smem
      // staging -> TMA store (full-line writes; staging recycled once the bulk store read it).
      const int q = warp & 3, h = (warp - 4) >> 2;
      uint8_t* stg = smem + C::EPI_OFF + (warp - 4) * 4096;
      int acc = 0, sbuf = 0;
      uint32_t acc_phase = 0;
      WorkIter wk(shp.streamk, num_work, num_kb, cluster_id, num_clusters);
      int tile, kb0, kb1;
      while (wk.next(num_work, num_kb, tile, kb0, kb1)) {
        int mb, nb;
        coords(tile, mb, nb);
        const bool first_chunk = kb0 == 0;                  // adds the decay exactly once
        // stream-K / split-K piece, or a launch that accumulates into D (fp32 mode): add-reduce
        const bool partial = kb0 != 0 || kb1 != num_kb || ep.accumulate;
        const int n_base = nb * kBN;
        // ordered split-K: this unit's reduce-adds start after split s - 1 of the tile completed
        constexpr unsigned int kStorers = 8 * kCG;
        // (stream-K runs are ordered only when none is empty: T >= clusters)
        unsigned int* sctr = (kEpi == kEpiDw && (shp.streamk >= 3 || (shp.streamk == 1 && wk.total >= wk.ncl)) &&
                              shp.ws != nullptr && tile < kSplitTiles)
                                 ? shp.ws + kWsSplit + tile : nullptr;
        const int sidx = wk.last_split;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        if (sctr != nullptr && sidx > 0) {
          if (lane == 0) {
            const unsigned int target = kStorers * static_cast<unsigned int>(sidx);
            const long long t0 = clock64();
            while (ld_acquire_gpu(sctr) < target) {
              if (clock64() - t0 >= 2000000) {  // order (determinism) dropped, sum still correct
                atomicAdd(shp.ws + kWsTimeouts, 1u);
                break;
              }
              __nanosleep(64);
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          __syncwarp();
        }
#pragma unroll 1
        for (int slab = 0; slab < kSlabs; ++slab) {
        const int m_w = mb * C::TILE_M + 128 * kCG * slab + 128 * rank + 32 * q;  // first row of this warp
        const int m = m_w + lane;
        float bias_v = 0.0f;
        if constexpr (kEpi == kEpiStore || kEpi == kEpiGeluAux) {
          if (ep.bias != nullptr) bias_v = bf16_to_f32(ep.bias[m]);
        }
        // the decay's W row and mask indices are prefetched one chunk ahead so their
        // latency hides behind the TMEM load and the math of the current chunk
        constexpr bool kPre = kEpi == kEpiDw;
        const int w_row = (kEpi == kEpiDw && ep.gate_ff > 0) ? gate_row_dev(m, ep.gate_ff) : m;
        uint4 pre[8];
        uint2 pre_idx = make_uint2(0, 0);
        const bool decay = kEpi == kEpiDw && ep.idx != nullptr && first_chunk;
        auto prefetch = [&](int cc) {
          const int n0p = n_base + 32 * cc;
          if (cc >= kBN / 32 || n0p >= shp.n || !decay) return;
          pre_idx = __ldg(reinterpret_cast<const uint2*>(ep.idx + static_cast<int64_t>(m >> 2) * (shp.n >> 2) +
                                                         (n0p >> 2)));
          if (ep.w_dtype == S24_BF16) {
            const uint4* wp = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(ep.w) +
                                                             static_cast<int64_t>(w_row) * shp.n + n0p);
#pragma unroll
            for (int u = 0; u < 4; ++u) pre[u] = __ldg(wp + u);
          } else {
            const uint4* wp = reinterpret_cast<const uint4*>(static_cast<const float*>(ep.w) +
                                                             static_cast<int64_t>(w_row) * shp.n + n0p);
#pragma unroll
            for (int u = 0; u < 8; ++u) pre[u] = __ldg(wp + u);
          }
        };
        if (kPre && !S24_EXP(32)) prefetch(h);
#pragma unroll 1
        for (int cc = h; cc < kBN / 32; cc += 2) {
          uint4 cur[8];
          uint2 cur_idx = pre_idx;
#pragma unroll
          for (int u = 0; u < 8; ++u) cur[u] = pre[u];
          if (kPre && !S24_EXP(32)) prefetch(cc + 2);
          uint32_t r[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * C::ACC_COLS + slab * kBN + 32 * cc, r);
          tmem_ld_wait();
          const int n0 = n_base + 32 * cc;
          if (n0 >= shp.n) continue;
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if constexpr (kEpi == kEpiDw) {
            if (decay) {  // the decay term lam (1 - M) W is added by one K chunk only
              const uint32_t iw[2] = {cur_idx.x, cur_idx.y};
              float wv[32];
              if (ep.w_dtype == S24_BF16) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const uint32_t xs[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    wv[8 * u + 2 * t] = __uint_as_float(xs[t] << 16);
                    wv[8 * u + 2 * t + 1] = __uint_as_float(xs[t] & 0xFFFF0000u);
                  }
                }
              } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  wv[4 * u] = __uint_as_float(cur[u].x);
                  wv[4 * u + 1] = __uint_as_float(cur[u].y);
                  wv[4 * u + 2] = __uint_as_float(cur[u].z);
                  wv[4 * u + 3] = __uint_as_float(cur[u].w);
                }
              }
#pragma unroll
              for (int blk = 0; blk < 8; ++blk) {
                const uint32_t pidx = (iw[blk >> 2] >> (8 * (blk & 3))) & 0xFF;
                const uint32_t rowmask = (c_gemm_pat_bits[min(pidx, 89u)] >> (4 * (m & 3))) & 0xF;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                  if (!((rowmask >> c) & 1)) v[4 * blk + c] += ep.lam * wv[4 * blk + c];
              }
            }
            // fp32 32x32 tile, 128B swizzle: 16-byte chunk c of row `lane` -> chunk c ^ (lane & 7)
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              // two 16-row boxes: the gated first weight's rows go back to [u; v] order
              const int y0 = ep.gate_ff > 0 ? gate_row_dev(m_w, ep.gate_ff) : m_w;
              const int y1 = ep.gate_ff > 0 ? gate_row_dev(m_w + 16, ep.gate_ff) : m_w + 16;
              if (partial) {
                tma_reduce_add_2d(&tmD, stg, n0, y0);
                tma_reduce_add_2d(&tmD, stg + 2048, n0, y1);
              } else {
                tma_store_2d(&tmD, stg, n0, y0);
                tma_store_2d(&tmD, stg + 2048, n0, y1);
              }
              bulk_commit();
            }
          } else {
            constexpr bool kTwo = kEpi == kEpiGeluAux;  // z and GELU(z), both in D's layout
            float v2[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += bias_v;
            if constexpr (kTwo) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v2[i] = gelu_fast(v[i]);
            }
            uint8_t* zb = stg + (kTwo ? 0 : sbuf * 2048);
            if (lane == 0) {
              if constexpr (kTwo) bulk_wait_read0();
              else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            __syncwarp();
            // stage a 32 x 32 bf16 tile: feature-major -> 64B-swizzled rows of this lane;
            // token-major (kOutT) -> transposed, row n holds the 32 features of this warp
            auto stage = [&](uint8_t* buf, const float(&x)[32], bool transposed) {
              if (transposed) {
                uint16_t* b16 = reinterpret_cast<uint16_t*>(buf);
#pragma unroll
                for (int i = 0; i < 32; ++i) b16[i * 32 + lane] = f32_to_bf16(x[i]);
              } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                  *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) =
                      make_uint4(pack_bf16x2(x[8 * c], x[8 * c + 1]), pack_bf16x2(x[8 * c + 2], x[8 * c + 3]),
                                 pack_bf16x2(x[8 * c + 4], x[8 * c + 5]), pack_bf16x2(x[8 * c + 6], x[8 * c + 7]));
              }
            };
            stage(zb, v, kOutT);
            if constexpr (kTwo) stage(stg + 2048, v2, kOutT);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmD, zb, kOutT ? m_w : n0, kOutT ? n0 : m_w);
              if constexpr (kTwo) tma_store_2d(&tmX, stg + 2048, kOutT ? m_w : n0, kOutT ? n0 : m_w);
              bulk_commit();
            }
            sbuf ^= 1;
          }
        }
        }  // slab
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCG == 2) mbar_arrive_cluster(&tempty_bar[acc], crank & ~1u);  // pair leader
          else mbar_arrive(&tempty_bar[acc]);
        }
        if (sctr != nullptr && lane == 0) {
          // this storer's reduce-adds of split s are complete -> release split s + 1
          bulk_wait0();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          const unsigned int old = atomicAdd(sctr, 1u);
          if (old == kStorers * static_cast<unsigned int>(wk.last_nsplit) - 1u) atomicExch(sctr, 0u);
        }
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (lane == 0) bulk_wait0();
    }
  }

  tc_fence_before();
  if constexpr (kCG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_cg<kCG>(tmem_base, C::TMEM_COLS);
  if (shp.ws != nullptr && shp.wave_sync && threadIdx.x == 0) {
    // the last CTA out resets the wave counter for the next launch on this stream
    if (atomicAdd(shp.ws + kWsExit, 1u) == gridDim.x - 1) {
      atomicExch(shp.ws + kWsWave, 0u);
      atomicExch(shp.ws + kWsExit, 0u);
    }
  }
}

// ---------------------------------------------------------------------------
// host helpers

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

enum MapKind { kMapBf16Sw128 = 0, kMapBf16Sw64 = 1, kMapF32Sw128 = 2, kMapU64 = 3, kMapBf16Plain = 4, kMapBf16Sw32 = 5 };

// 2-D tensor map: inner (contiguous) extent, outer extent, row pitch in elements.
static int make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t pitch_elems,
                    uint32_t box_inner, uint32_t box_outer, MapKind kind = kMapBf16Sw128) {
  EncodeTiledFn enc = get_encode_fn();
  S24_REQUIRE(enc != nullptr, S24_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int esz = kind == kMapU64 ? 8 : kind == kMapF32Sw128 ? 4 : 2;
  S24_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (pitch_elems * esz) % 16 == 0, S24_ERR_UNSUPPORTED,
              "TMA operands need 16-byte aligned base and row pitch");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_elems * esz)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = kind == kMapU64 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                                 : kind == kMapF32Sw128 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                        : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUtensorMapSwizzle sw = (kind == kMapU64 || kind == kMapBf16Plain) ? CU_TENSOR_MAP_SWIZZLE_NONE
                                : kind == kMapBf16Sw64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : kind == kMapBf16Sw32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  S24_REQUIRE(r == CUDA_SUCCESS, S24_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return S24_OK;
}

// 4-D map of a gated dense weight [u; v] (2 ff rows of `inner` elements, row pitch `pitch`) read
// in the u/v 16-row interleave of the fused gated epilogues: dims (inner, 16 rows, 2 halves at
// ff rows apart, ff / 16 row groups), box (box_inner, 16, 2, box_groups) -> smem row
// 32 g + 16 h + r = interleaved row p of gate_row_dev.  128-byte swizzle.
static int make_map_gate(CUtensorMap* map, const void* ptr, int64_t inner, int64_t ff, int64_t pitch_elems,
                         uint32_t box_inner, uint32_t box_groups) {
  EncodeTiledFn enc = get_encode_fn();
  S24_REQUIRE(enc != nullptr, S24_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  S24_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (pitch_elems * 2) % 16 == 0 && ff % 16 == 0,
              S24_ERR_UNSUPPORTED, "TMA operands need 16-byte aligned base and row pitch");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), 16, 2, static_cast<cuuint64_t>(ff / 16)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(pitch_elems * 2), static_cast<cuuint64_t>(ff * pitch_elems * 2),
                           static_cast<cuuint64_t>(16 * pitch_elems * 2)};
  cuuint32_t box[4] = {box_inner, 16, 2, box_groups};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  S24_REQUIRE(r == CUDA_SUCCESS, S24_ERR_CUDA, "cuTensorMapEncodeTiled (gate) failed (%d)", static_cast<int>(r));
  return S24_OK;
}

// SMs left free by the persistent GEMMs (the `reserved_sms` argument of every GEMM entry point):
// a data-parallel step reserves a few while its gradient all-reduce runs so the collective's
// kernel is co-resident with the dX GEMM instead of queueing behind it.

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Raster group: the M tiles whose A panels (all of K) stay L2-resident while the
// group sweeps every N tile, so the B operand streams from HBM num_m / group times.
// Sparse GEMMs (A = compressed weight, 1.125 B per logical K per row incl. metadata)
// take as many M tiles as fit a ~48 MB L2 budget; dense dW panels (K = tokens) are
// far larger than L2, so they keep the wave-square default of 8.
// Stream-K for a weight-gradient GEMM whose tiles do not fill one wave (C2 dW: 64 tiles on 74
// CTA pairs, 86 % fill); S24_STREAMK=1 turns it on, off by default.  Plain stream-K (runs
// processed in linear order) put the clusters at different K offsets of the same tiles, so they
// stopped sharing operand panels in L2: on B200 it quadrupled the HBM reads of the C2 dW GEMMs
// (176 -> 748 MB) and made them 20 % slower.  The K-aligned order (WorkIter mode 1: every run
// starts with the segment at k-block 0 of its last tile) keeps all clusters within
// (1 - tiles / clusters) of a tile's K range of each other (C2: 35 k-blocks, ~23 MB of panels),
// and the partial tiles reduce in K order through the workspace's split counters (deterministic).  Measured on B200
// at C2: HBM reads 203 MB (vs 176 MB one-tile-per-pair), kernel 98.7 vs 103.0 us under ncu --
// but only 4 % of the 13.5 % the fill promises, and with the zeroing memset of the fp32 output
// the dW step inside full training steps measured 7 % slower, so the automatic choice stays off.
static int use_streamk(int tiles, int clusters, int num_kb, bool auto_ok = false, double out_bytes = 0.0) {
#ifndef S24_EXPERIMENTS
  (void)tiles, (void)clusters, (void)num_kb, (void)auto_ok, (void)out_bytes;
  return 0;  // measured slower (see above): experiment builds only
#endif
  static const int env = getenv("S24_STREAMK") ? atoi(getenv("S24_STREAMK")) : -1;
  if (env >= 0) return env == 1 ? 1 : 0;
  static const bool auto_env = getenv("S24_STREAMK_AUTO") != nullptr;  // experiment: the rule below
  if (!auto_env || !auto_ok || clusters <= 0 || tiles > kSplitTiles || out_bytes > 32.0 * 1024 * 1024) return 0;
  if (static_cast<double>(tiles) > 0.9 * clusters) return 0;
  if (static_cast<int64_t>(tiles) * num_kb < 32LL * clusters) return 0;
  return 1;
}

// Lockstep split-K for the weight-gradient GEMMs (WorkIter mode S >= 2): a tile count that does
// not fill the last wave leaves CTA pairs idle (C5 dW: 100 tiles on 74 pairs = 2 tile-times for
// 1.35 of work).  Cutting K into S equal ranges makes T S units (C5, S = 2: 1.5 tile-times,
// measured 0.221 -> 0.182 ms per launch).  Unlike stream-K every wave stays at one K offset
// (panels shared in L2).  Partial tiles TMA-add-reduce into the zeroed output: with two addends
// (a + b = b + a) the result is order-independent, and for S >= 3 the splits of a tile reduce in
// split order (the workspace's split counters), so every split stays deterministic.  The automatic choice stops at
// S = 2: S = 8 would fill C2's 64-tile dW waves (0.875 tile-times) but measured 25 % slower on
// B200 (8 reduce passes of the fp32 tile through L2 per output), and C5 got slower too.  A split
// must save >= 3 %, each unit keeps K >= 64 * kb_min, and the fp32 output must fit well inside L2
// (<= 32 MB), otherwise every partial tile round-trips through HBM (C3 dW_in: 360 MB per pass).
// S24_SPLITK=0 off, =N forces N (up to 8).
static int use_splitk(int tiles, int clusters, int num_kb, int kb_min, double out_bytes) {
  static const int env = getenv("S24_SPLITK") ? atoi(getenv("S24_SPLITK")) : -1;
  if (env == 0 || env == 1) return 0;
  if (env >= 2) return num_kb >= env && env <= (tiles <= kSplitTiles ? 8 : 2) ? env : (num_kb >= 2 ? 2 : 0);
  const int smax = 2;
  // the partial tiles of different waves meet in L2 only if the fp32 output stays resident
  if (clusters <= 0 || out_bytes > 32.0 * 1024 * 1024) return 0;
  const double t1 = static_cast<double>((tiles + clusters - 1) / clusters);
  int best = 1;
  double bt = t1;
  for (int sp = 2; sp <= smax; ++sp) {
    if (num_kb < sp * kb_min) break;
    const double t = static_cast<double>((static_cast<int64_t>(tiles) * sp + clusters - 1) / clusters) / sp;
    if (t < bt - 1e-9) {
      bt = t;
      best = sp;
    }
  }
  return bt <= 0.97 * t1 ? best : 0;
}

static int dw_clusters(int reserved) {
  const int sms = reserved > 0 ? std::max(2, num_sms() - reserved) : num_sms();
  return sms / 2;
}

// Wave-synchronised schedule (workspace wave counter): on for the dW GEMMs (panels of K = tokens,
// far larger than L2) and for the forward / dX GEMMs with K >= 8192, whose tiles run long enough
// for the CTAs to drift apart (measured on B200, alternating A/B: C4 step -1.7 %, every sparse
// GEMM faster; C3's K = 4096 fused-epilogue GEMMs +2 % with it, its K = 11008 / 22016 ones
// unchanged).  S24_WAVESYNC=0/1 turns it off / on for every GEMM.
static int wave_on(bool dflt) {
  static const int env = getenv("S24_WAVESYNC") ? atoi(getenv("S24_WAVESYNC")) : -1;
  return (env < 0 ? dflt : env != 0) ? 1 : 0;
}

// Two-slab dense dW tiles (512 x 256 per CTA pair, one 512-column accumulator): -25 % operand
// bytes per MAC, which buys clock under the power cap (measured on B200: C3 dW2 1.98 -> 1.89 ms,
// C4 dW 12.98 -> 12.62 ms at +7..10 % SM clock) but halves the tile count and exposes the
// epilogue, so it is used only when the wave fill does not get worse (C3 dW_in 97.9 -> 93 %:
// 3.87 -> 3.95 ms).  S24_DW_SLABS=0/1 overrides.
static bool use_dw_slabs(int64_t m, int64_t n, int64_t k) {
  static const int env = getenv("S24_DW_SLABS") ? atoi(getenv("S24_DW_SLABS")) : -1;
  if (env >= 0) return env == 1;
  const int64_t clusters = num_sms() / 2;
  const int64_t t1 = (m / 256) * (n / 256), t2 = (m / 512) * (n / 256);
  auto fill = [&](int64_t t) { return static_cast<double>(t) / (((t + clusters - 1) / clusters) * clusters); };
  return k >= 8192 && t2 >= 2 * clusters && fill(t2) >= fill(t1) - 0.01;
}

// Two-slab tiles for the 2:4 weight-gradient GEMM (MVUE operand, K = tokens) with a K-major B:
// when K is long enough for the un-overlapped epilogue not to matter and the wave fill holds.
// S24_SDW_SLABS=0/1 overrides.
static bool use_sdw_slabs(int64_t m, int64_t n, int64_t k) {
  static const int env = getenv("S24_SDW_SLABS") ? atoi(getenv("S24_SDW_SLABS")) : -1;
  if (env >= 0) return env == 1;
  const int64_t clusters = num_sms() / 2;
  const int64_t t2 = (m / 512) * ((n + 223) / 224);
  return k >= 4096 && t2 >= 2 * clusters;
}

// Two-slab sparse tiles (Cfg kSlabs) for plain-store GEMMs whose main loop per tile dwarfs the
// then un-overlapped epilogue: K >= 4096 (measured on B200: C2's K = 4096 plain GEMMs -7 %,
// C3's K = 11008 / 22016 ones -10..12 %), as long as halving the tile count does not leave a
// wave worse filled.  S24_SLABS=0 off, =1 whenever the shape allows (m % 512 == 0).
static bool use_slabs(int64_t m, int64_t n, int64_t k) {
  static const int env = getenv("S24_SLABS") ? atoi(getenv("S24_SLABS")) : -1;
  if (m % 256 != 0 || env == 0) return false;
  if (env == 1) return true;
  const int64_t clusters = num_sms() / 2, nt = (n + 223) / 224;
  auto fill = [&](int64_t t) { return static_cast<double>(t) / (((t + clusters - 1) / clusters) * clusters); };
  // work in 256-row units: a ragged last slab tile costs a full tile
  const double t2 = static_cast<double>((m + 511) / 512 * nt), t1 = static_cast<double>(m / 256 * nt);
  return k >= 4096 && fill(static_cast<int64_t>(t2)) * t1 / (2.0 * t2) >= fill(static_cast<int64_t>(t1)) - 0.02;
}

// B multicast across two CTA pairs (gemm_kernel kMC = 2): halves the L2 reads of the token
// operand.  S24_MC=0/1 overrides; needs an even number of 256-row pair tiles.
[[maybe_unused]] static bool use_mc(int64_t m) {
  static const int env = getenv("S24_MC") ? atoi(getenv("S24_MC")) : -1;
  if (m % 512 != 0 || env == 0) return false;
  return env == 1;
}

// Two-slab tiles for the fused training epilogues as well, where K is long enough to carry the
// un-overlapped epilogue (measured on B200: C3's SwiGLU GEMM1, K = 4096, -4 %; C2's K = 1024
// GELU / dGELU GEMMs +17..35 %, so not there).  S24_SLABS_EPI=0/1 overrides.
static bool use_slabs_epi(int64_t m, int64_t n, int64_t k) {
  static const int env = getenv("S24_SLABS_EPI") ? atoi(getenv("S24_SLABS_EPI")) : -1;
  if (m % 256 != 0 || env == 0) return false;
  if (env == 1) return true;
  const int64_t clusters = num_sms() / 2, nt = (n + 223) / 224;
  auto fill = [&](int64_t t) { return static_cast<double>(t) / (((t + clusters - 1) / clusters) * clusters); };
  const double t2 = static_cast<double>((m + 511) / 512 * nt), t1 = static_cast<double>(m / 256 * nt);
  return k >= 4096 && fill(static_cast<int64_t>(t2)) * t1 / (2.0 * t2) >= fill(static_cast<int64_t>(t1)) - 0.02;
}

static int exp_flags() {
#ifdef S24_EXPERIMENTS
  static const int v = getenv("S24_EXP") ? atoi(getenv("S24_EXP")) : 0;
  return v;
#else
  return 0;
#endif
}

static int pick_group_m(int num_m, double a_bytes_per_mtile) {
  static const int env = getenv("S24_GROUP_M") ? atoi(getenv("S24_GROUP_M")) : 0;
  int g = env > 0 ? env : 12;  // 12 vs 8: -0.2..0.4 % C3 / C4 step, alternating A/B on one box
  (void)a_bytes_per_mtile;
  if (g < 1) g = 1;
  return g < num_m ? g : num_m;
}

template <bool kSparse, bool kAMN, bool kBMN, int kBN, int kStages, int kCG, int kEpi, bool kOutT = false,
          int kAcc = 2, int kSlabs = 1, int kMC = 1>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& me, const CUtensorMap& md,
                       const CUtensorMap& mx, const CUtensorMap& my, const GemmShape& shp, const EpiParams& ep,
                       int reserved, cudaStream_t st) {
  using C = Cfg<kSparse, kAMN, kBMN, kBN, kStages, kCG, kAcc, kSlabs>;
  auto kern = gemm_kernel<kSparse, kAMN, kBMN, kBN, kStages, kCG, kEpi, kOutT, kAcc, kSlabs, kMC>;
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    S24_REQUIRE(e == cudaSuccess, S24_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_done = true;
  }
  constexpr int kCS = kCG * kMC;  // CTAs per cluster
  const int tiles = ((shp.m + C::TILE_M - 1) / C::TILE_M / kMC) * ((shp.n + kBN - 1) / kBN);
  // persistent grid: as many clusters as are co-resident (a 4-CTA cluster needs 4 free SMs
  // in one GPC, so fewer than 148 / 4 may fit), never more than there are work tiles
  static int max_clusters = 0;  // per template instance
  if (max_clusters == 0) {
    max_clusters = num_sms() / kCS;
    if (kCS > 2) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(kCS * max_clusters);
      q.blockDim = dim3(kGemmThreads);
      q.dynamicSmemBytes = C::SMEM_BYTES;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = kCS;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n > 0 && n < max_clusters) max_clusters = n;
      (void)cudaGetLastError();
    }
  }
  int cap = max_clusters;
  if (reserved > 0) cap = std::max(1, std::min(cap, (num_sms() - reserved) / kCS));
  const int units = shp.streamk >= 2 ? tiles * shp.streamk : tiles;
  const int clusters = (shp.streamk == 1 || units > cap) ? cap : units;
  if (clusters <= 0) return S24_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * kCS);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, me, md, mx, my, shp, ep);
  S24_REQUIRE(e == cudaSuccess, S24_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(e));
  return s24_check_launch("gemm");
}

}  // namespace s24

using namespace s24;

static int cg_override() {
  static const int v = getenv("S24_GEMM_CG") ? atoi(getenv("S24_GEMM_CG")) : 0;
  return v;
}

extern "C" int64_t s24_gemm_workspace_bytes(void) { return S24_GEMM_WORKSPACE_BYTES; }


extern "C" int s24_spmm(const uint16_t* a_vals, const uint8_t* a_e, int64_t m, int64_t k, const uint16_t* b,
                        int b_mn, int64_t ldb, int64_t n, uint16_t* d, int64_t ldd, const uint16_t* bias,
                        int epilogue, uint16_t* aux, int64_t ldaux, uint16_t* aux2, float* dbias, int d_t,
                        int64_t gate_ff, void* workspace, int reserved, void* stream) {
  S24_REQUIRE(a_vals && a_e && b && d, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(reserved >= 0 && (reinterpret_cast<uintptr_t>(workspace) & 3) == 0, S24_ERR_ARG,
              "reserved_sms must be >= 0 and the workspace 4-byte aligned");
  S24_REQUIRE(m % 128 == 0 && k % 128 == 0 && n % 32 == 0 && m > 0 && k > 0 && n > 0, S24_ERR_SHAPE,
              "sparse GEMM needs m %% 128 == 0, k %% 128 == 0, n %% 32 == 0 (got m=%lld k=%lld n=%lld)",
              (long long)m, (long long)k, (long long)n);
  S24_REQUIRE(epilogue >= S24_EPI_STORE && epilogue <= S24_EPI_STORE_ADD, S24_ERR_ARG, "bad epilogue");
  const bool accumulate = epilogue == S24_EPI_STORE_ADD;
  S24_REQUIRE(!accumulate || d_t == 1, S24_ERR_ARG, "S24_EPI_STORE_ADD accumulates into a token-major output (d_t = 1)");
  if (accumulate) epilogue = S24_EPI_STORE;
  const bool gated_fwd = epilogue == S24_EPI_GEGLU_GRAD || epilogue == S24_EPI_SWIGLU_GRAD;
  const bool gated_bwd = epilogue == S24_EPI_DGATED;
  // logical width of the stored output: GEMM1 gated stores d_ff = m/2 gate features, GEMM3 gated
  // stores the interleaved 2m columns of dZ
  const int64_t d_cols = gated_fwd ? m / 2 : gated_bwd ? 2 * m : m;
  S24_REQUIRE(ldd >= (d_t ? d_cols : n) && ldd % 8 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0,
              S24_ERR_UNSUPPORTED, "output rows must be 16-byte aligned");
  const bool training = gated_fwd || gated_bwd || epilogue == S24_EPI_GELU_GRAD || epilogue == S24_EPI_DGELU;
  S24_REQUIRE(d_t == 1 || !training, S24_ERR_ARG, "training epilogues store token-major outputs (d_t = 1)");
  if (gated_fwd || gated_bwd) {
    S24_REQUIRE(gate_ff == (gated_fwd ? m / 2 : m) && gate_ff % 16 == 0, S24_ERR_SHAPE,
                "gated epilogue: gate_ff must be d_ff (%lld) and a multiple of 16", (long long)gate_ff);
    S24_REQUIRE(aux2 != nullptr && (reinterpret_cast<uintptr_t>(aux2) & 15) == 0, S24_ERR_ARG,
                "gated epilogues need a 16-byte aligned aux2 tensor");
  }
  if (epilogue == S24_EPI_GELU_AUX)
    S24_REQUIRE(aux != nullptr && ldaux >= (d_t ? m : n) && ldaux % 8 == 0 && (reinterpret_cast<uintptr_t>(aux) & 15) == 0,
                S24_ERR_ARG, "this epilogue needs a 16-byte aligned aux tensor");
  else if (epilogue != S24_EPI_STORE)  // blocked AUX layout (ldaux unused)
    S24_REQUIRE(aux != nullptr && (reinterpret_cast<uintptr_t>(aux) & 15) == 0, S24_ERR_ARG,
                "this epilogue needs a 16-byte aligned (blocked) aux tensor");
  S24_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX, S24_ERR_SHAPE, "dims exceed int32");
  const bool pair = (m % 256 == 0) && cg_override() != 1;
  constexpr int BN1 = 128, BN2 = 224;
  CUtensorMap ma, mb, me;
  if (int rc = make_map(&ma, a_vals, k / 2, m, k / 2, 64, 128)) return rc;
  if (int rc = make_map(&me, a_e, 256, (m / 128) * (k / 128), 256, 256, 1, kMapU64)) return rc;
  CUtensorMap md, mx, my;
  if (gated_fwd) {
    // A: [n tokens][d_ff] boxes of 16 features x 32 tokens (32B-swizzled stmatrix staging);
    // AUX, AUX2 go straight to global in the fragment layout (aux_frag)
    if (int rc = make_map(&md, d, m / 2, n, ldd, 16, 32, kMapBf16Sw32)) return rc;
    mx = my = md;
  } else if (gated_bwd) {
    // dZ interleaved, token-major: boxes of 32 columns x 32 tokens, 64B-swizzled staging
    if (int rc = make_map(&md, d, 2 * m, n, ldd, 32, 32, kMapBf16Sw64)) return rc;
    mx = my = md;
  } else {
    // D[m, n] feature-major (64B-swizzled staging) or D^T[n, m] token-major (d_t: stmatrix.trans into
    // 64B-swizzled staging; the API's z / GELU(z) epilogue: transposed two-byte staging, no swizzle)
    if (d_t) {
      if (int rc = make_map(&md, d, m, n, ldd, 32, 32, epilogue == S24_EPI_GELU_AUX ? kMapBf16Plain : kMapBf16Sw64))
        return rc;
    } else {
      if (int rc = make_map(&md, d, n, m, ldd, 32, 32, kMapBf16Sw64)) return rc;
    }
    if (epilogue == S24_EPI_GELU_AUX) {
      if (d_t) {
        if (int rc = make_map(&mx, aux, m, n, ldaux, 32, 32, kMapBf16Plain)) return rc;
      } else {
        if (int rc = make_map(&mx, aux, n, m, ldaux, 32, 32, kMapBf16Sw64)) return rc;
      }
    } else {
      mx = md;
    }
    my = md;
  }
  const int bn_cta = pair ? BN2 / 2 : BN1;
  if (b_mn) {
    S24_REQUIRE(ldb >= n, S24_ERR_SHAPE, "ldb < n");
    if (int rc = make_map(&mb, b, n, k, ldb, 64, 128)) return rc;
  } else {
    S24_REQUIRE(ldb >= k, S24_ERR_SHAPE, "ldb < k");
    if (int rc = make_map(&mb, b, k, n, ldb, 64, bn_cta)) return rc;
  }
  const int tile_m = pair ? 256 : 128;
  GemmShape shp{static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 0,
                pick_group_m(static_cast<int>(m / tile_m), 1.125 * tile_m * static_cast<double>(k)),
                static_cast<unsigned int*>(workspace), wave_on(k >= 8192), exp_flags()};
  EpiParams ep{d,       ldd,
               bias,    aux,
               ldaux,   dbias,
               aux2,    epilogue == S24_EPI_SWIGLU_GRAD ? S24_ACT_SWIGLU : S24_ACT_GEGLU,
               gate_ff, nullptr,
               0,       nullptr,
               0.0f,    accumulate ? 1 : 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define S24_SP(BMN, BNV, CG, EPI)                                                                          \
  if (d_t)                                                                                                  \
    return launch_gemm<true, false, BMN, BNV, stages_for<Cfg<true, false, BMN, BNV, 1, CG>::STAGE_BYTES>(), CG, \
                       EPI, true>(ma, mb, me, md, mx, my, shp, ep, reserved, st);                                     \
  return launch_gemm<true, false, BMN, BNV, stages_for<Cfg<true, false, BMN, BNV, 1, CG>::STAGE_BYTES>(), CG,   \
                     EPI, false>(ma, mb, me, md, mx, my, shp, ep, reserved, st)
#define S24_SPT(BMN, BNV, CG, EPI)                                                                           \
  return launch_gemm<true, false, BMN, BNV, stages_for<Cfg<true, false, BMN, BNV, 1, CG>::STAGE_BYTES>(), CG, EPI, \
                     true>(ma, mb, me, md, mx, my, shp, ep, reserved, st)
#define S24_SP_EPI(BMN, BNV, CG)                                              \
  switch (epilogue) {                                                           \
    case S24_EPI_GELU_AUX: S24_SP(BMN, BNV, CG, kEpiGeluAux);                   \
    case S24_EPI_GELU_GRAD: S24_SPT(BMN, BNV, CG, kEpiGeluGrad);                \
    case S24_EPI_DGELU: S24_SPT(BMN, BNV, CG, kEpiDAct);                        \
    case S24_EPI_GEGLU_GRAD:                                                    \
    case S24_EPI_SWIGLU_GRAD: S24_SPT(BMN, BNV, CG, kEpiGatedGrad);             \
    case S24_EPI_DGATED: S24_SPT(BMN, BNV, CG, kEpiDGated);                     \
    default: S24_SP(BMN, BNV, CG, kEpiStore);                                   \
  }
  const bool slabs = pair && !b_mn && d_t && epilogue == S24_EPI_STORE && use_slabs(m, n, k);
#ifdef S24_EXPERIMENTS
  if (!slabs && pair && !b_mn && d_t && epilogue != S24_EPI_GELU_AUX && use_mc(m)) {
    // 4-CTA clusters, B multicast across the two pairs: B boxes of BN_CTA / 2 rows
    if (int rc = make_map(&mb, b, k, n, ldb, 64, BN2 / 4)) return rc;
#define S24_SPMC(EPI)                                                                                             \
  return launch_gemm<true, false, false, BN2, stages_for<Cfg<true, false, false, BN2, 1, 2>::STAGE_BYTES>(), 2, EPI, \
                     true, 2, 1, 2>(ma, mb, me, md, mx, my, shp, ep, reserved, st)
    switch (epilogue) {
      case S24_EPI_GELU_GRAD: S24_SPMC(kEpiGeluGrad);
      case S24_EPI_DGELU: S24_SPMC(kEpiDAct);
      case S24_EPI_GEGLU_GRAD:
      case S24_EPI_SWIGLU_GRAD: S24_SPMC(kEpiGatedGrad);
      case S24_EPI_DGATED: S24_SPMC(kEpiDGated);
      default: S24_SPMC(kEpiStore);
    }
#undef S24_SPMC
  }
#endif
  if (slabs) {
    // two A slabs per CTA, one accumulator: 512 x 224 pair tiles
    using CS = Cfg<true, false, false, BN2, 1, 2, 1, 2>;
    return launch_gemm<true, false, false, BN2, stages_for<CS::STAGE_BYTES>(), 2, kEpiStore, true, 1, 2>(
        ma, mb, me, md, mx, my, shp, ep, reserved, st);
  }
  if (pair && !b_mn && d_t && epilogue != S24_EPI_STORE && epilogue != S24_EPI_GELU_AUX && use_slabs_epi(m, n, k)) {
    using CS = Cfg<true, false, false, BN2, 1, 2, 1, 2>;
#define S24_SPSL(EPI) \
  return launch_gemm<true, false, false, BN2, stages_for<CS::STAGE_BYTES>(), 2, EPI, true, 1, 2>(ma, mb, me, md, mx, my, shp, ep, reserved, st)
    switch (epilogue) {
      case S24_EPI_GELU_GRAD: S24_SPSL(kEpiGeluGrad);
      case S24_EPI_DGELU: S24_SPSL(kEpiDAct);
      case S24_EPI_GEGLU_GRAD:
      case S24_EPI_SWIGLU_GRAD: S24_SPSL(kEpiGatedGrad);
      default: S24_SPSL(kEpiDGated);
    }
#undef S24_SPSL
  }
  if (pair) {
    if (b_mn) S24_SP_EPI(true, BN2, 2);
    S24_SP_EPI(false, BN2, 2);
  }
  if (b_mn) S24_SP_EPI(true, BN1, 1);
  S24_SP_EPI(false, BN1, 1);
#undef S24_SP_EPI
#undef S24_SPT
#undef S24_SP
}

// Dense counterpart of s24_spmm's token-major training products: the same persistent CTA-pair
// kernel with kind::f16 MMAs on the dense weight and the same fused epilogues (bias, GELU / GELU',
// dGELU + bias gradient, gated forward / backward, add-reduce store).  Serves the dense fine-tune
// phase (gated_ffn.py:286-289 with masks=None, trainer.py:111-114) and the fused dense baseline.
extern "C" int s24_gemm_act(const uint16_t* w, int w_t, int64_t ldw, int64_t w_gate_ff, int64_t m, int64_t k,
                            const uint16_t* b, int64_t ldb, int64_t n, uint16_t* d, int64_t ldd, const uint16_t* bias,
                            int epilogue, uint16_t* aux, uint16_t* aux2, float* dbias, int64_t gate_ff,
                            void* workspace, int reserved, void* stream) {
  S24_REQUIRE(w && b && d, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(reserved >= 0 && (reinterpret_cast<uintptr_t>(workspace) & 3) == 0, S24_ERR_ARG,
              "reserved_sms must be >= 0 and the workspace 4-byte aligned");
  S24_REQUIRE(m % 128 == 0 && k % 64 == 0 && n % 32 == 0 && m > 0 && k > 0 && n > 0, S24_ERR_SHAPE,
              "dense GEMM needs m %% 128 == 0, k %% 64 == 0, n %% 32 == 0 (got m=%lld k=%lld n=%lld)",
              (long long)m, (long long)k, (long long)n);
  S24_REQUIRE(epilogue >= S24_EPI_STORE && epilogue <= S24_EPI_STORE_ADD && epilogue != S24_EPI_GELU_AUX,
              S24_ERR_ARG, "bad epilogue for the dense token-major GEMM");
  S24_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX, S24_ERR_SHAPE, "dims exceed int32");
  const bool accumulate = epilogue == S24_EPI_STORE_ADD;
  if (accumulate) epilogue = S24_EPI_STORE;
  const bool gated_fwd = epilogue == S24_EPI_GEGLU_GRAD || epilogue == S24_EPI_SWIGLU_GRAD;
  const bool gated_bwd = epilogue == S24_EPI_DGATED;
  const int64_t d_cols = gated_fwd ? m / 2 : gated_bwd ? 2 * m : m;
  S24_REQUIRE(ldd >= d_cols && ldd % 8 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0, S24_ERR_UNSUPPORTED,
              "output rows must be 16-byte aligned");
  if (gated_fwd || gated_bwd) {
    S24_REQUIRE(gate_ff == (gated_fwd ? m / 2 : m) && gate_ff % 16 == 0, S24_ERR_SHAPE,
                "gated epilogue: gate_ff must be d_ff (%lld) and a multiple of 16", (long long)gate_ff);
    S24_REQUIRE(aux2 != nullptr && (reinterpret_cast<uintptr_t>(aux2) & 15) == 0, S24_ERR_ARG,
                "gated epilogues need a 16-byte aligned aux2 tensor");
  }
  if (gated_fwd) S24_REQUIRE(w_gate_ff == m / 2 && !w_t, S24_ERR_SHAPE, "gated forward reads the [u; v] weight interleaved");
  if (epilogue != S24_EPI_STORE)
    S24_REQUIRE(aux != nullptr && (reinterpret_cast<uintptr_t>(aux) & 15) == 0, S24_ERR_ARG,
                "this epilogue needs a 16-byte aligned (blocked) aux tensor");
  const int64_t w_rows = w_t ? k : m, w_cols = w_t ? m : k;
  S24_REQUIRE(ldw >= w_cols && ldb >= k, S24_ERR_SHAPE, "ldw / ldb too small");
  if (w_gate_ff > 0)
    S24_REQUIRE(w_rows == 2 * w_gate_ff && w_gate_ff % 16 == 0, S24_ERR_SHAPE,
                "interleaved weight: its [u; v] dimension must be 2 * d_ff with d_ff %% 16 == 0");
  // CTA pairs (M = 256, BN = 224) when m allows, else single CTAs (M = 128, BN = 128)
  const bool pair = m % 256 == 0 && cg_override() != 1;
  constexpr int BN = 224, BN1 = 128;
  CUtensorMap ma, mb, md;
  if (w_gate_ff > 0) {
    if (int rc = make_map_gate(&ma, w, w_cols, w_gate_ff, ldw, 64, w_t ? 2 : 4)) return rc;
  } else if (w_t) {
    if (int rc = make_map(&ma, w, m, k, ldw, 64, 64)) return rc;
  } else {
    if (int rc = make_map(&ma, w, k, m, ldw, 64, 128)) return rc;
  }
  if (int rc = make_map(&mb, b, k, n, ldb, 64, pair ? BN / 2 : BN1)) return rc;
  if (gated_fwd) {
    if (int rc = make_map(&md, d, m / 2, n, ldd, 16, 32, kMapBf16Sw32)) return rc;
  } else if (gated_bwd) {
    if (int rc = make_map(&md, d, 2 * m, n, ldd, 32, 32, kMapBf16Sw64)) return rc;
  } else {
    if (int rc = make_map(&md, d, m, n, ldd, 32, 32, kMapBf16Sw64)) return rc;
  }
  GemmShape shp{static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), 0,
                pick_group_m(static_cast<int>(m / (pair ? 256 : 128)), 0.0), static_cast<unsigned int*>(workspace),
                wave_on(k >= 8192), 0, w_gate_ff > 0 ? 1 : 0};
  EpiParams ep{d,       ldd,   bias,    aux,     0,   dbias, aux2,
               epilogue == S24_EPI_SWIGLU_GRAD ? S24_ACT_SWIGLU : S24_ACT_GEGLU,
               gate_ff, nullptr, 0,     nullptr, 0.0f, accumulate ? 1 : 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define S24_DA(AMN, BNV, CG, EPI)                                                                               \
  return launch_gemm<false, AMN, false, BNV, stages_for<Cfg<false, AMN, false, BNV, 1, CG>::STAGE_BYTES>(), CG, \
                     EPI, true>(ma, mb, mb, md, md, md, shp, ep, reserved, st)
#define S24_DA_EPI(AMN, BNV, CG)                                   \
  switch (epilogue) {                                              \
    case S24_EPI_GELU_GRAD: S24_DA(AMN, BNV, CG, kEpiGeluGrad);    \
    case S24_EPI_DGELU: S24_DA(AMN, BNV, CG, kEpiDAct);            \
    case S24_EPI_GEGLU_GRAD:                                       \
    case S24_EPI_SWIGLU_GRAD: S24_DA(AMN, BNV, CG, kEpiGatedGrad); \
    case S24_EPI_DGATED: S24_DA(AMN, BNV, CG, kEpiDGated);         \
    default: S24_DA(AMN, BNV, CG, kEpiStore);                      \
  }
  if (pair) {
    if (w_t) S24_DA_EPI(true, BN, 2);
    S24_DA_EPI(false, BN, 2);
  }
  if (w_t) S24_DA_EPI(true, BN1, 1);
  S24_DA_EPI(false, BN1, 1);
#undef S24_DA_EPI
#undef S24_DA
}

extern "C" int s24_gemm_dw(const uint16_t* a, int a_mn, int64_t lda, const uint16_t* b, int b_mn, int64_t ldb,
                           int64_t m, int64_t n, int64_t k, float* d, int64_t ldd, const void* w, int w_dtype,
                           const uint8_t* idx, float lambda_w, int64_t gate_ff, int accumulate, void* workspace,
                           int reserved, void* stream) {
  if (gate_ff > 0)
    S24_REQUIRE(m == 2 * gate_ff && gate_ff % 16 == 0, S24_ERR_SHAPE, "gated dW: m must be 2 * d_ff");
  S24_REQUIRE(a && b && d, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(reserved >= 0 && (reinterpret_cast<uintptr_t>(workspace) & 3) == 0, S24_ERR_ARG,
              "reserved_sms must be >= 0 and the workspace 4-byte aligned");
  S24_REQUIRE(m % 128 == 0 && n % 128 == 0 && k % 64 == 0 && m > 0 && n > 0 && k > 0, S24_ERR_SHAPE,
              "dW GEMM needs m %% 128 == 0, n %% 128 == 0, k %% 64 == 0 (got m=%lld n=%lld k=%lld)", (long long)m,
              (long long)n, (long long)k);
  S24_REQUIRE(ldd >= n && ldd % 4 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0, S24_ERR_UNSUPPORTED,
              "dW rows must be 16-byte aligned");
  if (idx != nullptr) {
    S24_REQUIRE(w != nullptr && (w_dtype == S24_BF16 || w_dtype == S24_F32), S24_ERR_UNSUPPORTED,
                "masked decay needs bf16 or fp32 weights");
  }
  S24_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX, S24_ERR_SHAPE, "dims exceed int32");
  const bool wide = n % 256 == 0;
  const bool pair = wide && m % 256 == 0 && cg_override() != 1;
  const int BN = wide ? 256 : 128;
  const int bn_cta = pair ? BN / 2 : BN;
  CUtensorMap ma, mb, me;
  if (a_mn) {
    S24_REQUIRE(lda >= m, S24_ERR_SHAPE, "lda < m");
    if (int rc = make_map(&ma, a, m, k, lda, 64, 64)) return rc;
  } else {
    S24_REQUIRE(lda >= k, S24_ERR_SHAPE, "lda < k");
    if (int rc = make_map(&ma, a, k, m, lda, 64, 128)) return rc;
  }
  if (b_mn) {
    S24_REQUIRE(ldb >= n, S24_ERR_SHAPE, "ldb < n");
    if (int rc = make_map(&mb, b, n, k, ldb, 64, 64)) return rc;
  } else {
    S24_REQUIRE(ldb >= k, S24_ERR_SHAPE, "ldb < k");
    if (int rc = make_map(&mb, b, k, n, ldb, 64, bn_cta)) return rc;
  }
  me = mb;  // unused by the dense kernels
  CUtensorMap md;
  if (int rc = make_map(&md, d, n, m, ldd, 32, 16, kMapF32Sw128)) return rc;  // 16-row store boxes
  const int clusters = num_sms() / (pair ? 2 : 1);
  const int tiles = static_cast<int>((m / (pair ? 256 : 128)) * (n / BN));
  const bool slabs = pair && a_mn && b_mn && m % 512 == 0 && use_dw_slabs(m, n, k);
  int streamk = slabs ? 0 : use_streamk(tiles, pair ? dw_clusters(reserved) : 2 * dw_clusters(reserved), static_cast<int>(k / 64),
                                         true, 4.0 * m * n);
  if (!streamk)
    streamk = use_splitk(slabs ? static_cast<int>((m / 512) * (n / 256)) : tiles,
                         pair ? dw_clusters(reserved) : 2 * dw_clusters(reserved), static_cast<int>(k / 64), 32, 4.0 * m * n);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (streamk && !accumulate) {  // accumulate: the partial tiles add onto D's current values
    cudaError_t e = cudaMemset2DAsync(d, ldd * sizeof(float), 0, n * sizeof(float), m, st);
    S24_REQUIRE(e == cudaSuccess, S24_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  const int tile_m = pair ? 256 : 128;
  static const int env_dw = getenv("S24_GROUP_M_DW") ? atoi(getenv("S24_GROUP_M_DW")) : 8;
  GemmShape shp{static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), streamk,
                static_cast<int>(m / tile_m) < env_dw ? static_cast<int>(m / tile_m) : env_dw,
                static_cast<unsigned int*>(workspace), wave_on(true), exp_flags()};
  EpiParams ep{d, ldd, nullptr, nullptr, 0, nullptr, nullptr, 0, gate_ff, w, w_dtype, idx, lambda_w, accumulate ? 1 : 0};

#define S24_DW(AMN, BMN, BNV, CG)                                                                      \
  return launch_gemm<false, AMN, BMN, BNV, stages_for<Cfg<false, AMN, BMN, BNV, 1, CG>::STAGE_BYTES>(), CG, \
                     kEpiDw>(ma, mb, me, md, md, md, shp, ep, reserved, st)
  if (slabs) {
    using CS = Cfg<false, true, true, 256, 1, 2, 1, 2>;
    return launch_gemm<false, true, true, 256, stages_for<CS::STAGE_BYTES>(), 2, kEpiDw, false, 1, 2>(
        ma, mb, me, md, md, md, shp, ep, reserved, st);
  }
  if (pair) {
    if (a_mn && b_mn) S24_DW(true, true, 256, 2);
    if (a_mn) S24_DW(true, false, 256, 2);
    if (b_mn) S24_DW(false, true, 256, 2);
    S24_DW(false, false, 256, 2);
  }
  if (wide) {
    if (a_mn && b_mn) S24_DW(true, true, 256, 1);
    if (a_mn) S24_DW(true, false, 256, 1);
    if (b_mn) S24_DW(false, true, 256, 1);
    S24_DW(false, false, 256, 1);
  }
  if (a_mn && b_mn) S24_DW(true, true, 128, 1);
  if (a_mn) S24_DW(true, false, 128, 1);
  if (b_mn) S24_DW(false, true, 128, 1);
  S24_DW(false, false, 128, 1);
#undef S24_DW
}

extern "C" int s24_spmm_dw(const uint16_t* a_vals, const uint8_t* a_e, int64_t m, int64_t k, const uint16_t* b,
                           int b_mn, int64_t ldb, int64_t n, float* d, int64_t ldd, const void* w, int w_dtype,
                           const uint8_t* idx, float lambda_w, int64_t gate_ff, int accumulate, void* workspace,
                           int reserved, void* stream) {
  S24_REQUIRE(a_vals && a_e && b && d, S24_ERR_ARG, "NULL operand");
  S24_REQUIRE(reserved >= 0 && (reinterpret_cast<uintptr_t>(workspace) & 3) == 0, S24_ERR_ARG,
              "reserved_sms must be >= 0 and the workspace 4-byte aligned");
  S24_REQUIRE(m % 128 == 0 && k % 128 == 0 && n % 128 == 0 && m > 0 && k > 0 && n > 0, S24_ERR_SHAPE,
              "sparse dW GEMM needs m %% 128 == 0, k %% 128 == 0, n %% 128 == 0 (got m=%lld k=%lld n=%lld)",
              (long long)m, (long long)k, (long long)n);
  S24_REQUIRE(ldd >= n && ldd % 4 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0, S24_ERR_UNSUPPORTED,
              "dW rows must be 16-byte aligned");
  if (idx != nullptr)
    S24_REQUIRE(w != nullptr && (w_dtype == S24_BF16 || w_dtype == S24_F32), S24_ERR_UNSUPPORTED,
                "masked decay needs bf16 or fp32 weights");
  if (gate_ff > 0) S24_REQUIRE(m == 2 * gate_ff && gate_ff % 16 == 0, S24_ERR_SHAPE, "gated dW: m must be 2 * d_ff");
  S24_REQUIRE(m <= INT32_MAX && n <= INT32_MAX && k <= INT32_MAX, S24_ERR_SHAPE, "dims exceed int32");
  const bool pair = m % 256 == 0 && cg_override() != 1;
  const bool wide = n % 256 == 0;
  // two-slab tiles (512 x 224 per CTA pair, one 448-column accumulator + 8 metadata columns) for
  // a K-major (token-contiguous) B: -22 % operand bytes per MAC against 256 x 256 tiles on this
  // L2-bound GEMM; the B operand must be K-major (an MN-major 112-row half needs two 64-wide
  // swizzle boxes, and the 68 KB stage leaves room for only two stages)
  const bool sdw_slabs = pair && !b_mn && m % 512 == 0 && use_sdw_slabs(m, n, k);
  const int bn_cta = sdw_slabs ? 112 : (wide ? 256 : 128) / (pair ? 2 : 1);
  CUtensorMap ma, mb, me, md;
  if (int rc = make_map(&ma, a_vals, k / 2, m, k / 2, 64, 128)) return rc;
  if (int rc = make_map(&me, a_e, 256, (m / 128) * (k / 128), 256, 256, 1, kMapU64)) return rc;
  if (b_mn) {
    S24_REQUIRE(ldb >= n, S24_ERR_SHAPE, "ldb < n");
    if (int rc = make_map(&mb, b, n, k, ldb, 64, 128)) return rc;
  } else {
    S24_REQUIRE(ldb >= k, S24_ERR_SHAPE, "ldb < k");
    if (int rc = make_map(&mb, b, k, n, ldb, 64, bn_cta)) return rc;
  }
  if (int rc = make_map(&md, d, n, m, ldd, 32, 16, kMapF32Sw128)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sk_tiles = sdw_slabs ? static_cast<int>((m / 512) * ((n + 223) / 224))
                                  : static_cast<int>((m / (pair ? 256 : 128)) * (n / (wide ? 256 : 128)));
  int streamk = use_streamk(sk_tiles, num_sms() / (pair ? 2 : 1), static_cast<int>(k / 128));
  if (!streamk)
    streamk = use_splitk(sk_tiles, pair ? dw_clusters(reserved) : 2 * dw_clusters(reserved), static_cast<int>(k / 128), 16, 4.0 * m * n);
  if (streamk && !accumulate) {  // accumulate: the partial tiles add onto D's current values
    cudaError_t e = cudaMemset2DAsync(d, ldd * sizeof(float), 0, n * sizeof(float), m, st);
    S24_REQUIRE(e == cudaSuccess, S24_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  }
  GemmShape shp{static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), streamk, 8,
                static_cast<unsigned int*>(workspace), streamk == 1 ? 0 : wave_on(true), 0};
  EpiParams ep{d, ldd, nullptr, nullptr, 0, nullptr, nullptr, 0, gate_ff, w, w_dtype, idx, lambda_w, accumulate ? 1 : 0};
  // BN = 256 with one TMEM accumulator (256 + 4 metadata columns): K = tokens is long, so the
  // un-overlapped epilogue is a small share; the B half per CTA is exactly two 64-wide chunks
#define S24_SDW(BMN, BNV, CG, ACC)                                                                            \
  return launch_gemm<true, false, BMN, BNV, stages_for<Cfg<true, false, BMN, BNV, 1, CG, ACC>::STAGE_BYTES>(), \
                     CG, kEpiDw, false, ACC>(ma, mb, me, md, md, md, shp, ep, reserved, st)
  if (sdw_slabs)
    return launch_gemm<true, false, false, 224, stages_for<Cfg<true, false, false, 224, 1, 2, 1, 2>::STAGE_BYTES>(), 2,
                       kEpiDw, false, 1, 2>(ma, mb, me, md, md, md, shp, ep, reserved, st);
  if (wide) {
    if (pair) {
      if (b_mn) S24_SDW(true, 256, 2, 1);
      S24_SDW(false, 256, 2, 1);
    }
    if (b_mn) S24_SDW(true, 256, 1, 1);
    S24_SDW(false, 256, 1, 1);
  }
  if (pair) {
    if (b_mn) S24_SDW(true, 128, 2, 2);
    S24_SDW(false, 128, 2, 2);
  }
  if (b_mn) S24_SDW(true, 128, 1, 2);
  S24_SDW(false, 128, 1, 2);
#undef S24_SDW
}
