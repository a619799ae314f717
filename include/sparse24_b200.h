/*
 * sparse24_b200.h -- C ABI of the B200 (sm_100a) 2:4-sparse FFN hot path.
 *
 * This is the drop-in boundary for the reference package `sparse24`
 * (/root/reference/pkg/src/sparse24).  The reference selects its kernel
 * module at import time (backend.py:13-36) and calls it through
 * `kernels.<fn>` from sparsity.py / spmm.py / gated_ffn.py / optim.py; each
 * entry point below names the reference interface it replaces.
 *
 * Conventions:
 *   - plain pointers to DEVICE memory + sizes; no torch / C++ types;
 *   - the caller allocates every output and workspace; nothing is retained;
 *   - every call is asynchronous on the caller's cudaStream_t (passed as
 *     void*; NULL = legacy default stream) and CUDA-graph capturable;
 *   - return an int status; s24_last_error_string() describes the last
 *     failure of the calling thread.  The Python layer maps
 *     S24_ERR_SHAPE -> ShapeError, S24_ERR_FORMAT -> FormatError (both
 *     ValueError subclasses, matrix.py:11-16), others -> RuntimeError.
 *
 * Data layouts
 *   W       row-major (rows x cols), dtype S24_BF16 / S24_F32 / S24_F64.
 *   idx     uint8 (rows/4 x cols/4): canonical pattern index (0..89) of
 *           every aligned 4x4 block (sparsity.py:208-217 ordering).
 *   vals    bf16 row-major (m x k/2): the two kept values of every row-wise
 *           group of four, ascending (Compressed24.values, spmm.py:38-106).
 *           "fwd" = groups along W's rows (m=rows, k=cols); "bwd" = groups
 *           along W's columns, i.e. the compressed W^T (m=cols, k=rows).
 *   E       the same metadata nibbles (i0 | i1<<2, spmm.py:98-104) arranged
 *           for the sm_100 sparse tensor core: one 2048-byte tile per
 *           (128-row m tile, 128-column k tile), tiles ordered
 *           [m/128][k/128]; inside a tile byte 16*L + 4*c + 2*h holds the
 *           16-bit word of lane L, column c, half h, bits 4g..4g+3 of which
 *           are the nibble of row m = (L%8) + 16*(L/16) + 8*h and group
 *           k/4 = 8*c + 4*((L/8)%2) + g.  Requires m, k multiples of 128.
 *   activations: token-major (tokens x features, row-major) on the hot path;
 *           the sparse GEMM can also emit feature-major (features x tokens,
 *           the storage order of the reference's column-major FST outputs,
 *           gated_ffn.py:162 / _core.pyx:67-69).
 */
#ifndef SPARSE24_B200_H
#define SPARSE24_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S24_ABI_VERSION 2

/* GEMM workspace (every tensor-core GEMM entry point takes `void* workspace, int reserved_sms`):
 * the caller allocates S24_GEMM_WORKSPACE_BYTES of device memory per stream, zeroes it once, and
 * passes it to every GEMM on that stream; the kernels leave it zeroed except for the uint32 at
 * byte 8, a sticky count of bounded cross-CTA waits that gave up (the persistent dW GEMMs'
 * wave-synchronised schedule and the ordered split-K reduce wait for CTAs that were not
 * co-resident, e.g. while another stream's kernels held SMs: the result stays correct, only the
 * L2-locality / summation-order guarantee of that launch was dropped).  workspace = NULL: no
 * wave synchronisation and no ordering -- fully stateless.  reserved_sms: leave that many SMs
 * free (a data-parallel step lets its gradient all-reduce run beside the dX GEMM); 0 = all.
 * The library keeps no mutable state between calls beyond per-process caches of immutable
 * facts (SM count, kernel attributes). */
#define S24_GEMM_WORKSPACE_BYTES 8448
#define S24_GEMM_WS_TIMEOUTS_WORD 2
int64_t s24_gemm_workspace_bytes(void);

/* status codes */
#define S24_OK 0
#define S24_ERR_SHAPE 1       /* -> ShapeError  (matrix.py:11) */
#define S24_ERR_FORMAT 2      /* -> FormatError (matrix.py:15) */
#define S24_ERR_UNSUPPORTED 3 /* dtype / arch / layout not supported */
#define S24_ERR_CUDA 4        /* CUDA runtime / launch failure */
#define S24_ERR_ARG 5         /* null pointer or bad enum */

/* element types */
#define S24_BF16 0
#define S24_F32 1
#define S24_F64 2

/* activations (gated_ffn.py:47-50; SWIGLU is an extension, not in the reference) */
#define S24_ACT_RELU 0
#define S24_ACT_GELU 1
#define S24_ACT_GEGLU 2
#define S24_ACT_SWIGLU 3

/* sparse GEMM epilogues */
#define S24_EPI_STORE 0      /* D = acc (+ bias[m])                                        */
#define S24_EPI_GELU_AUX 1   /* D = z = acc + bias[m]; AUX = gelu(z)          (API fwd GEMM1)  */
#define S24_EPI_GELU_GRAD 2  /* D = gelu(z); AUX = gelu'(z), z = acc + bias[m] (train fwd GEMM1) */
#define S24_EPI_DGELU 3      /* D = acc * AUX (AUX = gelu'(z) input); dbias[m] += sum_n D[m, n]
                                (train bwd GEMM3: activation backward + bias gradient fused)    */
/* gated layers (GEGLU / SwiGLU), first weight compressed u/v-interleaved (gate_ff = d_ff, see
 * s24_search_compress): GEMM1 writes A = act(u) * v (n x d_ff, token-major) and AUX = v act'(u),
 * AUX2 = act(u) (d_ff x n, feature-major); GEMM3 (m = d_ff) reads AUX/AUX2 and writes
 * dZ = [dA AUX | dA AUX2] in the interleaved order (n x 2 d_ff) plus dbias ([b; c] order). */
#define S24_EPI_GEGLU_GRAD 4
#define S24_EPI_SWIGLU_GRAD 5
#define S24_EPI_DGATED 6
/* D += acc (+ bias[m]) into an existing token-major bf16 D (d_t = 1): the store is a TMA bf16
 * add-reduce, so a residual stream's gradient (dh_l = dh_{l+1} + dX_l, the backward of
 * _FFNStack trainer.py:159-262) is accumulated by the dX GEMM itself. */
#define S24_EPI_STORE_ADD 7

const char* s24_last_error_string(void);
int s24_abi_version(void);
/* S24_OK when the current device is sm_100 and the kernels are loadable. */
int s24_device_check(void);

/* ---- K1: transposable mask search ------------------------------------------
 * Replaces transposable_search_conv (sparsity.py:258-271) and its kernel
 * kernels.pattern_scores (_core.pyx:83-110): per 4x4 block the pattern with
 * the largest retained |w| sum, ties -> lowest canonical index; bit-exact
 * with the reference's ascending float64 accumulation for every input.
 * rows, cols: multiples of 4 (else S24_ERR_SHAPE). */
int s24_transposable_search(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx, void* stream);

/* K1 fused: search + compress both orientations in one pass over W.
 * Replaces transposable_search_conv + compress (spmm.py:92-106) +
 * FFNMasks.plans/_GatherPlan (gated_ffn.py:131-188).  Any of fwd_vals,
 * fwd_e, bwd_vals, bwd_e may be NULL; E outputs need rows, cols % 128 == 0.
 * perm_ff > 0 (gated W_in = [u; v], rows = 2 perm_ff): every output (idx, values, E)
 * is produced for the u/v-interleaved row order p -> (p%32 < 16 ? u row 16(p/32) + p%32
 * : v row 16(p/32) + p%32 - 16); 4x4 blocks never straddle u/v, so the masks are the
 * reference's masks with block rows permuted. */
int s24_search_compress(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx, uint16_t* fwd_vals,
                        uint8_t* fwd_e, uint16_t* bwd_vals, uint8_t* bwd_e, int64_t perm_ff, void* stream);

/* K1 of two weights in one launch (the mask refresh of W_in and W2): same semantics as two
 * s24_search_compress calls; one grid over both weights' 128 x 128 tiles. */
int s24_search_compress_pair(const void* w0, const void* w1, int dtype, int64_t rows0, int64_t cols0, int64_t rows1,
                             int64_t cols1, uint8_t* idx0, uint8_t* idx1, uint16_t* fwd_vals0, uint8_t* fwd_e0,
                             uint16_t* bwd_vals0, uint8_t* bwd_e0, uint16_t* fwd_vals1, uint8_t* fwd_e1,
                             uint16_t* bwd_vals1, uint8_t* bwd_e1, int64_t perm_ff0, int64_t perm_ff1, void* stream);

/* ---- K2: per-step prune / compress with a cached mask ----------------------
 * Replaces _GatherPlan.product's gather `w.ravel()[take]` (gated_ffn.py:159-162)
 * for both orientations (in_fwd/in_bwd, out_fwd/out_bwd). */
int s24_prune_compress(const void* w, int dtype, int64_t rows, int64_t cols, const uint8_t* idx,
                       uint16_t* fwd_vals, uint8_t* fwd_e, uint16_t* bwd_vals, uint8_t* bwd_e, int64_t perm_ff,
                       void* stream);

/* K2 of two weights in one launch (the per-step prune of W_in and W2; kept values only,
 * E tiles unchanged): same semantics as two s24_prune_compress calls with NULL E outputs. */
int s24_prune_compress_pair(const void* w0, const void* w1, int dtype, int64_t rows0, int64_t cols0, int64_t rows1,
                            int64_t cols1, const uint8_t* idx0, const uint8_t* idx1, uint16_t* fwd_vals0,
                            uint16_t* bwd_vals0, uint16_t* fwd_vals1, uint16_t* bwd_vals1, int64_t perm_ff0,
                            int64_t perm_ff1, void* stream);

/* ---- format conversions (parity export / TransposableMask API) ------------ */
/* idx -> full 0/1 mask, uint8 rows x cols (TransposableMask.bits, sparsity.py:270-271) */
int s24_idx_to_bits(const uint8_t* idx, int64_t rows, int64_t cols, uint8_t* bits, void* stream);
/* 0/1 mask -> idx; blocks that are not one of the 90 patterns get idx 255 and
 * are counted into *bad_count (device int32, caller zeroes it); the caller
 * raises FormatError when nonzero (TransposableMask.validate, sparsity.py:122-131). */
int s24_bits_to_idx(const uint8_t* bits, int64_t rows, int64_t cols, uint8_t* idx, int32_t* bad_count,
                    void* stream);
/* reference-layout metadata, one nibble per uint8 (Compressed24.meta,
 * spmm.py:98-104): fwd (rows x cols/4), bwd (cols x rows/4); either may be NULL */
int s24_meta_flat(const uint8_t* idx, int64_t rows, int64_t cols, uint8_t* fwd_meta, uint8_t* bwd_meta,
                  void* stream);
/* E tiles (m x k logical) -> reference-layout nibbles (m x k/4) */
int s24_e_to_flat(const uint8_t* e, int64_t m, int64_t k, uint8_t* meta, void* stream);

/* ---- packed 2:4 storage of the API's packed route (Compressed24, spmm.py:38-147) ----
 * Groups of four run along rows (colwise = 0: groups row-major) or down columns
 * (colwise = 1: groups column-major); values hold the two kept entries of every group in
 * group order, meta one nibble i0 | i1 << 2 (i0 < i1) per uint8.
 * s24_pack24: compress (spmm.py:92-106) of w under the 0/1 mask `bits` (both rows x cols
 * row-major; values copied verbatim in w's dtype, rows*cols/2 of them; meta rows*cols/4).
 * Groups whose mask is not exactly two ones are counted into *bad (device int32, caller
 * zeroes; -> FormatError, Mask24.validate sparsity.py:98-105).  w / vals / meta may be NULL
 * (validation only).
 * s24_unpack24: decompress / mask_of (spmm.py:109-135) into a dense row-major out (w's
 * dtype) and / or a 0/1 mask (either may be NULL); groups with i0 >= i1 are counted into
 * *bad (kept_indices, spmm.py:61-67).
 * s24_flat_to_e: reference nibbles of a row-wise (m x k) operand -> E tiles (inverse of
 * s24_e_to_flat), so a bf16 row-wise Compressed24 feeds s24_spmm as (vals, E). */
int s24_pack24(const void* w, int dtype, const uint8_t* bits, int64_t rows, int64_t cols, int colwise, void* vals,
               uint8_t* meta, int32_t* bad, void* stream);
int s24_unpack24(const void* vals, int dtype, const uint8_t* meta, int64_t rows, int64_t cols, int colwise, void* out,
                 uint8_t* bits, int32_t* bad, void* stream);
int s24_flat_to_e(const uint8_t* meta, int64_t m, int64_t k, uint8_t* e, void* stream);

/* ---- K3/K4: 2:4-sparse tcgen05 GEMM ----------------------------------------
 * D[m, n] = sum_k A[m, k] * B[n, k] with A 2:4-sparse (vals m x k/2 + E tiles).
 * Replaces kernels.spmm_colwise (_core.pyx:63-80) as driven by
 * _GatherPlan.product for in_fwd / out_fwd / out_bwd / in_bwd
 * (gated_ffn.py:294, :297, :329, :352).  B: b_mn = 0 -> stored n x k (ldb >= k),
 * b_mn = 1 -> stored k x n (ldb >= n).  D bf16: d_t = 0 -> stored m x n (feature-major,
 * ldd >= n); d_t = 1 -> stored n x m (token-major, ldd >= m).  AUX uses D's layout
 * for S24_EPI_GELU_AUX.  The training epilogues (GELU_GRAD / DGELU, GEGLU_GRAD /
 * SWIGLU_GRAD / DGATED) need d_t = 1 and exchange AUX / AUX2 in the FRAGMENT layout of an
 * F x n matrix (F = m, or gate_ff for the gated ones; ldaux is ignored): 16-feature x
 * 32-token sub-blocks of 512 elements, sub-block (f/16, t/32) at element
 * ((f/16) * (n/32) + t/32) * 512; inside, the 8-element unit 32*s + 4*r + p holds feature
 * 8*s + r of the sub-block (s = (f%16)/8, r = f%8) at tokens 8*c + 2*p + k (element 2*c + k,
 * c = 0..3, k = 0, 1) -- the register layout of a tcgen05.ld 16x256b, so the producing and
 * consuming epilogues move it with coalesced 512-byte accesses.  The buffer holds
 * ceil(F/16) * 16 * n elements.
 * bias (bf16, m) may be NULL.  dbias (fp32, m, zeroed by the caller) is used by
 * S24_EPI_DGELU / S24_EPI_DGATED.  aux2 / gate_ff: gated epilogues only (gate_ff = d_ff).
 * m % 128 == 0, k % 128 == 0, n % 32 == 0. */
int s24_spmm(const uint16_t* a_vals, const uint8_t* a_e, int64_t m, int64_t k, const uint16_t* b, int b_mn,
             int64_t ldb, int64_t n, uint16_t* d, int64_t ldd, const uint16_t* bias, int epilogue, uint16_t* aux,
             int64_t ldaux, uint16_t* aux2, float* dbias, int d_t, int64_t gate_ff, void* workspace, int reserved_sms,
             void* stream);

/* ---- dense token-major GEMM with the training epilogues of s24_spmm ---------------
 * D^T[n, m] (token-major bf16, ldd) = epilogue(sum_k A[m, k] B[n, k]) with A the DENSE bf16
 * weight: w_t = 0 -> A[m, k] = w[m * ldw + k], w_t = 1 -> A[m, k] = w[k * ldw + m] (the
 * transposed orientation of the backward).  w_gate_ff > 0: w's [u; v] dimension (its rows,
 * 2 w_gate_ff of them) is read in the u/v 16-row interleave of the gated epilogues, so the
 * weight stays in the reference's [u; v] order (FFNLayer.w_in_cat, gated_ffn.py:111-115).
 * B token-major (n x k, ldb >= k).  Epilogues, bias / aux / aux2 / dbias / gate_ff: as
 * s24_spmm with d_t = 1 (not S24_EPI_GELU_AUX).  The masks=None route of fst_forward /
 * fst_backward (gated_ffn.py:286-289; the dense fine-tune phase, trainer.py:111-114,
 * :435-437) and the fused dense baseline of bench.py.  m % 128 (CTA pairs when m % 256 == 0), k % 64, n % 32 == 0. */
int s24_gemm_act(const uint16_t* w, int w_t, int64_t ldw, int64_t w_gate_ff, int64_t m, int64_t k, const uint16_t* b,
                 int64_t ldb, int64_t n, uint16_t* d, int64_t ldd, const uint16_t* bias, int epilogue,
                 uint16_t* aux, uint16_t* aux2, float* dbias, int64_t gate_ff, void* workspace, int reserved_sms,
                 void* stream);



/* ---- K5: dense tcgen05 dW GEMM with fused masked decay ---------------------
 * D[m, n] (fp32, ldd) = sum_k A[m, k] B[n, k] + lambda_w * (1 - M[m, n]) * W[m, n]
 * Replaces _grad_weight(mvue=False) (gated_ffn.py:367-371) followed by
 * masked_decay_gradient (optim.py:105-114, applied at trainer.py:439-441).
 * a_mn = 0 -> A stored m x k, 1 -> k x m; b_mn likewise (n x k / k x n).
 * idx/w may be NULL (no decay).  gate_ff > 0: A's rows (m = 2 gate_ff) are in the gated
 * u/v-interleaved order (idx too); D rows and the W rows read for the decay are in [u; v]
 * order.  accumulate = 1: D += the product (TMA fp32 add-reduce into D's current values; the
 * decay, if given, is added once) -- the split-bf16 products of the fp32 mode.
 * m % 128 == 0, n % 256 == 0 (or % 128), k % 64 == 0. */
int s24_gemm_dw(const uint16_t* a, int a_mn, int64_t lda, const uint16_t* b, int b_mn, int64_t ldb, int64_t m,
                int64_t n, int64_t k, float* d, int64_t ldd, const void* w, int w_dtype, const uint8_t* idx,
                float lambda_w, int64_t gate_ff, int accumulate, void* workspace, int reserved_sms, void* stream);

/* ---- K8: MVUE sparsification of an upstream gradient (next row 1 of SURVEY 8f) ----
 * G is n tokens x f features (token-major, ldg); the sparsified matrix is G^T with
 * groups of 4 consecutive tokens per feature -- mvue_slots_rowwise(G^T, seed)
 * (sparsity.py:401-413) as used by _grad_weight(mvue=True) (gated_ffn.py:367-373).
 * (state, inc) = numpy default_rng(seed).bit_generator.state after seeding
 * (128-bit values split hi/lo).  Outputs the kept values g/pi (f x n/2 bf16) and
 * E tiles of the f x n operand; `pairs` (optional, f x n/4) gets each group's kept
 * pair index 0..5 (MVUE_PAIRS order).  gate_ff > 0: feature p of G is row
 * gate_row(p) of [u; v] for the random-stream index.  exact = 1: numpy's PCG64 stream and the
 * reference's float64 decisions, bit-identical to the reference draw (each group in fp32 under a
 * rigorous error certificate, in float64 where the certificate fails; exact = 2 forces float64
 * for every group -- a test hook); exact = 0: the same
 * estimator in fp32 with a counter-based uniform (unbiased, throughput mode).
 * n, f % 128 == 0. */
int s24_mvue_compress(const uint16_t* g, int64_t ldg, int64_t n, int64_t f, uint64_t state_hi, uint64_t state_lo,
                      uint64_t inc_hi, uint64_t inc_lo, int64_t gate_ff, uint16_t* vals, uint8_t* e,
                      uint8_t* pairs, int exact, void* stream);

/* s24_mvue_compress for a token count that is not a multiple of 128 (the reference accepts any
 * multiple of 4): G holds n_valid tokens (rows), the operand is padded to n = n_valid rounded up
 * to 128 (vals f x n/2, E tiles of f x n).  The padded tokens read as zeros (G needs only n_valid
 * rows) and the random-stream index is row * (n_valid / 4) + group -- the reference's draws for
 * its n_valid tokens; the padded groups keep zeros.  The B operand of the weight-gradient GEMM
 * must be zero-padded to n tokens as well.  s24_mvue_compress(..) == this with n_valid = n. */
int s24_mvue_compress_ragged(const uint16_t* g, int64_t ldg, int64_t n, int64_t n_valid, int64_t f,
                             uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                             int64_t gate_ff, uint16_t* vals, uint8_t* e, uint8_t* pairs, int exact, void* stream);

/* mvue_prune (sparsity.py:379-398) of a whole (rows x cols) matrix (bf16 / f32 / f64), groups
 * along rows (colwise = 0, groups row-major) or down columns (colwise = 1, groups
 * column-major): the exact float64 estimator and numpy PCG64 stream of s24_mvue_compress,
 * stream index = group index.  out: dense float64 estimate (kept g / pi, zeros elsewhere);
 * bits (optional): its 0/1 mask.  Bit-exact with the reference. */
int s24_mvue_prune(const void* g, int dtype, int64_t rows, int64_t cols, int colwise, uint64_t state_hi,
                   uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double* out, uint8_t* bits, void* stream);

/* sparse-A weight-gradient GEMM: D[m, n] fp32 = sum_k A~[m, k] B[n, k] + decay, with A~ an
 * MVUE-compressed operand (vals m x k/2, E tiles; k = tokens).  Replaces
 * kernels.spmm_rowwise (_core.pyx:44-60) in _grad_weight(mvue=True).  B layout and
 * w / idx / lambda_w / gate_ff as s24_gemm_dw.  m % 128, k % 128, n % 128 == 0. */
int s24_spmm_dw(const uint16_t* a_vals, const uint8_t* a_e, int64_t m, int64_t k, const uint16_t* b, int b_mn,
                int64_t ldb, int64_t n, float* d, int64_t ldd, const void* w, int w_dtype, const uint8_t* idx,
                float lambda_w, int64_t gate_ff, int accumulate, void* workspace, int reserved_sms, void* stream);

/* ---- K6/K7: fused (gated) activation, token-major ----------------------------
 * Z is n tokens x r_in (r_in = 2r gated, = r plain), row pitch ldz; A is n x r.
 * fwd: A[t, j] = act(Z[t, j]) * Z[t, r + j] (gated) or act(Z[t, j]) (plain);
 * replaces kernels.gate_gelu (_core.pyx:222-250) / _activate (gated_ffn.py:264-270).
 * bwd: dZ (n x r_in) and the bias gradient dbias[j] = sum_t dZ[t, j] (fp32, r_in,
 * zeroed and accumulated by the call); replaces the activation block of
 * fst_backward (gated_ffn.py:336-348). */
int s24_act_fwd(const uint16_t* z, int64_t ldz, int64_t r, int64_t n, int act, uint16_t* a, int64_t lda,
                void* stream);
int s24_act_bwd(const uint16_t* z, int64_t ldz, const uint16_t* da, int64_t ldda, int64_t r, int64_t n, int act,
                uint16_t* dz, int64_t lddz, float* dbias, void* stream);

/* dst (cols x rows, ld ldd) = src^T (rows x cols, ld lds), bf16: the K-major (token-contiguous)
 * B operand of the two-slab MVUE weight-gradient GEMM (s24_spmm_dw with b_mn = 0).  rows, cols,
 * lds, ldd divisible by 8, 16-byte aligned base pointers. */
int s24_transpose_bf16(const uint16_t* src, int64_t rows, int64_t cols, int64_t lds, uint16_t* dst, int64_t ldd,
                       void* stream);

/* ---- fp32 mode (the reference's float32 fused type, _core.pyx:21-23; C1 is fp32) ----------
 * tf32 structured sparsity is 1:2 per 32-bit pair and cannot hold a transposable 2:4 mask, so
 * the fp32 mode runs every product as three bf16 2:4 products on split operands
 * (x = x_hi + x_lo, A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation through the
 * accumulate flag of s24_spmm_dw / s24_gemm_dw).  Activations are FEATURE-major fp32
 * (features x tokens, ld >= n), the storage order of the reference's column-major outputs.
 * s24_split_bf16: hi = bf16(x), lo = bf16(x - hi) over n elements.
 * s24_act_fwd_f32: Z (r_in x n; r_in = 2r gated with rows [u; v], else r) += bias (fp32, may
 *   be NULL) in place, then A = act(z) or act(z_u) z_v (exact erf GELU, exp SiLU) into A
 *   (r x n fp32) and its split A_hi / A_lo (bf16, pitch lda) -- gated_ffn.py:264-270, 293-297.
 * s24_act_bwd_f32: dZ (fp32, may be NULL) and its split dZ_hi / dZ_lo (pitch lddz) from the
 *   pre-activation Z and dA (r x n), and dbias[r_in] = sum over tokens (fixed-order reduction,
 *   written not accumulated) -- gated_ffn.py:336-348. */
int s24_split_bf16(const float* x, int64_t n, uint16_t* hi, uint16_t* lo, void* stream);
int s24_act_fwd_f32(float* z, int64_t ldz, const float* bias, int64_t r, int64_t n, int act, float* a, int64_t lda,
                    uint16_t* a_hi, uint16_t* a_lo, void* stream);
int s24_act_bwd_f32(const float* z, int64_t ldz, const float* da, int64_t ldda, int64_t r, int64_t n, int act,
                    float* dz, int64_t lddz, uint16_t* dz_hi, uint16_t* dz_lo, float* dbias, void* stream);

/* ---- comparators ----------------------------------
 * Greedy 2-approximate transposable search (transposable_search_greedy, sparsity.py:
 * 229-238; kernels.greedy_masks, _core.pyx:139-219), bit-exact, emitted as pattern
 * indices like s24_transposable_search; blocks the greedy scan cannot complete get
 * idx 255 and are counted into *failures (device int32, caller zeroes; the reference
 * raises RuntimeError).  rows, cols % 4 == 0. */
int s24_greedy_search(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* idx, int32_t* failures,
                      void* stream);
/* Directional 2:4 pruning (prune_2of4, sparsity.py:274-279; kernels.prune_2of4_keep,
 * _core.pyx:113-136): bits (uint8 rows x cols) keeps the two largest |w| of each aligned
 * group of four consecutive columns (colwise = 0) or rows (colwise = 1); ties keep the
 * lowest indices.  Bit-exact. */
int s24_prune_2of4(const void* w, int dtype, int64_t rows, int64_t cols, int colwise, uint8_t* bits, void* stream);

/* ---- optimizer step -----------------------------
 * One fused pass per parameter: masked decay on the gradient (decay_mode
 * S24_DECAY_ON_GRADIENTS: g + lambda_w (1 - M) W, optim.py:105-114), Adam
 * (adam_step, optim.py:128-147: u = b1 u + (1 - b1) g, v = b2 v + (1 - b2) g^2,
 * W -= lr u / ((sqrt(v / bias_corr2) + eps) bias_corr1)), and the SR-STE decay at
 * the update site (S24_DECAY_ON_WEIGHTS: W -= lr_lambda (1 - M) W_before,
 * srste_weight_decay optim.py:117-125, trainer.py:442-447).  W, u, v are updated in
 * place; state_dtype S24_F64 reproduces the reference bit for bit when the scalars are
 * passed as Python computes them (one_minus_beta1 = 1.0 - beta1, bias_corr1 =
 * 1.0 - beta1**t, lr_lambda = lr * lambda_w, ...); S24_F32 is the fp32-master-weight
 * path.  g: fp32 or the state's dtype.  idx (pattern indices of the rows x cols
 * weight's mask) is required by the decay modes; without it the parameter is treated
 * as a flat vector of rows * cols elements (biases). */
#define S24_DECAY_NONE 0
#define S24_DECAY_ON_GRADIENTS 1
#define S24_DECAY_ON_WEIGHTS 2
int s24_adam_step(void* w, void* u, void* v, int state_dtype, const void* g, int g_dtype, int64_t rows, int64_t cols,
                  const uint8_t* idx, double lr, double beta1, double beta2, double eps, double one_minus_beta1,
                  double one_minus_beta2, double bias_corr1, double bias_corr2, double lambda_w, double lr_lambda,
                  int decay_mode, void* stream);

/* The fp32 optimizer step of a 2:4 weight fused with the next step's per-step compression:
 * s24_adam_step (state S24_F32, g fp32) on w, u, v in place, and the updated weight's kept
 * values written into both orientations (fwd_vals rows x cols/2, bwd_vals cols x rows/2,
 * either may be NULL) under the cached mask idx -- the same outputs as s24_prune_compress
 * on the updated weight, so the next forward needs no K2 launch (trainer.py:438-447
 * followed by gated_ffn.py:159-162).  idx and the outputs are in the operand's row order:
 * perm_ff > 0 is the gated u/v interleave of s24_search_compress (w, u, v, g stay in [u; v]
 * order).  The masked decay reads its mask from idx.  rows, cols % 128 == 0. */
int s24_adam_compress(float* w, float* u, float* v, const float* g, int64_t rows, int64_t cols, const uint8_t* idx,
                      double lr, double beta1, double beta2, double eps, double one_minus_beta1,
                      double one_minus_beta2, double bias_corr1, double bias_corr2, double lambda_w, double lr_lambda,
                      int decay_mode, uint16_t* fwd_vals, uint16_t* bwd_vals, int64_t perm_ff, void* stream);

/* Mask flips of a refresh (flip_rate optim.py:94-102 = changed_bits / (rows cols); the
 * per-block counts of block_flip_stats optim.py:164-192): adds to *changed_bits (device
 * uint64, caller zeroes) the number of mask bits that differ between two pattern-index
 * maps of nblocks 4x4 blocks, and to block_flips[i] (int32, optional) block i's count. */
int s24_mask_flips(const uint8_t* idx_prev, const uint8_t* idx_curr, int64_t nblocks, unsigned long long* changed_bits,
                   int32_t* block_flips, void* stream);

/* Retained-L1 gap of every 4x4 block (the block_gaps of block_flip_stats,
 * optim.py:164-192): the best minus the second-best of the 90 pattern scores, each score
 * summed in float64 over the pattern's kept positions in ascending order as
 * kernels.pattern_scores does (_core.pyx:102-105), so the gaps are bit-exact; ties give 0.
 * w: (rows, cols) row-major bf16 / f32 / f64, rows, cols % 4 == 0; gaps: (rows/4)(cols/4)
 * float64 in block order. */
int s24_block_gaps(const void* w, int dtype, int64_t rows, int64_t cols, double* gaps, void* stream);

/* ---- standalone masked decay on an fp32 gradient (optim.py:105-114) -------- */
int s24_masked_decay(float* g, const void* w, int w_dtype, const uint8_t* idx, int64_t rows, int64_t cols,
                     float lambda_w, void* stream);
/* The same under an arbitrary 0/1 mask `bits` (uint8, one per element) over n elements of any
 * shape -- masked_decay_gradient on a flat parameter vector with a dense mask
 * (optim.py:105-114, trainer.py:439-441). */
int s24_masked_decay_bits(float* g, const void* w, int w_dtype, const uint8_t* bits, int64_t n, float lambda_w,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSE24_B200_H */
