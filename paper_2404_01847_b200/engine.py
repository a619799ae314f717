"""Raw-tensor engine of the 2:4 FFN hot path (one FFN block fwd + bwd).

Every function here is a thin sequence of C-ABI kernel launches on the
current CUDA stream; the reference-facing API (gated_ffn.py) and the autograd
module (module.py) are built on it.

Layouts (see include/sparse24_b200.h):
  x, dy            token-major  (N x d, row-major) -- the caller's tensors
  zt, at, dat, dzt feature-major (features x N, row-major): the sparse GEMM
                   writes D[m = feature, n = token], which is the reference's
                   column-major FST output (gated_ffn.py:162, _core.pyx:67-69)
  yt, dxt          feature-major (d x N); the API returns them as the
                   column-major logical views y = yt.t(), dx = dxt.t()

Reference call stack replaced:
  forward : in_fwd.product -> +bias -> _activate -> out_fwd.product   (gated_ffn.py:293-297)
  backward: out_bwd.product, _grad_weight x2, activation bwd, in_bwd.product (gated_ffn.py:327-356)
  update  : masked_decay_gradient (optim.py:105-114) fused into the dW epilogue
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import torch

from . import _capi as C
from .matrix import ShapeError


class _NoTimer:
    def __call__(self, name):
        return self

    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# Optional per-launch timer hook (bench.py installs a CUDA-event timer to
# attribute step time to kernels); the default is a no-op.
TIMER = _NoTimer()

# Per-(device, stream) GEMM workspace (include/sparse24_b200.h, S24_GEMM_WORKSPACE_BYTES): the
# counters of the dW GEMMs' wave-synchronised schedule and ordered split-K live here, owned by the
# caller, so launches on different streams never share them and the library keeps no state.
_WORKSPACES: dict = {}
# SMs every GEMM leaves free (the data-parallel step sets it while its all-reduce is in flight)
RESERVED_SMS = 0


def gemm_workspace(t: torch.Tensor) -> torch.Tensor:
    dev = t.device
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = torch.zeros(C.GEMM_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
        _WORKSPACES[key] = ws
    return ws


def gemm_timeouts(device=None) -> int:
    """Bounded cross-CTA waits that gave up on the current stream's GEMMs so far (their L2-locality
    or summation-order guarantee was dropped; the results are correct either way)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = _WORKSPACES.get((dev.index, torch.cuda.current_stream(dev).cuda_stream))
    return 0 if ws is None else int(ws[C.GEMM_WS_TIMEOUTS_WORD].item())


class reserved_sms:
    """Context: every GEMM launched inside leaves `n` SMs free (per-call argument of the ABI)."""

    def __init__(self, n: int):
        self.n = int(n)

    def __enter__(self):
        global RESERVED_SMS
        self.prev, RESERVED_SMS = RESERVED_SMS, self.n
        return self

    def __exit__(self, *a):
        global RESERVED_SMS
        RESERVED_SMS = self.prev
        return False


ACT_CODES = {"relu": C.ACT_RELU, "gelu": C.ACT_GELU, "geglu": C.ACT_GEGLU, "swiglu": C.ACT_SWIGLU}
GATED = {"geglu", "swiglu"}


@dataclass
class CompressedOperand:
    """Both 2:4 orientations of one weight under one transposable mask -- the
    B200 counterpart of a pair of _GatherPlans (gated_ffn.py:131-188)."""

    rows: int
    cols: int
    idx: torch.Tensor  # (rows/4, cols/4) pattern indices (the mask)
    fwd_vals: torch.Tensor  # (rows, cols/2) bf16: A operand of W x (fwd)
    fwd_e: torch.Tensor  # E tiles for fwd_vals
    bwd_vals: torch.Tensor  # (cols, rows/2) bf16: A operand of W^T (bwd)
    bwd_e: torch.Tensor  # E tiles for bwd_vals
    perm_ff: int = 0  # > 0: gated W_in = [u; v] stored u/v-interleaved (16-row groups), d_ff = perm_ff

    @classmethod
    def empty(cls, rows: int, cols: int, device, perm_ff: int = 0) -> "CompressedOperand":
        if rows % 128 or cols % 128:
            raise ShapeError(
                f"2:4 tensor-core operands need both weight dims divisible by 128, got ({rows}, {cols})")
        e_bytes = (rows // 128) * (cols // 128) * 2048
        u8 = dict(dtype=torch.uint8, device=device)
        bf = dict(dtype=torch.bfloat16, device=device)
        if perm_ff and (rows != 2 * perm_ff or perm_ff % 16):
            raise ShapeError(f"gated interleave needs rows == 2 * d_ff and d_ff % 16 == 0, got {rows}, {perm_ff}")
        return cls(rows, cols, torch.empty((rows // 4, cols // 4), **u8),
                   torch.empty((rows, cols // 2), **bf), torch.empty(e_bytes, **u8),
                   torch.empty((cols, rows // 2), **bf), torch.empty(e_bytes, **u8), perm_ff)

    def mask_idx(self) -> torch.Tensor:
        """Pattern indices in the weight's own row order (undoing the gated interleave)."""
        if not self.perm_ff:
            return self.idx
        p = torch.arange(0, self.rows, 4, device=self.idx.device)
        orig = torch.where(p % 32 < 16, 16 * (p // 32) + p % 32, self.perm_ff + 16 * (p // 32) + p % 32 - 16)
        out = torch.empty_like(self.idx)
        out[orig // 4] = self.idx
        return out


def search_compress(w: torch.Tensor, op: CompressedOperand) -> None:
    """K1 fused: new mask + metadata + kept values (mask refresh step)."""
    with TIMER("k1_search_compress"):
        C.call("s24_search_compress", w.data_ptr(), C.dtype_code(w), op.rows, op.cols, op.idx.data_ptr(),
               op.fwd_vals.data_ptr(), op.fwd_e.data_ptr(), op.bwd_vals.data_ptr(), op.bwd_e.data_ptr(),
               op.perm_ff, C.stream_of(w))


def search_compress_pair(w0: torch.Tensor, op0: CompressedOperand, w1: torch.Tensor,
                         op1: CompressedOperand) -> None:
    """K1 of both weights of a block in one launch (the mask refresh of W_in and W2)."""
    if w0.dtype != w1.dtype:
        raise ShapeError("search_compress_pair needs both weights in one dtype")
    with TIMER("k1_search_compress"):
        C.call("s24_search_compress_pair", w0.data_ptr(), w1.data_ptr(), C.dtype_code(w0), op0.rows, op0.cols,
               op1.rows, op1.cols, op0.idx.data_ptr(), op1.idx.data_ptr(), op0.fwd_vals.data_ptr(),
               op0.fwd_e.data_ptr(), op0.bwd_vals.data_ptr(), op0.bwd_e.data_ptr(), op1.fwd_vals.data_ptr(),
               op1.fwd_e.data_ptr(), op1.bwd_vals.data_ptr(), op1.bwd_e.data_ptr(), op0.perm_ff, op1.perm_ff,
               C.stream_of(w0))


def compress_with_meta(w: torch.Tensor, op: CompressedOperand) -> None:
    """K2 with metadata: (re)build E tiles and values from a given mask (op.idx)."""
    C.call("s24_prune_compress", w.data_ptr(), C.dtype_code(w), op.rows, op.cols, op.idx.data_ptr(),
           op.fwd_vals.data_ptr(), op.fwd_e.data_ptr(), op.bwd_vals.data_ptr(), op.bwd_e.data_ptr(),
           op.perm_ff, C.stream_of(w))


def compress_values(w: torch.Tensor, op: CompressedOperand) -> None:
    """K2: per-step prune/compress of the current weight values (mask cached)."""
    with TIMER("k2_prune_compress"):
        C.call("s24_prune_compress", w.data_ptr(), C.dtype_code(w), op.rows, op.cols, op.idx.data_ptr(),
               op.fwd_vals.data_ptr(), None, op.bwd_vals.data_ptr(), None, op.perm_ff, C.stream_of(w))


def compress_values_pair(w0: torch.Tensor, op0: CompressedOperand, w1: torch.Tensor,
                         op1: CompressedOperand) -> None:
    """K2 of both weights of a block in one launch (same results as two compress_values calls)."""
    if w0.dtype != w1.dtype:
        compress_values(w0, op0)
        compress_values(w1, op1)
        return
    with TIMER("k2_prune_compress"):
        C.call("s24_prune_compress_pair", w0.data_ptr(), w1.data_ptr(), C.dtype_code(w0), op0.rows, op0.cols,
               op1.rows, op1.cols, op0.idx.data_ptr(), op1.idx.data_ptr(), op0.fwd_vals.data_ptr(),
               op0.bwd_vals.data_ptr(), op1.fwd_vals.data_ptr(), op1.bwd_vals.data_ptr(), op0.perm_ff, op1.perm_ff,
               C.stream_of(w0))


def spmm(vals: torch.Tensor, e: torch.Tensor, m: int, k: int, b: torch.Tensor, b_mn: bool, n: int,
         out: torch.Tensor, bias: torch.Tensor | None = None, gelu_aux: torch.Tensor | None = None,
         tag: str = "k34_spmm", epi: int | None = None, aux: torch.Tensor | None = None,
         dbias: torch.Tensor | None = None, out_t: bool = False, aux2: torch.Tensor | None = None,
         gate_ff: int = 0) -> None:
    """D[m, n] = W~[m, k] (2:4) . B[n, k]^T, stored as out[m, n] (feature-major)
    or, with out_t, as out[n, m] (token-major); epilogues: EPI_STORE (+bias),
    EPI_GELU_AUX (out = z, aux = gelu(z)), EPI_GELU_GRAD (out = gelu(z),
    aux = gelu'(z)), EPI_DGELU (out = acc * aux, dbias += sums over tokens)."""
    if epi is None:
        epi = C.EPI_GELU_AUX if gelu_aux is not None else C.EPI_STORE
    if gelu_aux is not None:
        aux = gelu_aux
    with TIMER(tag):
        C.call("s24_spmm", vals.data_ptr(), e.data_ptr(), m, k, b.data_ptr(), int(b_mn), b.stride(0), n,
               out.data_ptr(), out.stride(0), C.ptr(bias), epi, C.ptr(aux), aux.stride(0) if aux is not None else 0,
               C.ptr(aux2), C.ptr(dbias), int(out_t), gate_ff, gemm_workspace(out).data_ptr(),
               RESERVED_SMS, C.stream_of(out))


def gemm_dw(a: torch.Tensor, a_mn: bool, b: torch.Tensor, b_mn: bool, m: int, n: int, k: int,
            out: torch.Tensor, w: torch.Tensor | None = None, idx: torch.Tensor | None = None,
            lam: float = 0.0, tag: str = "k5_gemm_dw", gate_ff: int = 0, accumulate: bool = False) -> None:
    """out[m, n] fp32 (+)= sum_k A[m, k] B[n, k] + lam (1 - M) W  (dense tcgen05)."""
    decay = idx is not None and lam != 0.0
    with TIMER(tag):
        C.call("s24_gemm_dw", a.data_ptr(), int(a_mn), a.stride(0), b.data_ptr(), int(b_mn), b.stride(0), m, n,
               k, out.data_ptr(), out.stride(0), C.ptr(w) if decay else None, C.dtype_code(w) if decay else 0,
               C.ptr(idx) if decay else None, float(lam if decay else 0.0), gate_ff, int(accumulate),
               gemm_workspace(out).data_ptr(),
               RESERVED_SMS, C.stream_of(out))


def mvue_seed(rng_seed: int, salt: int) -> int:
    """Per-product seed of _grad_weight (gated_ffn.py:372): (seed << 2) ^ salt."""
    return (int(rng_seed) << 2) ^ salt


def pcg64_state(seed: int) -> tuple[int, int, int, int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy default_rng(seed) after seeding
    (sparsity.py:364) -- the device regenerates the same PCG64 stream."""
    import numpy as np

    st = np.random.default_rng(int(seed) & 0xFFFF_FFFF_FFFF_FFFF).bit_generator.state["state"]
    s, i = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    return s >> 64, s & m64, i >> 64, i & m64


def mvue_compress(g: torch.Tensor, seed: int, gate_ff: int = 0, want_pairs: bool = False, exact: bool = True):
    """K8: MVUE-sparsify g^T (features x tokens) along tokens (sparsity.py:401-413)
    into the tensor-core operand.  g: token-major (N x F) bf16.  Returns
    (vals F x N/2, E tiles, pairs F x N/4 or None).  exact=True: numpy's PCG64 stream and the
    reference's float64 decisions (fp32 under an error certificate, float64 where the certificate
    fails; exact=2 forces float64 everywhere, a test hook).  exact=False: fp32 math and a
    counter-based uniform (unbiased, not numpy's stream) for throughput.  N not a multiple of 128
    (any multiple of 4, as the reference allows): the operand covers N rounded up to 128 tokens
    (s24_mvue_compress_ragged: the reference's draws for the N real tokens, zeros after them),
    so the GEMM's other operand must be padded the same way (pad_tokens)."""
    n_valid, f = g.shape
    n = (n_valid + 127) // 128 * 128
    dev = g.device
    vals = torch.empty((f, n // 2), dtype=torch.bfloat16, device=dev)
    e = torch.empty((f // 128) * (n // 128) * 2048, dtype=torch.uint8, device=dev)
    pairs = torch.empty((f, n // 4), dtype=torch.uint8, device=dev) if want_pairs else None
    sh, sl, ih, il = pcg64_state(seed)
    with TIMER("k8_mvue"):
        C.call("s24_mvue_compress_ragged", g.data_ptr(), g.stride(0), n, n_valid, f, sh, sl, ih, il, gate_ff,
               vals.data_ptr(), e.data_ptr(), C.ptr(pairs), int(exact), C.stream_of(g))
    return vals, e, pairs


def pad_tokens(x: torch.Tensor, granule: int = 128) -> torch.Tensor:
    """x (tokens x features) with zero rows up to a multiple of `granule` tokens (x itself when
    aligned): 128 for the token operand of an MVUE weight-gradient GEMM, 64 for a batch entering
    the tensor-core path (the reference takes any batch; zero tokens change no real output and,
    with a zero upstream gradient, no gradient sum)."""
    n = x.shape[0]
    if n % granule == 0:
        return x
    out = torch.zeros(((n + granule - 1) // granule * granule, x.shape[1]), dtype=x.dtype, device=x.device)
    out[:n].copy_(x)
    return out


def transpose_bf16(x: torch.Tensor) -> torch.Tensor:
    """x^T (bf16, contiguous) by the repo's tiled transpose kernel."""
    rows, cols = x.shape
    out = torch.empty((cols, rows), dtype=torch.bfloat16, device=x.device)
    with TIMER("k14_transpose"):
        C.call("s24_transpose_bf16", x.data_ptr(), rows, cols, x.stride(0), out.data_ptr(), rows, C.stream_of(x))
    return out


def _sdw_slabs(m: int, n: int, k: int, dev) -> bool:
    """Mirror of the library's choice of two-slab tiles for the 2:4 weight-gradient GEMM
    (s24_gemm.cu use_sdw_slabs): worth a K-major copy of the token operand."""
    env = os.environ.get("S24_SDW_SLABS")
    if env is not None:
        return env == "1" and m % 512 == 0
    clusters = torch.cuda.get_device_properties(dev).multi_processor_count // 2
    return m % 512 == 0 and k >= 4096 and (m // 512) * ((n + 223) // 224) >= 2 * clusters


def spmm_dw_tokens(vals, e, m: int, k: int, b_tok: torch.Tensor, n: int, out: torch.Tensor, w, idx, lam: float,
                   gate_ff: int, tag: str) -> None:
    """The MVUE weight gradient out[m, n] = A~[m, k] . B_tok[k, n] with B_tok token-major (k = tokens):
    large shapes transpose B_tok once (k14, HBM-bound) so the GEMM runs two-slab 512 x 224 tiles on a
    K-major B (-22 % operand bytes per MAC on this L2-bound GEMM); small ones read B_tok MN-major."""
    if _sdw_slabs(m, n, k, b_tok.device):
        spmm_dw(vals, e, m, k, transpose_bf16(b_tok), False, n, out, w, idx, lam, gate_ff, tag=tag)
    else:
        spmm_dw(vals, e, m, k, b_tok, True, n, out, w, idx, lam, gate_ff, tag=tag)


def spmm_dw(vals: torch.Tensor, e: torch.Tensor, m: int, k: int, b: torch.Tensor, b_mn: bool, n: int,
            out: torch.Tensor, w: torch.Tensor | None = None, idx: torch.Tensor | None = None, lam: float = 0.0,
            gate_ff: int = 0, tag: str = "k8_spmm_dw", accumulate: bool = False) -> None:
    """out[m, n] fp32 (+)= 2:4 A~[m, k] . B[n, k]^T + lam (1 - M) W (2:4 tensor cores); A~ an MVUE
    operand or a compressed weight (the fp32 mode's split-bf16 products)."""
    decay = idx is not None and lam != 0.0
    with TIMER(tag):
        C.call("s24_spmm_dw", vals.data_ptr(), e.data_ptr(), m, k, b.data_ptr(), int(b_mn), b.stride(0), n,
               out.data_ptr(), out.stride(0), C.ptr(w) if decay else None, C.dtype_code(w) if decay else 0,
               C.ptr(idx) if decay else None, float(lam if decay else 0.0), gate_ff, int(accumulate),
               gemm_workspace(out).data_ptr(),
               RESERVED_SMS, C.stream_of(out))


@dataclass
class DenseOperand:
    """A dense bf16 weight on the tensor-core path (masks=None: the dense fine-tune phase,
    gated_ffn.py:286-289, and the fused dense baseline).  perm_ff > 0: the gated first weight
    [u; v] (rows = 2 perm_ff) is read u/v-interleaved by the GEMM's TMA map, so it stays in the
    reference's order and needs no copy."""

    w: torch.Tensor  # (rows, cols) bf16, row-major
    perm_ff: int = 0

    @property
    def rows(self) -> int:
        return self.w.shape[0]

    @property
    def cols(self) -> int:
        return self.w.shape[1]

    idx = None  # no mask: no masked decay

    @classmethod
    def of(cls, w: torch.Tensor, perm_ff: int = 0) -> "DenseOperand":
        if w.dtype != torch.bfloat16 or w.stride(1) != 1 or w.stride(0) % 8 or w.data_ptr() % 16:
            raise ShapeError("dense tensor-core weights must be bf16, row-major, 16-byte aligned rows")
        return cls(w, perm_ff)


def _mm(op, bwd: bool, b: torch.Tensor, n: int, out: torch.Tensor, tag: str, epi: int = C.EPI_STORE,
        bias: torch.Tensor | None = None, aux: torch.Tensor | None = None, aux2: torch.Tensor | None = None,
        dbias: torch.Tensor | None = None, gate_ff: int = 0) -> None:
    """One token-major product of the FFN step: out^T = op (W or W^T when bwd) . b^T with a
    training epilogue -- the 2:4 GEMM on a CompressedOperand, the dense one on a DenseOperand."""
    m, k = (op.cols, op.rows) if bwd else (op.rows, op.cols)
    if isinstance(op, CompressedOperand):
        spmm(op.bwd_vals if bwd else op.fwd_vals, op.bwd_e if bwd else op.fwd_e, m, k, b, False, n, out, bias,
             tag=tag, epi=epi, aux=aux, dbias=dbias, out_t=True, aux2=aux2, gate_ff=gate_ff)
        return
    with TIMER(tag):
        C.call("s24_gemm_act", op.w.data_ptr(), int(bwd), op.w.stride(0), op.perm_ff, m, k, b.data_ptr(),
               b.stride(0), n, out.data_ptr(), out.stride(0), C.ptr(bias), epi, C.ptr(aux), C.ptr(aux2),
               C.ptr(dbias), gate_ff, gemm_workspace(out).data_ptr(),
               RESERVED_SMS, C.stream_of(out))


def aux_empty(f: int, n: int, device) -> torch.Tensor:
    """Buffer for an AUX matrix (f features x n tokens) in the fragment layout exchanged by the
    training epilogues (include/sparse24_b200.h, s24_spmm)."""
    return torch.empty((-(-f // 16) * 16, n), dtype=torch.bfloat16, device=device)


def aux_to_feature_major(g: torch.Tensor, f: int, n: int) -> torch.Tensor:
    """Fragment-layout AUX -> (f, n) feature-major (inspection / tests).
    Storage order per 16 x 32 sub-block: [s][r][p][c][k] for feature 8 s + r, token 8 c + 2 p + k."""
    fb = -(-f // 16)
    return g.reshape(fb, n // 32, 2, 8, 4, 4, 2).permute(0, 2, 3, 1, 5, 4, 6).reshape(fb * 16, n)[:f]


def aux_from_feature_major(x: torch.Tensor) -> torch.Tensor:
    """(f, n) feature-major -> fragment-layout AUX (tests)."""
    f, n = x.shape
    fb = -(-f // 16)
    xp = torch.zeros((fb * 16, n), dtype=x.dtype, device=x.device)
    xp[:f] = x
    return xp.reshape(fb, 2, 8, n // 32, 4, 4, 2).permute(0, 3, 1, 2, 5, 4, 6).contiguous().reshape(fb * 16, n)


def _rows(t: torch.Tensor) -> torch.Tensor:
    """Row-major (token-major) storage with a 16-byte aligned pitch."""
    if t.stride(1) == 1 and t.stride(0) >= t.shape[1] and t.stride(0) % 8 == 0 and t.data_ptr() % 16 == 0:
        return t
    return t.contiguous()


@dataclass
class FwdState:
    x: torch.Tensor  # (N, d) bf16, token-major
    z: torch.Tensor | None  # (N, r_in) pre-activation (None on the fused training path)
    a: torch.Tensor  # (N, d_ff)
    y: torch.Tensor  # (N, d)
    g: torch.Tensor | None = None  # GELU'(z) / gated v act'(u), fragment layout (d_ff x N), fused path only
    g2: torch.Tensor | None = None  # gated act(u), fragment layout (d_ff x N), fused gated path only


def ffn_forward(x: torch.Tensor, w_in: "CompressedOperand | DenseOperand", bias_in: torch.Tensor | None,
                w2: "CompressedOperand | DenseOperand", act: str, fused: bool = False) -> FwdState:
    """Z = X W_in~^T + b -> A = act(Z) -> Y = A W2~^T (gated_ffn.py:293-297).

    fused=True (GELU / gated): GEMM1's epilogue stores A = GELU(z) and
    G = GELU'(z) (gated: A = act(u) v, G = v act'(u), G2 = act(u)) instead of z,
    so the backward's GEMM3 epilogue applies the activation derivative and
    reduces the bias gradient (no separate K7).  DenseOperand weights run the same
    epilogues on dense tensor-core GEMMs (masks=None, gated_ffn.py:286-289)."""
    n, d = x.shape
    r_in = w_in.rows
    d_ff = w2.cols
    if w_in.cols != d or w2.rows != d or (r_in != (2 * d_ff if act in GATED else d_ff)):
        raise ShapeError("layer weight shapes are inconsistent with the activation / input width")
    if n % 64:
        raise ShapeError(f"token count must be a multiple of 64 on the tensor-core path, got {n}")
    dev = x.device
    x = _rows(x)
    a = torch.empty((n, d_ff), dtype=torch.bfloat16, device=dev)
    y = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    if fused and act in GATED:
        if w_in.perm_ff != d_ff:
            raise ShapeError("the fused gated path needs the first weight read u/v-interleaved (perm_ff = d_ff)")
        g = aux_empty(d_ff, n, dev)  # v act'(u), fragment layout
        g2 = aux_empty(d_ff, n, dev)  # act(u), fragment layout
        _mm(w_in, False, x, n, a, "k3_spmm_fwd_in", bias=bias_in,
            epi=C.EPI_SWIGLU_GRAD if act == "swiglu" else C.EPI_GEGLU_GRAD, aux=g, aux2=g2, gate_ff=d_ff)
        _mm(w2, False, a, n, y, "k3_spmm_fwd_out")
        return FwdState(x, None, a, y, g, g2)
    if w_in.perm_ff:
        raise ShapeError("an interleaved gated operand is only valid on the fused path")
    if fused and act == "gelu":
        g = aux_empty(d_ff, n, dev)  # GELU'(z), fragment layout, read back by GEMM3's epilogue
        _mm(w_in, False, x, n, a, "k3_spmm_fwd_in", bias=bias_in, epi=C.EPI_GELU_GRAD, aux=g)
        _mm(w2, False, a, n, y, "k3_spmm_fwd_out")
        return FwdState(x, None, a, y, g)
    z = torch.empty((n, r_in), dtype=torch.bfloat16, device=dev)
    if act == "gelu" and isinstance(w_in, CompressedOperand):
        spmm(w_in.fwd_vals, w_in.fwd_e, r_in, d, x, False, n, z, bias_in, gelu_aux=a, tag="k3_spmm_fwd_in",
             out_t=True)
    else:
        _mm(w_in, False, x, n, z, "k3_spmm_fwd_in", bias=bias_in)
        with TIMER("k6_act_fwd"):
            C.call("s24_act_fwd", z.data_ptr(), r_in, d_ff, n, ACT_CODES[act], a.data_ptr(), d_ff, C.stream_of(z))
    _mm(w2, False, a, n, y, "k3_spmm_fwd_out")
    return FwdState(x, z, a, y)


@dataclass
class Grads:
    dx: torch.Tensor  # (N, d) bf16
    dw_in: torch.Tensor  # (r_in, d) fp32
    dbias_in: torch.Tensor  # (r_in,) fp32
    dw2: torch.Tensor  # (d, d_ff) fp32


def ffn_backward(st: FwdState, dy: torch.Tensor, w_in: CompressedOperand, w2: CompressedOperand, act: str,
                 w_in_dense: torch.Tensor | None = None, w2_dense: torch.Tensor | None = None,
                 lam: float = 0.0, dw_in_out: torch.Tensor | None = None,
                 dw2_out: torch.Tensor | None = None, mvue: bool = False, rng_seed: int = 0,
                 mvue_exact: bool = True, dbias_out: torch.Tensor | None = None,
                 grads_ready=None, dx_accumulate: torch.Tensor | None = None, dw2_ready=None,
                 n_valid: int | None = None) -> Grads:
    """dA = dY W2~ (out_bwd, W2's transposed orientation) -> dZ (activation
    backward, bias gradient) -> dX = dZ W_in~ (in_bwd); dense dW2 = dY^T A and
    dW_in = dZ^T X with the masked decay lam (1 - M) W fused (gated_ffn.py:327-356).
    mvue=True: both weight gradients use the MVUE-sparsified upstream gradients
    (dY^T with salt 1, dZ^T with salt 2, seeds (rng_seed << 2) ^ salt) on the
    2:4 tensor cores (gated_ffn.py:367-373).

    Launch order: dA/dZ (+ bias gradient), dW2, dW_in, then dX, so that
    `dw2_ready()` -- called once dW2 and the bias gradient are enqueued (before the dW_in GEMM) -- and
    `grads_ready()` -- called once every weight/bias gradient is enqueued -- can start
    the data-parallel all-reduce of the gradient bucket while dX is still computing.
    dbias_out / dw_in_out / dw2_out let the caller hand in views of that bucket.
    dx_accumulate: a residual stream's gradient buffer; dX is added into it by the dX GEMM's
    store (S24_EPI_STORE_ADD) instead of being written to a fresh tensor.  It may be `dy`
    itself: every reader of dy is enqueued before the dX GEMM on the same stream.
    n_valid: the caller padded the token batch with zero rows to a multiple of 64 (gated_ffn);
    the MVUE draws then cover the first n_valid tokens, as the reference's do for its batch."""
    n, d = st.x.shape
    r_in, d_ff = w_in.rows, w2.cols
    if tuple(dy.shape) != (n, d):
        raise ShapeError(f"upstream shape {tuple(dy.shape)} != output shape {(n, d)}")
    dev = dy.device
    dy = _rows(dy)
    dz = torch.empty((n, r_in), dtype=torch.bfloat16, device=dev)
    gate_ff = w_in.perm_ff
    if st.g2 is not None:
        # gated: dZ_u = dA v act'(u), dZ_v = dA act(u) straight into the interleaved dZ, bias grads fused
        dbias = dbias_out.zero_() if dbias_out is not None else torch.zeros(r_in, dtype=torch.float32, device=dev)
        _mm(w2, True, dy, n, dz, "k4_spmm_bwd_out", epi=C.EPI_DGATED, aux=st.g, aux2=st.g2, dbias=dbias,
            gate_ff=d_ff)
    elif st.g is not None:
        # dZ = (dY W2~) * GELU'(z) with the bias gradient reduced in the same epilogue
        dbias = dbias_out.zero_() if dbias_out is not None else torch.zeros(r_in, dtype=torch.float32, device=dev)
        _mm(w2, True, dy, n, dz, "k4_spmm_bwd_out", epi=C.EPI_DGELU, aux=st.g, dbias=dbias)
    else:
        da = torch.empty((n, d_ff), dtype=torch.bfloat16, device=dev)
        _mm(w2, True, dy, n, da, "k4_spmm_bwd_out")
        dbias = dbias_out if dbias_out is not None else torch.empty(r_in, dtype=torch.float32, device=dev)
        with TIMER("k7_act_bwd"):
            C.call("s24_act_bwd", st.z.data_ptr(), r_in, da.data_ptr(), d_ff, d_ff, n, ACT_CODES[act],
                   dz.data_ptr(), r_in, dbias.data_ptr(), C.stream_of(dz))
    # dW2[d, d_ff] = dY^T A and dW_in[r_in, d] = dZ^T X: K = tokens, both operands token-major (MN-major)
    dw2 = dw2_out if dw2_out is not None else torch.empty((d, d_ff), dtype=torch.float32, device=dev)
    dw_in = dw_in_out if dw_in_out is not None else torch.empty((r_in, d), dtype=torch.float32, device=dev)
    if mvue:
        # the MVUE operand is tiled in 128-token groups: a batch that is not a multiple of 128 (legal
        # for the reference, any multiple of 4) runs the GEMM over the padded token count, with the
        # reference's draws for the real tokens and zero rows after them in both operands
        n_op = (n + 127) // 128 * 128
        nv = n if n_valid is None else n_valid
        v2, e2, _ = mvue_compress(dy[:nv], mvue_seed(rng_seed, 1), exact=mvue_exact)
        spmm_dw_tokens(v2, e2, d, n_op, pad_tokens(st.a), d_ff, dw2, w2_dense, w2.idx, lam, 0, "k8_spmm_dw2")
        if dw2_ready is not None:
            dw2_ready()
        v1, e1, _ = mvue_compress(dz[:nv], mvue_seed(rng_seed, 2), gate_ff, exact=mvue_exact)
        spmm_dw_tokens(v1, e1, r_in, n_op, pad_tokens(st.x), d, dw_in, w_in_dense, w_in.idx, lam, gate_ff,
                       "k8_spmm_dw_in")
    else:
        gemm_dw(dy, True, st.a, True, d, d_ff, n, dw2, w2_dense, w2.idx, lam, tag="k5_gemm_dw2")
        if dw2_ready is not None:
            dw2_ready()
        gemm_dw(dz, True, st.x, True, r_in, d, n, dw_in, w_in_dense, w_in.idx, lam, tag="k5_gemm_dw_in",
                gate_ff=gate_ff)
    if grads_ready is not None:
        grads_ready()
    if dx_accumulate is not None:
        # residual stream: dX is add-reduced into the caller's (n, d) gradient by the GEMM's store
        if tuple(dx_accumulate.shape) != (n, d) or dx_accumulate.dtype != torch.bfloat16 \
                or not dx_accumulate.is_contiguous():
            raise ShapeError("dx_accumulate must be a contiguous (tokens, d) bf16 tensor")
        dx = dx_accumulate
        _mm(w_in, True, dz, n, dx, "k4_spmm_bwd_in", epi=C.EPI_STORE_ADD)
    else:
        dx = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
        _mm(w_in, True, dz, n, dx, "k4_spmm_bwd_in")
    return Grads(dx, dw_in, dbias, dw2)


# ---------------------------------------------------------------------------
# fp32 mode: split-bf16 products on the 2:4 tensor cores (include/sparse24_b200.h, s24_fp32.cu)


def split_bf16(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """x (fp32, contiguous) -> (hi, lo) bf16 with hi = bf16(x), lo = bf16(x - hi)."""
    x = x.contiguous()
    hi = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    lo = torch.empty_like(hi)
    C.call("s24_split_bf16", x.data_ptr(), x.numel(), hi.data_ptr(), lo.data_ptr(), C.stream_of(x))
    return hi, lo


@dataclass
class SplitOperand:
    """An fp32 weight under one transposable mask as two 2:4 operands: hi = bf16(W) and
    lo = bf16(W - hi), sharing the pattern indices and E tiles (both orientations)."""

    hi: CompressedOperand
    lo: CompressedOperand

    @property
    def rows(self) -> int:
        return self.hi.rows

    @property
    def cols(self) -> int:
        return self.hi.cols

    @property
    def idx(self) -> torch.Tensor:
        return self.hi.idx

    @classmethod
    def empty(cls, rows: int, cols: int, device) -> "SplitOperand":
        hi = CompressedOperand.empty(rows, cols, device)
        lo = CompressedOperand(rows, cols, hi.idx, torch.empty_like(hi.fwd_vals), hi.fwd_e,
                               torch.empty_like(hi.bwd_vals), hi.bwd_e)
        return cls(hi, lo)

    def compress(self, w: torch.Tensor, with_meta: bool = False) -> None:
        """Kept values of both halves (K2) from the current fp32 weight; with_meta also (re)builds
        the E tiles from the pattern indices."""
        w_hi, w_lo = split_bf16(w.float())
        (compress_with_meta if with_meta else compress_values)(w_hi, self.hi)
        compress_values(w_lo, self.lo)


@dataclass
class DenseSplitOperand:
    """A dense fp32 weight as hi = bf16(W) and lo = bf16(W - hi) (the fp32 mode's masks=None
    route): products on the dense tcgen05 GEMM with fp32 output."""

    hi: torch.Tensor
    lo: torch.Tensor
    idx = None

    @property
    def rows(self) -> int:
        return self.hi.shape[0]

    @property
    def cols(self) -> int:
        return self.hi.shape[1]

    @classmethod
    def of(cls, w: torch.Tensor) -> "DenseSplitOperand":
        return cls(*split_bf16(w.float()))


def _split_spmm(op, bwd: bool, b_hi: torch.Tensor, b_lo: torch.Tensor, b_mn: bool, n: int,
                out: torch.Tensor, tag: str) -> None:
    """out[m, n] fp32 = W~ (or W~^T) . B^T as hi.hi + hi.lo + lo.hi (fixed order): the 2:4 GEMM
    on a SplitOperand, the dense one on a DenseSplitOperand."""
    m, k = (op.cols, op.rows) if bwd else (op.rows, op.cols)
    for i, (a_op, b) in enumerate(((op.hi, b_hi), (op.hi, b_lo), (op.lo, b_hi))):
        if isinstance(op, DenseSplitOperand):
            gemm_dw(a_op, bwd, b, b_mn, m, n, k, out, tag=tag, accumulate=i > 0)
        else:
            spmm_dw(a_op.bwd_vals if bwd else a_op.fwd_vals, a_op.bwd_e if bwd else a_op.fwd_e, m, k, b, b_mn, n,
                    out, tag=tag, accumulate=i > 0)


def _split_dw(a_hi, a_lo, a_mn, b_hi, b_lo, b_mn, m, n, k, out, w=None, idx=None, lam=0.0, tag="k5_gemm_dw"):
    for i, (a, b) in enumerate(((a_hi, b_hi), (a_hi, b_lo), (a_lo, b_hi))):
        gemm_dw(a, a_mn, b, b_mn, m, n, k, out, w if i == 0 else None, idx if i == 0 else None,
                lam if i == 0 else 0.0, tag=tag, accumulate=i > 0)


@dataclass
class FwdStateF32:
    x_hi: torch.Tensor  # (N, d) bf16, token-major
    x_lo: torch.Tensor
    zt: torch.Tensor  # (r_in, N) fp32 feature-major pre-activation (bias added)
    at: torch.Tensor  # (d_ff, N) fp32
    a_hi: torch.Tensor  # (d_ff, N) bf16
    a_lo: torch.Tensor
    yt: torch.Tensor  # (d, N) fp32


def ffn_forward_f32(x: torch.Tensor, w_in: SplitOperand, bias_in: torch.Tensor | None, w2: SplitOperand,
                    act: str) -> FwdStateF32:
    """fp32 mode forward (gated_ffn.py:293-297 on the float32 type): every product is three bf16
    2:4 products with fp32 accumulation; activations feature-major fp32."""
    n, d = x.shape
    r_in, d_ff = w_in.rows, w2.cols
    if w_in.cols != d or w2.rows != d or (r_in != (2 * d_ff if act in GATED else d_ff)):
        raise ShapeError("layer weight shapes are inconsistent with the activation / input width")
    if n % 128:
        raise ShapeError(f"the fp32 mode needs a token count divisible by 128, got {n}")
    dev = x.device
    x_hi, x_lo = split_bf16(x.float())
    zt = torch.empty((r_in, n), dtype=torch.float32, device=dev)
    _split_spmm(w_in, False, x_hi, x_lo, False, n, zt, "k3_spmm_fwd_in")
    at = torch.empty((d_ff, n), dtype=torch.float32, device=dev)
    a_hi = torch.empty((d_ff, n), dtype=torch.bfloat16, device=dev)
    a_lo = torch.empty_like(a_hi)
    b = None if bias_in is None else bias_in.float().contiguous()
    with TIMER("k6_act_fwd"):
        C.call("s24_act_fwd_f32", zt.data_ptr(), n, C.ptr(b), d_ff, n, ACT_CODES[act], at.data_ptr(), n,
               a_hi.data_ptr(), a_lo.data_ptr(), C.stream_of(zt))
    yt = torch.empty((d, n), dtype=torch.float32, device=dev)
    _split_spmm(w2, False, a_hi, a_lo, True, n, yt, "k3_spmm_fwd_out")
    return FwdStateF32(x_hi, x_lo, zt, at, a_hi, a_lo, yt)


@dataclass
class GradsF32:
    dxt: torch.Tensor  # (d, N) fp32 feature-major
    dw_in: torch.Tensor  # (r_in, d) fp32
    dbias_in: torch.Tensor  # (r_in,) fp32
    dw2: torch.Tensor  # (d, d_ff) fp32


def ffn_backward_f32(st: FwdStateF32, dy: torch.Tensor, w_in: SplitOperand, w2: SplitOperand, act: str,
                     w_in_dense: torch.Tensor | None = None, w2_dense: torch.Tensor | None = None,
                     lam: float = 0.0) -> GradsF32:
    """fp32 mode backward (gated_ffn.py:327-356, mvue=False): dA, the activation backward with
    the bias gradient, dX, and the dense dW GEMMs with the masked decay, all as split products."""
    d, n = st.yt.shape
    r_in, d_ff = w_in.rows, w2.cols
    if tuple(dy.shape) != (n, d):
        raise ShapeError(f"upstream shape {tuple(dy.shape)} != output shape {(n, d)}")
    dev = dy.device
    dy_hi, dy_lo = split_bf16(dy.float())
    dat = torch.empty((d_ff, n), dtype=torch.float32, device=dev)
    _split_spmm(w2, True, dy_hi, dy_lo, False, n, dat, "k4_spmm_bwd_out")
    dz_hi = torch.empty((r_in, n), dtype=torch.bfloat16, device=dev)
    dz_lo = torch.empty_like(dz_hi)
    dbias = torch.empty(r_in, dtype=torch.float32, device=dev)
    with TIMER("k7_act_bwd"):
        C.call("s24_act_bwd_f32", st.zt.data_ptr(), n, dat.data_ptr(), n, d_ff, n, ACT_CODES[act], None, n,
               dz_hi.data_ptr(), dz_lo.data_ptr(), dbias.data_ptr(), C.stream_of(dat))
    dw2 = torch.empty((d, d_ff), dtype=torch.float32, device=dev)
    _split_dw(dy_hi, dy_lo, True, st.a_hi, st.a_lo, False, d, d_ff, n, dw2, w2_dense, w2.idx, lam, "k5_gemm_dw2")
    dw_in = torch.empty((r_in, d), dtype=torch.float32, device=dev)
    _split_dw(dz_hi, dz_lo, False, st.x_hi, st.x_lo, True, r_in, d, n, dw_in, w_in_dense, w_in.idx, lam,
              "k5_gemm_dw_in")
    dxt = torch.empty((d, n), dtype=torch.float32, device=dev)
    _split_spmm(w_in, True, dz_hi, dz_lo, True, n, dxt, "k4_spmm_bwd_in")
    return GradsF32(dxt, dw_in, dbias, dw2)
