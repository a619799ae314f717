"""Masked decay, the fused Adam step and mask-flip statistics (optim.py:51-192 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch

from . import _capi as C
from .matrix import ShapeError
from .sparsity import TransposableMask


class DecayMode(Enum):
    NONE = "none"
    ON_WEIGHTS = "on_weights"
    ON_GRADIENTS = "on_gradients"


@dataclass
class DecayConfig:
    """optim.py:51-61: lambda_w, mode, refresh_period (mask search every l steps)."""

    lambda_w: float = 0.0
    mode: DecayMode = DecayMode.NONE
    refresh_period: int = 40

    def __post_init__(self) -> None:
        if self.lambda_w < 0:
            raise ValueError("lambda_w must be nonnegative")
        if self.refresh_period < 1:
            raise ValueError("refresh_period must be >= 1")


def masked_decay_gradient(g: torch.Tensor, w: torch.Tensor, m, lambda_w: float) -> torch.Tensor:
    """g + lambda_w * (1 - m) * w (optim.py:105-114), computed by the
    s24_masked_decay kernel on an fp32 copy of g.  `m` is a TransposableMask
    (the hot-path form; the fused dW epilogue does the same in the GEMM) or a
    0/1 tensor of w's shape."""
    C.require_cuda(g, w)
    if isinstance(m, TransposableMask):
        if m.shape != tuple(g.shape) or tuple(w.shape) != tuple(g.shape):
            raise ShapeError("gradient, weights and mask must have equal shapes")
        out = g.to(torch.float32).contiguous().clone()
        wc = w.contiguous()
        C.call("s24_masked_decay", out.data_ptr(), wc.data_ptr(), C.dtype_code(wc), m.idx.data_ptr(),
               g.shape[0], g.shape[1], float(lambda_w), C.stream_of(out))
        return out
    m = torch.as_tensor(m, device=g.device)
    if not (g.shape == w.shape == m.shape):
        raise ShapeError("gradient, weights and mask must have equal shapes")
    out = g.to(torch.float32).contiguous().clone()
    wc = w.contiguous()
    mb = (m != 0).to(torch.uint8).contiguous()
    C.call("s24_masked_decay_bits", out.data_ptr(), wc.data_ptr(), C.dtype_code(wc), mb.data_ptr(), out.numel(),
           float(lambda_w), C.stream_of(out))
    return out


def srste_weight_decay(w_next_base: torch.Tensor, w: torch.Tensor, m, lr: float, lambda_w: float) -> torch.Tensor:
    """w_next_base - lr lambda_w (1 - m) w (optim.py:117-125): the decay at the update site.
    Same kernel as masked_decay_gradient with the coefficient -lr lambda_w (fp32 result);
    the training step fuses it into the Adam kernel (DecayMode.ON_WEIGHTS)."""
    return masked_decay_gradient(w_next_base, w, m, -lr * lambda_w)


# ---------------------------------------------------------------------------
# optimizer step and mask statistics, one fused kernel each


@dataclass
class OptimizerState:
    """Adam state of one parameter (optim.py:64-86), device tensors.  w, u, v share a
    dtype: float64 reproduces the reference bit for bit, float32 is the fp32-master-weight
    training path."""

    w: torch.Tensor
    u: torch.Tensor
    v: torch.Tensor
    t: int = 0
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def init(cls, w: torch.Tensor, lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
             eps: float = 1e-8, dtype: torch.dtype | None = None) -> "OptimizerState":
        w = w.detach().to(dtype or (w.dtype if w.dtype in (torch.float32, torch.float64) else torch.float32))
        w = w.contiguous().clone()
        return cls(w=w, u=torch.zeros_like(w), v=torch.zeros_like(w), t=0, lr=lr, beta1=beta1, beta2=beta2,
                   eps=eps)


_DECAY_CODE = {DecayMode.NONE: 0, DecayMode.ON_GRADIENTS: 1, DecayMode.ON_WEIGHTS: 2}


def adam_step(state: OptimizerState, g: torch.Tensor, mask: TransposableMask | None = None,
              decay: DecayConfig | None = None, compress_into=None) -> OptimizerState:
    """One Adam update in place (optim.py:128-147), fused with the masked decay of the
    training loop when `decay` asks for it (trainer.py:438-447): ON_GRADIENTS adds
    lambda_w (1 - m) w to g first (masked_decay_gradient, optim.py:105-114), ON_WEIGHTS
    subtracts lr lambda_w (1 - m) w_before after the step (srste_weight_decay,
    optim.py:117-125).  One HBM pass over w, g, u, v (s24_adam_step).

    compress_into (an engine.CompressedOperand of this weight, fp32 state): the same update
    fused with the next forward's per-step compression (s24_adam_compress) -- the updated
    weight's kept values land in both orientations of the operand under its cached mask, which
    also supplies the decay mask, so the next step needs no K2 launch."""
    C.require_cuda(state.w, state.u, state.v, g)
    if compress_into is not None:
        return _adam_compress(state, g, decay, compress_into)
    if tuple(g.shape) != tuple(state.w.shape):
        raise ShapeError("gradient shape differs from weights")
    mode = decay.mode if (decay is not None and decay.lambda_w > 0) else DecayMode.NONE
    if mode is not DecayMode.NONE and mask is None:
        raise ValueError("masked decay needs the weight's TransposableMask")
    if mask is not None and mask.shape != tuple(state.w.shape):
        raise ShapeError("mask shape differs from weights")
    for t_ in (state.w, state.u, state.v):
        if not t_.is_contiguous() or t_.dtype != state.w.dtype:
            raise ValueError("w, u, v must be contiguous tensors of one dtype")
    g = g.contiguous()
    if g.dtype not in (torch.float32, state.w.dtype):
        g = g.to(state.w.dtype)
    state.t += 1
    t = state.t
    lam = decay.lambda_w if mode is not DecayMode.NONE else 0.0
    rows, cols = (state.w.shape if state.w.dim() == 2 else (1, state.w.numel()))
    # the scalars exactly as the reference's Python evaluates them
    C.call("s24_adam_step", state.w.data_ptr(), state.u.data_ptr(), state.v.data_ptr(), C.dtype_code(state.w),
           g.data_ptr(), C.dtype_code(g), rows, cols, mask.idx.data_ptr() if mode is not DecayMode.NONE else None,
           state.lr, state.beta1, state.beta2, state.eps, 1.0 - state.beta1, 1.0 - state.beta2,
           1.0 - state.beta1 ** t, 1.0 - state.beta2 ** t, lam, state.lr * lam, _DECAY_CODE[mode],
           C.stream_of(state.w))
    return state


def _adam_compress(state: OptimizerState, g: torch.Tensor, decay: DecayConfig | None, op) -> OptimizerState:
    if state.w.dtype != torch.float32 or state.w.dim() != 2 or tuple(state.w.shape) != (op.rows, op.cols):
        raise ShapeError("the fused optimizer + compression takes the fp32 2-D weight of its operand")
    for t_ in (state.w, state.u, state.v):
        if not t_.is_contiguous() or t_.dtype != torch.float32:
            raise ValueError("w, u, v must be contiguous fp32 tensors")
    g = g.contiguous()
    if g.dtype != torch.float32 or tuple(g.shape) != tuple(state.w.shape):
        raise ShapeError("the fused path takes an fp32 gradient of the weight's shape")
    mode = decay.mode if (decay is not None and decay.lambda_w > 0) else DecayMode.NONE
    lam = decay.lambda_w if mode is not DecayMode.NONE else 0.0
    state.t += 1
    t = state.t
    C.call("s24_adam_compress", state.w.data_ptr(), state.u.data_ptr(), state.v.data_ptr(), g.data_ptr(), op.rows,
           op.cols, op.idx.data_ptr(), state.lr, state.beta1, state.beta2, state.eps, 1.0 - state.beta1,
           1.0 - state.beta2, 1.0 - state.beta1 ** t, 1.0 - state.beta2 ** t, lam, state.lr * lam, _DECAY_CODE[mode],
           op.fwd_vals.data_ptr(), op.bwd_vals.data_ptr(), op.perm_ff, C.stream_of(state.w))
    return state


def mask_flips(m_prev: TransposableMask, m_curr: TransposableMask,
               block_flips: torch.Tensor | None = None) -> torch.Tensor:
    """Number of mask bits that differ between two transposable masks (device int64
    scalar); adds each 4x4 block's count to `block_flips` (int32, rows/4 x cols/4) when
    given -- the cumulative per-block flips of block_flip_stats (optim.py:164-192)."""
    if m_prev.shape != m_curr.shape:
        raise ShapeError(f"mask shapes differ: {m_prev.shape} vs {m_curr.shape}")
    C.require_cuda(m_prev.idx, m_curr.idx)
    if m_prev._raw is not None or m_curr._raw is not None:
        # masks given as arbitrary 0/1 bits (e.g. a reference-style mask_fn): count the changed
        # bits per 4x4 block from the bits themselves, not from pattern indices
        rows, cols = m_prev.shape
        diff = (m_prev.bits != m_curr.bits).to(torch.int32)
        per = diff.reshape(rows // 4, 4, cols // 4, 4).sum(dim=(1, 3)).reshape(-1)
        if block_flips is not None:
            if block_flips.dtype != torch.int32 or block_flips.numel() != per.numel():
                raise ShapeError("block_flips must be int32 with one entry per 4x4 block")
            block_flips.view(-1).add_(per)
        return per.sum(dtype=torch.int64)
    out = torch.zeros(1, dtype=torch.int64, device=m_prev.idx.device)
    if block_flips is not None and (block_flips.dtype != torch.int32 or block_flips.numel() != m_prev.idx.numel()):
        raise ShapeError("block_flips must be int32 with one entry per 4x4 block")
    C.call("s24_mask_flips", m_prev.idx.data_ptr(), m_curr.idx.data_ptr(), m_prev.idx.numel(), out.data_ptr(),
           C.ptr(block_flips), C.stream_of(out))
    return out[0]


def flip_rate(m_prev: TransposableMask, m_curr: TransposableMask, d: int | None = None) -> float:
    """Fraction of mask bits that changed, ||m_curr - m_prev||_1 / d (optim.py:94-102)."""
    n = mask_flips(m_prev, m_curr)
    if d is None:
        d = m_prev.shape[0] * m_prev.shape[1]
    return float(n.item()) / d


@dataclass
class FlipTrace:
    """Per-step flip rates plus per-block oscillation statistics (optim.py:85-91)."""

    rates: torch.Tensor | None = None
    block_flips: torch.Tensor | None = None  # cumulative flips per 4x4 block, int64, block order
    block_gaps: torch.Tensor | None = None  # best minus second-best pattern score, float64


def block_flip_stats(w_history, table=None, mask_fn=None) -> FlipTrace:
    """Cumulative mask flips and retained-L1 gap per 4x4 block (optim.py:164-192) on the GPU.

    Flips: K1 search of every snapshot (or `mask_fn(w)` -> 0/1 bits as in the reference, or a
    TransposableMask) and the
    per-block changed-bit counts of consecutive masks (s24_mask_flips).  Gaps: best minus
    second-best of the 90 float64 pattern scores on the final snapshot (s24_block_gaps),
    bit-exact with the reference.  `table` is accepted for signature compatibility (only
    the canonical table is supported)."""
    from .sparsity import transposable_search_conv

    snaps = list(w_history)
    if len(snaps) < 2:
        raise ShapeError("need at least two weight snapshots")
    if mask_fn is None:
        mask_fn = transposable_search_conv
    last = snaps[-1]
    if last.dim() != 2:
        raise ShapeError(f"expected 2-D snapshots, got ndim={last.dim()}")
    C.require_cuda(last)
    rows, cols = last.shape
    if rows % 4 or cols % 4:
        raise ShapeError(f"shape {(rows, cols)} not divisible into 4x4 blocks")
    nb = (rows // 4) * (cols // 4)
    counts = torch.zeros(nb, dtype=torch.int32, device=last.device)
    def as_mask(m):
        # the reference's mask_fn returns a 0/1 bits array (optim.py:176-177); ours may also
        # return a TransposableMask
        if isinstance(m, TransposableMask):
            return m
        bits = torch.as_tensor(m, device=last.device)
        return TransposableMask(bits=bits)

    prev = as_mask(mask_fn(snaps[0]))
    for w in snaps[1:]:
        if tuple(w.shape) != (rows, cols):
            raise ShapeError("snapshots differ in shape")
        curr = as_mask(mask_fn(w))
        mask_flips(prev, curr, counts)
        prev = curr
    last = last.contiguous()
    gaps = torch.empty(nb, dtype=torch.float64, device=last.device)
    C.call("s24_block_gaps", last.data_ptr(), C.dtype_code(last), rows, cols, gaps.data_ptr(), C.stream_of(last))
    return FlipTrace(rates=torch.zeros(0, dtype=torch.float64), block_flips=counts.to(torch.int64), block_gaps=gaps)


# ---------------------------------------------------------------------------
# decay factor determination (optim.py:195-259): host control logic over GPU warm-up runs

FEASIBLE_MU_BAND = (0.60, 0.95)  # optim.py:38
DEFAULT_LAMBDA_GRID = (1e-6, 2e-6, 6e-6, 2e-5, 6e-5, 2e-4, 6e-4, 2e-3)  # optim.py:42


@dataclass
class SearchEntry:
    lambda_w: float
    mu: float
    feasible: bool
    accuracy_risk: bool  # mu >= 1: flips not inhibited below the dense rate


@dataclass
class SearchResult:
    chosen: float | None
    entries: list
    dense_reference: float

    def to_csv(self) -> str:
        lines = ["lambda,mu,feasible"]
        for e in self.entries:
            lines.append(f"{e.lambda_w:g},{e.mu:.6g},{str(e.feasible).lower()}")
        return "\n".join(lines) + "\n"


def decay_factor_search(candidates, warmup_steps: int, run_warmup, window_fraction: float = 0.10) -> SearchResult:
    """optim.py:220-259: mu = (mean sparse flip rate) / (mean dense-proxy flip rate) over the
    trailing window of the warm-up; the largest candidate inside FEASIBLE_MU_BAND wins.
    `run_warmup` is trainer.make_warmup_runner (GPU warm-up runs)."""
    import numpy as np

    if not candidates:
        raise ValueError("candidate list is empty")
    if warmup_steps < 1:
        raise ValueError("warmup_steps must be >= 1")
    window = max(1, int(round(window_fraction * warmup_steps)))
    dense_trace = np.asarray(run_warmup(None), dtype=np.float64)
    dense_ref = float(dense_trace[-window:].mean())
    entries = []
    lo, hi = FEASIBLE_MU_BAND
    for lam in candidates:
        trace = np.asarray(run_warmup(float(lam)), dtype=np.float64)
        sparse_rate = float(trace[-window:].mean())
        mu = sparse_rate / dense_ref if dense_ref > 0 else float("inf")
        entries.append(SearchEntry(lambda_w=float(lam), mu=mu, feasible=bool(lo <= mu <= hi),
                                   accuracy_risk=bool(mu >= 1.0)))
    feasible = [e.lambda_w for e in entries if e.feasible]
    return SearchResult(chosen=max(feasible) if feasible else None, entries=entries, dense_reference=dense_ref)
