"""CPU oracle for the 2:4 FFN hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy (float64, fixed accumulation order), the
reference `sparse24` algorithms that the B200 path replaces.  It is the checker
for the CUDA path: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product package (`paper_2404_01847_b200`) never imports it and has no CPU
fallback.

Parity is pinned (see tests/test_oracle_golden.py):
  * the pattern table against the reference golden file (md5 313a02e7...);
  * mask search, compress, FST forward/backward and masked decay against
    golden vectors produced by the reference package itself
    (tests/golden/make_golden.py, committed .npz fixtures).
SwiGLU is NOT in the reference (`gated_ffn.py:47-50`); the `silu_gate` rows
below are a restatement of GEGLU with silu substituted -- parity unpinned.

Where the compiled reference kernels are available (oracle/_ref/_core*.so,
built by oracle/Makefile from /root/reference/pkg/src/sparse24/_core.pyx),
`ref_kernels()` returns that module so the CPU baseline can time the
reference's own compiled loops.

Reference citations are to /root/reference/pkg/src/sparse24/<file>:<line>.
"""

from __future__ import annotations

import glob
import importlib.util
import itertools
import math
import os
from dataclasses import dataclass

import numpy as np

try:  # scipy is the reference's erf (gated_ffn.py:23, _core_py.py:12)
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover - scipy is present in this image
    _erf = np.vectorize(math.erf)

RSQRT2 = 0.7071067811865476  # _core.pyx:19, gated_ffn.py:43
RSQRT2PI = 0.3989422804014327  # gated_ffn.py:44


# ---------------------------------------------------------------------------
# errors (matrix.py:11-16)


class ShapeError(ValueError):
    """Operand shapes violate an operation's preconditions (matrix.py:11)."""


class FormatError(ValueError):
    """A mask / compressed buffer violates its invariants (matrix.py:15)."""


# ---------------------------------------------------------------------------
# the 90 transposable 4x4 patterns (sparsity.py:203-222)


def _row_choices():
    # every 4-bit row with exactly two ones, as tuples
    return [r for r in itertools.product((0, 1), repeat=4) if sum(r) == 2]


def pattern_table() -> tuple[np.ndarray, np.ndarray]:
    """(patterns (90,4,4) uint8, positions (90,8) int32).

    Canonical order = ascending lexicographic order of the row-major 16-bit
    tuples (sparsity.py:210-216); positions = kept flat indices ascending
    (sparsity.py:203-205).
    """
    rows = _row_choices()
    found = []
    for r0, r1, r2, r3 in itertools.product(rows, repeat=4):
        colsum = [r0[j] + r1[j] + r2[j] + r3[j] for j in range(4)]
        if colsum == [2, 2, 2, 2]:
            found.append(r0 + r1 + r2 + r3)
    found.sort()
    pats = np.array(found, dtype=np.uint8).reshape(-1, 4, 4)
    pos = np.array([np.flatnonzero(p.reshape(16)) for p in pats], dtype=np.int32)
    return pats, pos


def pattern_text(pats: np.ndarray) -> str:
    """Text form: one 16-char line per pattern (sparsity.py:180-182)."""
    return "".join("".join(str(int(b)) for b in p.reshape(16)) + "\n" for p in pats)


# ---------------------------------------------------------------------------
# 4x4 block tiling (sparsity.py:65-79)


def blocks16(arr: np.ndarray) -> np.ndarray:
    r, c = arr.shape
    if r % 4 or c % 4:
        raise ShapeError(f"shape {arr.shape} not divisible into 4x4 blocks")
    return np.ascontiguousarray(arr.reshape(r // 4, 4, c // 4, 4).swapaxes(1, 2).reshape(-1, 16))


def unblocks16(b16: np.ndarray, shape) -> np.ndarray:
    r, c = shape
    return np.ascontiguousarray(b16.reshape(r // 4, c // 4, 4, 4).swapaxes(1, 2).reshape(r, c))


# ---------------------------------------------------------------------------
# transposable mask search (sparsity.py:258-271; kernel _core.pyx:83-110)


def pattern_scores(absblocks: np.ndarray, positions: np.ndarray):
    """score[b,t] = sum of |w| over the 8 kept positions, accumulated
    strictly ascending in position (_core.pyx:102-105); best = first argmax
    (strict '>' so ties keep the lowest pattern index, _core.pyx:106)."""
    absblocks = np.asarray(absblocks, dtype=np.float64)
    nb = absblocks.shape[0]
    scores = np.empty((nb, positions.shape[0]), dtype=np.float64)
    for t in range(positions.shape[0]):
        acc = absblocks[:, positions[t, 0]].copy()
        for p in positions[t, 1:]:
            acc = acc + absblocks[:, p]
        scores[:, t] = acc
    # np.argmax returns the first maximum == sequential strict '>' scan
    return scores, np.argmax(scores, axis=1).astype(np.int64)


def search_pattern_idx(w: np.ndarray) -> np.ndarray:
    """Per-block canonical pattern index, shape (rows/4, cols/4) uint8."""
    arr = np.asarray(w, dtype=np.float64)  # sparsity.py:265 casts to f64
    _, pos = pattern_table()
    _, best = pattern_scores(np.abs(blocks16(arr)), pos)
    r, c = arr.shape
    return best.astype(np.uint8).reshape(r // 4, c // 4)


def idx_to_bits(idx: np.ndarray) -> np.ndarray:
    """Expand per-block pattern indices to the full 0/1 mask (sparsity.py:270-271)."""
    pats, _ = pattern_table()
    nbr, nbc = idx.shape
    return unblocks16(pats.reshape(90, 16)[idx.reshape(-1)], (4 * nbr, 4 * nbc))


def transposable_search_conv(w: np.ndarray) -> np.ndarray:
    """Full mask bits (uint8, same shape as w)."""
    return idx_to_bits(search_pattern_idx(w))


def validate_transposable(bits: np.ndarray) -> None:
    """TransposableMask.validate (sparsity.py:122-131)."""
    bits = np.asarray(bits)
    if bits.ndim != 2:
        raise FormatError("mask must be 2-D")
    b = blocks16(bits).reshape(-1, 4, 4)
    if bits.size and bits.max() > 1:
        raise FormatError("mask bits must be 0/1")
    if not (b.sum(axis=(1, 2)) == 8).all():
        raise FormatError("every 4x4 block must contain exactly 8 ones")
    if not (b.sum(axis=2) == 2).all() or not (b.sum(axis=1) == 2).all():
        raise FormatError("every block row and column must contain exactly 2 ones")


# ---------------------------------------------------------------------------
# packed 2:4 format (spmm.py:38-147, compress at :92-106)


def compress_rowwise(values: np.ndarray, bits: np.ndarray):
    """Row-wise groups of 4 (row-major group order): kept values (m, k/2) and
    one meta nibble per group (m, k/4) = i0 | i1 << 2 with i0 < i1
    (spmm.py:98-104).  `values` is copied verbatim (f64 here)."""
    m, k = bits.shape
    if k % 4:
        raise ShapeError(f"cols={k} not divisible by 4 for row-wise groups")
    g = np.asarray(bits, dtype=np.uint8).reshape(m, k // 4, 4)
    if not (g.sum(axis=2) == 2).all() or (g.size and g.max() > 1):
        raise FormatError("every group of 4 must contain exactly 2 ones")
    i0 = np.argmax(g, axis=2)  # first set bit
    i1 = 3 - np.argmax(g[:, :, ::-1], axis=2)  # last set bit
    v = np.asarray(values).reshape(m, k // 4, 4)
    r_ix = np.arange(m)[:, None]
    c_ix = np.arange(k // 4)[None, :]
    kept = np.stack([v[r_ix, c_ix, i0], v[r_ix, c_ix, i1]], axis=2).reshape(m, k // 2)
    meta = (i0 | (i1 << 2)).astype(np.uint8)
    return kept, meta


def decompress_rowwise(kept: np.ndarray, meta: np.ndarray, k: int) -> np.ndarray:
    """Inverse of compress_rowwise; rejects non-ascending meta (spmm.py:61-67)."""
    m = kept.shape[0]
    i0 = (meta & 3).astype(np.int64)
    i1 = ((meta >> 2) & 3).astype(np.int64)
    if not (i0 < i1).all():
        raise FormatError("metadata indices must be distinct and ascending")
    out = np.zeros((m, k // 4, 4), dtype=np.asarray(kept).dtype)
    kv = np.asarray(kept).reshape(m, k // 4, 2)
    r_ix = np.arange(m)[:, None]
    c_ix = np.arange(k // 4)[None, :]
    out[r_ix, c_ix, i0] = kv[:, :, 0]
    out[r_ix, c_ix, i1] = kv[:, :, 1]
    return out.reshape(m, k)


def compress_groups(values: np.ndarray, bits: np.ndarray, colwise: bool):
    """compress (spmm.py:92-106) in either direction: column-wise groups (column-major group
    order, to_groups sparsity.py:45-54) are the row-wise groups of the transpose.  Returns the
    flat (values, meta) buffers of Compressed24."""
    v, b = (np.ascontiguousarray(values.T), np.ascontiguousarray(bits.T)) if colwise else (values, bits)
    kept, meta = compress_rowwise(v, b)
    return kept.reshape(-1), meta.reshape(-1)


def decompress_groups(values: np.ndarray, meta: np.ndarray, shape, colwise: bool) -> np.ndarray:
    """decompress (spmm.py:117-129) of flat buffers in either direction."""
    rows, cols = shape
    lead, grouped = (cols, rows) if colwise else (rows, cols)
    out = decompress_rowwise(np.asarray(values).reshape(lead, grouped // 2),
                             np.asarray(meta).reshape(lead, grouped // 4), grouped)
    return np.ascontiguousarray(out.T) if colwise else out


def mvue_prune(g: np.ndarray, colwise: bool, rng_seed: int):
    """mvue_prune (sparsity.py:379-398): (dense float64 estimate, 0/1 mask)."""
    arr = np.asarray(g, dtype=np.float64)
    src = np.ascontiguousarray(arr.T) if colwise else arr
    values, kept, _ = mvue_kept(src.reshape(-1, 4), rng_seed)
    out = np.zeros((src.size // 4, 4))
    bits = np.zeros((src.size // 4, 4), dtype=np.uint8)
    rows = np.arange(src.size // 4)
    for slot in (0, 1):
        out[rows, kept[:, slot]] = values[:, slot]
        bits[rows, kept[:, slot]] = 1
    out, bits = out.reshape(src.shape), bits.reshape(src.shape)
    if colwise:
        return np.ascontiguousarray(out.T), np.ascontiguousarray(bits.T)
    return out, bits


# ---------------------------------------------------------------------------
# gather plan + column-wise sparse product (gated_ffn.py:131-162, _core.pyx:63-80)


def gather_plan(bits: np.ndarray, transposed_source: bool):
    """(take, pos_t): flat source indices of kept entries per row of `bits`
    (slots ascending), and their contraction positions transposed
    (gated_ffn.py:142-157)."""
    m, k = bits.shape
    g = np.asarray(bits, dtype=np.int64).reshape(m, k // 4, 4)
    i0 = np.argmax(g, axis=2)
    i1 = 3 - np.argmax(g[:, :, ::-1], axis=2)
    base = 4 * np.arange(k // 4, dtype=np.int64)[None, :]
    cols = np.empty((m, k // 2), dtype=np.int64)
    cols[:, 0::2] = i0 + base
    cols[:, 1::2] = i1 + base
    take = np.arange(m, dtype=np.int64)[:, None] * k + cols
    if transposed_source:
        take = (take % k) * m + take // k
    return take, np.ascontiguousarray(cols.T)


def spmm_colwise(a: np.ndarray, values: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """C = A @ B, B column-wise 2:4 as (values, absolute row positions) of
    shape (s, n); each output cell accumulates over kept k ascending, no FMA
    (_core.pyx:63-80, _core_py.py:41-48).  Output column-major."""
    a = np.asarray(a, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    out = np.zeros((a.shape[0], values.shape[1]), dtype=np.float64, order="F")
    for t in range(values.shape[0]):
        out += a[:, pos[t, :]] * values[t : t + 1, :]
    return out


def plan_product(a: np.ndarray, w_source: np.ndarray, bits: np.ndarray, transposed_source: bool):
    """a @ (masked weight).T via the gather plan (gated_ffn.py:159-162)."""
    take, pos_t = gather_plan(bits, transposed_source)
    vals = np.ascontiguousarray(w_source, dtype=np.float64).ravel()[take]
    return spmm_colwise(a, vals.T, pos_t)


# ---------------------------------------------------------------------------
# activations (gated_ffn.py:58-70, _core.pyx:222-250)


def gelu(x):
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + _erf(x * RSQRT2))


def gelu_grad(x):
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * (1.0 + _erf(x * RSQRT2)) + x * (RSQRT2PI * np.exp(-0.5 * x * x))


def silu(x):  # SwiGLU extension: NOT in the reference (parity unpinned)
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def silu_grad(x):  # SwiGLU extension: NOT in the reference (parity unpinned)
    x = np.asarray(x, dtype=np.float64)
    s = 1.0 / (1.0 + np.exp(-x))
    return s * (1.0 + x * (1.0 - s))


def gate(z1, z2, act: str = "geglu"):
    """gate_gelu (_core.pyx:222-250): act(z1) * z2, column-major result."""
    f = gelu if act == "geglu" else silu
    return np.asfortranarray(f(z1) * np.asarray(z2, dtype=np.float64))


# ---------------------------------------------------------------------------
# fully sparse FFN layer (gated_ffn.py:273-373), mvue=False branch


@dataclass
class Layer:
    """Mirror of FFNLayer (gated_ffn.py:77-128).  `act` is 'gelu', 'relu',
    'geglu' or 'swiglu' (the last is the unpinned extension).  For gated
    layers w_in = [u; v] (r_in = 2 d_ff) and bias_in = [b; c]."""

    w_in: np.ndarray  # (r_in, d)
    bias_in: np.ndarray  # (r_in,)
    w2: np.ndarray  # (d, d_ff)
    act: str

    @property
    def gated(self) -> bool:
        return self.act in ("geglu", "swiglu")

    @property
    def d_ff(self) -> int:
        return self.w2.shape[1]


def _activate(layer: Layer, z: np.ndarray) -> np.ndarray:
    r = layer.d_ff
    if layer.gated:
        return gate(z[:, :r], z[:, r:], layer.act)
    if layer.act == "gelu":
        return gelu(z)
    return np.maximum(z, 0.0)


def fst_forward(layer: Layer, x: np.ndarray, mask_in, mask_out, exact: bool = True):
    """Returns dict(z, a, y).  masks None -> dense path (gated_ffn.py:286-289).
    exact=True runs the reference's gather + ascending spmm route
    (gated_ffn.py:293-297); exact=False uses BLAS on the masked dense weight,
    equal to the exact route within 1e-12 (the reference's own check,
    test_gated_ffn.py:173-179) and fast enough for large parity cases."""
    x = np.asarray(x, dtype=np.float64)
    w_in = np.asarray(layer.w_in, dtype=np.float64)
    w2 = np.asarray(layer.w2, dtype=np.float64)
    if mask_in is None:
        z = x @ w_in.T + layer.bias_in
        a = _activate(layer, z)
        y = a @ w2.T
    else:
        if mask_in.shape != w_in.shape or mask_out.shape != w2.shape:
            raise ShapeError("mask shapes do not match layer weights")
        if exact:
            z = plan_product(x, w_in, mask_in, False)
            z += layer.bias_in
            a = _activate(layer, z)
            y = plan_product(a, w2, mask_out, False)
        else:
            z = x @ (w_in * mask_in).T + layer.bias_in
            a = _activate(layer, z)
            y = a @ (w2 * mask_out).T
    return {"x": x, "z": z, "a": a, "y": y}


def fst_backward(layer: Layer, fwd: dict, dy: np.ndarray, mask_in, mask_out, exact: bool = True):
    """mvue=False backward (gated_ffn.py:304-373): dA via the transposed mask,
    dense dW, activation backward, dX via the transposed mask.  Returns
    dict(dx, dw_in, dbias_in, dw2, dz)."""
    dy = np.asarray(dy, dtype=np.float64)
    if dy.shape != fwd["y"].shape:
        raise ShapeError(f"upstream shape {dy.shape} != output shape {fwd['y'].shape}")
    w_in = np.asarray(layer.w_in, dtype=np.float64)
    w2 = np.asarray(layer.w2, dtype=np.float64)
    sparse = mask_in is not None
    if sparse and exact:
        da = plan_product(dy, w2, np.ascontiguousarray(mask_out.T), True)
    elif sparse:
        da = dy @ (w2 * mask_out)
    else:
        da = dy @ w2
    dw2 = dy.T @ fwd["a"]
    z = fwd["z"]
    r = layer.d_ff
    if layer.gated:
        z1, z2 = z[:, :r], z[:, r:]
        f, fp = (gelu, gelu_grad) if layer.act == "geglu" else (silu, silu_grad)
        g1 = da * z2 * fp(z1)
        g2 = da * f(z1)
        dz = np.concatenate([g1, g2], axis=1)
    elif layer.act == "gelu":
        dz = da * gelu_grad(z)
    else:
        dz = da * (z > 0)
    dbias = dz.sum(axis=0)
    if sparse and exact:
        dx = plan_product(dz, w_in, np.ascontiguousarray(mask_in.T), True)
    elif sparse:
        dx = dz @ (w_in * mask_in)
    else:
        dx = dz @ w_in
    dw_in = dz.T @ fwd["x"]
    return {"dx": dx, "dw_in": dw_in, "dbias_in": dbias, "dw2": dw2, "dz": dz, "da": da}


# ---------------------------------------------------------------------------
# optimizer pieces on the path (optim.py:105-114, trainer.py:111-119)


def masked_decay_gradient(g, w, m, lambda_w: float):
    g = np.asarray(g, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    m = np.asarray(m)
    if not (g.shape == w.shape == m.shape):
        raise ShapeError("gradient, weights and mask must have equal shapes")
    return g + lambda_w * ((1 - m) * w)


def switch_step(steps: int, dense_ft_fraction: float) -> int:
    return math.ceil(steps * (1.0 - dense_ft_fraction))


def flip_rate(m_prev, m_curr) -> float:  # optim.py:94-102
    a = np.asarray(m_prev).ravel().astype(np.int64)
    b = np.asarray(m_curr).ravel().astype(np.int64)
    return float(np.abs(b - a).sum()) / a.size


def greedy_masks(absblocks: np.ndarray) -> np.ndarray:
    """kernels.greedy_masks (_core.pyx:139-219) restated: (nb, 16) |w| -> (nb, 16) 0/1 masks.
    Scan cells by descending magnitude (lowest flat index on ties: a stable sort), pick while
    the block row and column hold < 2 picks; a 7-pick block takes the single swap with the
    largest (a[rdef,c2] + a[r2,cdef]) - a[r2,c2] (first best on ties)."""
    a_all = np.asarray(absblocks, dtype=np.float64)
    out = np.zeros(a_all.shape, dtype=np.uint8)
    for bi, a in enumerate(a_all):
        order = np.argsort(-a, kind="stable")
        rowc, colc, picked = [0] * 4, [0] * 4, np.zeros(16, dtype=np.uint8)
        for idx in order:
            r, c = idx >> 2, idx & 3
            if rowc[r] < 2 and colc[c] < 2:
                picked[idx] = 1
                rowc[r] += 1
                colc[c] += 1
        if picked.sum() == 7:
            rdef = max(i for i in range(4) if rowc[i] < 2)
            cdef = max(i for i in range(4) if colc[i] < 2)
            best = None
            for r2 in range(4):
                for c2 in range(4):
                    if r2 == rdef or c2 == cdef or not picked[r2 * 4 + c2]:
                        continue
                    gain = (a[rdef * 4 + c2] + a[r2 * 4 + cdef]) - a[r2 * 4 + c2]
                    if best is None or gain > best[0]:
                        best = (gain, r2, c2)
            _, br, bc = best
            picked[br * 4 + bc] = 0
            picked[rdef * 4 + bc] = 1
            picked[br * 4 + cdef] = 1
        if picked.sum() != 8:
            raise RuntimeError("greedy mask completion failed")
        out[bi] = picked
    return out


def transposable_search_greedy(w: np.ndarray) -> np.ndarray:  # sparsity.py:229-238
    arr = np.asarray(w, dtype=np.float64)
    return unblocks16(greedy_masks(np.abs(blocks16(arr))), arr.shape)


def prune_2of4_bits(w: np.ndarray, colwise: bool = False) -> np.ndarray:
    """prune_2of4 (sparsity.py:274-279; kernels.prune_2of4_keep _core.pyx:113-136): keep the
    two largest |w| per group of four consecutive columns (or rows); first max wins ties."""
    a = np.abs(np.asarray(w, dtype=np.float64))
    if colwise:
        a = a.T
    g = a.reshape(-1, 4)
    i1 = np.argmax(g, axis=1)  # first maximum
    g2 = g.copy()
    g2[np.arange(len(g)), i1] = -np.inf
    i2 = np.argmax(g2, axis=1)
    keep = np.zeros(g.shape, dtype=np.uint8)
    keep[np.arange(len(g)), i1] = 1
    keep[np.arange(len(g)), i2] = 1
    keep = keep.reshape(a.shape)
    return np.ascontiguousarray(keep.T) if colwise else keep


def adam_step(w, u, v, t: int, g, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """optim.py:128-147 restated in float64 with the reference's evaluation order; returns
    new (w, u, v) for step number t (1-based, already incremented)."""
    w, u, v = (np.array(a, dtype=np.float64) for a in (w, u, v))
    g = np.asarray(g, dtype=np.float64)
    u *= beta1
    u += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * (g * g)
    denom = np.sqrt(v / (1.0 - beta2 ** t))
    denom += eps
    denom *= 1.0 - beta1 ** t
    w -= lr * u / denom
    return w, u, v


def srste_weight_decay(w_next_base, w, m, lr: float, lambda_w: float):  # optim.py:117-125
    return np.asarray(w_next_base, dtype=np.float64) - lr * lambda_w * ((1 - np.asarray(m)) * np.asarray(w, dtype=np.float64))


def train_update(w, u, v, t: int, g, m, lambda_w: float, mode: str, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """trainer.py:438-447: masked decay on the gradient (mode 'on_gradients') or at the
    update site ('on_weights') around one Adam step."""
    if mode == "on_gradients" and lambda_w > 0:
        g = masked_decay_gradient(g, w, m, lambda_w)
    w_before = np.array(w, dtype=np.float64)
    w1, u1, v1 = adam_step(w, u, v, t, g, lr, beta1, beta2, eps)
    if mode == "on_weights" and lambda_w > 0:
        w1 = srste_weight_decay(w1, w_before, m, lr, lambda_w)
    return w1, u1, v1


def block_flips(m_prev, m_curr) -> np.ndarray:
    """Per-4x4-block count of changed mask bits (the flips of block_flip_stats, optim.py:164-192)."""
    a = blocks16(np.asarray(m_prev, dtype=np.int64))
    b = blocks16(np.asarray(m_curr, dtype=np.int64))
    return np.abs(b - a).sum(axis=1)


def block_gaps(w) -> np.ndarray:
    """Retained-L1 gap per 4x4 block of block_flip_stats (optim.py:186-190): best minus
    second-best pattern score (np.partition's multiset order: ties give 0), scores from
    pattern_scores on |w| in float64."""
    _, pos = pattern_table()
    scores, _ = pattern_scores(np.abs(blocks16(np.asarray(w, dtype=np.float64))), pos)
    top2 = -np.partition(-scores, 1, axis=1)[:, :2]
    return top2[:, 0] - top2[:, 1]


def block_flip_stats(w_history):
    """(block_flips int64, block_gaps float64) of block_flip_stats (optim.py:164-192) with
    the default conv search as the mask function."""
    if len(w_history) < 2:
        raise ShapeError("need at least two weight snapshots")
    masks = [transposable_search_conv(np.asarray(w, dtype=np.float64)) for w in w_history]
    flips = np.zeros(blocks16(masks[0]).shape[0], dtype=np.int64)
    for a, b in zip(masks, masks[1:]):
        flips += block_flips(a, b)
    return flips, block_gaps(w_history[-1])


# ---------------------------------------------------------------------------
# the reference's own compiled kernels (oracle/_ref), when built


def ref_kernels():
    """The reference's `_core` extension compiled by oracle/Makefile from
    /root/reference/pkg/src/sparse24/_core.pyx, or None when not built."""
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
    hits = glob.glob(os.path.join(here, "_core*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_core", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# deterministic synthetic data (integer-only, bit-reproducible on any host)

_M64 = (1 << 64) - 1


def _splitmix64(n: int, seed: int) -> np.ndarray:
    """n outputs of splitmix64 starting from `seed` (uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        x = (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(seed & _M64))
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def det_normal(shape, seed: int, scale_log2: int = 0) -> np.ndarray:
    """Approximately N(0, 2**scale_log2) float64 values built from an
    Irwin-Hall sum of 12 integer uniforms: exact integer arithmetic plus a
    power-of-two scale, so every host produces identical bits."""
    n = int(np.prod(shape))
    u = _splitmix64(12 * n, seed) >> np.uint64(44)  # 20-bit uniforms
    s = u.reshape(n, 12).astype(np.int64).sum(axis=1) - 6 * (1 << 20)
    return np.ldexp(s.astype(np.float64), scale_log2 - 20).reshape(shape)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bf16 (round-to-nearest-even via f32), back to f64."""
    f = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (f >> np.uint64(16)) & np.uint64(1)
    f = (f + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return f.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bf16 encoding of bf16-representable float64 values."""
    return (np.asarray(x, dtype=np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# MVUE: unbiased stochastic 2:4 sparsification along rows (sparsity.py:285-413)
# and the mvue=True weight gradient (gated_ffn.py:367-373).  Every array op is
# the reference's sequence of IEEE float64 operations (sums over a group of 4
# are sequential, as numpy reduces a (n, 4) C-contiguous array along axis 1).

MVUE_PAIRS = np.array([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], dtype=np.int64)


def mvue_inclusion_probs(groups: np.ndarray) -> np.ndarray:
    """pi_i = min(1, c |x_i|) with sum(pi) = 2 per group (sparsity.py:290-324)."""
    a = np.abs(np.asarray(groups, dtype=np.float64))
    total = ((a[:, 0] + a[:, 1]) + a[:, 2]) + a[:, 3]
    amax = a.max(axis=1)
    fm = np.arange(4)[None, :] == a.argmax(axis=1)[:, None]
    b = np.where(fm, 0.0, a)
    rest = ((b[:, 0] + b[:, 1]) + b[:, 2]) + b[:, 3]
    clamp = amax > rest
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        plain = (2.0 * a) / total[:, None]
        capped = a / rest[:, None]
    capped = np.where(fm, 1.0, capped)
    pi = np.where(clamp[:, None], capped, plain)
    nnz = np.count_nonzero(a, axis=1)
    pi[nnz == 1] = np.where(a[nnz == 1] > 0, 1.0, 1.0 / 3.0)
    pi[nnz == 0] = 0.5
    return pi


def mvue_pair_probs(pi: np.ndarray) -> np.ndarray:
    """Greedy transportation fill over the six pairs (sparsity.py:327-355)."""
    pi = np.asarray(pi, dtype=np.float64)
    r0, r1, r2, r3 = (pi[:, i].copy() for i in range(4))
    s = 0.5 * (((pi[:, 0] + pi[:, 1]) + pi[:, 2]) + pi[:, 3])
    p01 = np.maximum(np.minimum(np.minimum(np.minimum(r0, r1), s - r2), s - r3), 0.0)
    r0 = r0 - p01
    r1 = r1 - p01
    s = s - p01
    p02 = np.maximum(np.minimum(np.minimum(r0, r2), s - r3), 0.0)
    r0 = r0 - p02
    r2 = r2 - p02
    s = s - p02
    p03 = np.maximum(np.minimum(r0, r3), 0.0)
    r3 = r3 - p03
    s = s - p03
    p12 = np.maximum(np.minimum(np.minimum(r1, r2), s - r3), 0.0)
    r1 = r1 - p12
    r2 = r2 - p12
    p13 = np.maximum(np.minimum(r1, r3), 0.0)
    r3 = r3 - p13
    p23 = np.maximum(np.minimum(r2, r3), 0.0)
    return np.stack([p01, p02, p03, p12, p13, p23], axis=1)


def mvue_kept(groups: np.ndarray, rng_seed: int):
    """(values (n, 2), kept pair indices (n, 2)) -- sparsity.py:358-376: one
    numpy default_rng(seed).random() draw per group, in group order."""
    groups = np.asarray(groups, dtype=np.float64)
    pi = mvue_inclusion_probs(groups)
    probs = mvue_pair_probs(pi)
    u = np.random.default_rng(int(rng_seed) & 0xFFFF_FFFF_FFFF_FFFF).random(len(groups))
    cum = np.cumsum(probs, axis=1)
    draw = u * cum[:, -1]
    idx = np.minimum(np.sum(cum <= draw[:, None], axis=1), 5)
    kept = MVUE_PAIRS[idx]
    rows = np.arange(len(groups))
    values = np.stack([groups[rows, kept[:, s]] / pi[rows, kept[:, s]] for s in (0, 1)], axis=1)
    return values, kept, idx


def mvue_slots_rowwise(arr: np.ndarray, rng_seed: int):
    """(values (m, k/2), absolute column positions (m, k/2)) -- sparsity.py:401-413."""
    arr = np.ascontiguousarray(np.asarray(arr, dtype=np.float64))
    m, k = arr.shape
    if k % 4:
        raise ShapeError(f"cols={k} not divisible by 4 for row-wise groups")
    values, kept, _ = mvue_kept(arr.reshape(-1, 4), rng_seed)
    pos = kept.reshape(m, k // 4, 2) + (4 * np.arange(k // 4, dtype=np.int64))[None, :, None]
    return values.reshape(m, k // 2), pos.reshape(m, k // 2)


def mvue_seed(rng_seed: int, salt: int) -> int:
    """Per-product seed of _grad_weight (gated_ffn.py:372): (seed << 2) ^ salt."""
    return (int(rng_seed) << 2) ^ salt


def grad_weight_mvue(dz: np.ndarray, x: np.ndarray, rng_seed: int, salt: int) -> np.ndarray:
    """dz^T @ x with dz^T MVUE-sparsified row-wise (gated_ffn.py:367-373), as
    the dense product of the sparsified operand (equal to spmm_rowwise's
    ascending-order result within float64 rounding)."""
    dzt = np.ascontiguousarray(np.asarray(dz, dtype=np.float64).T)
    vals, pos = mvue_slots_rowwise(dzt, mvue_seed(rng_seed, salt))
    dense = np.zeros_like(dzt)
    np.put_along_axis(dense, pos, vals, axis=1)
    return dense @ np.asarray(x, dtype=np.float64)


def fst_backward_mvue(layer: "Layer", fwd: dict, dy: np.ndarray, mask_in, mask_out, rng_seed: int = 0):
    """fst_backward(mvue=True) (gated_ffn.py:304-364): as fst_backward but both
    weight gradients through the MVUE-sparsified upstream gradients (salts 1, 2)."""
    out = fst_backward(layer, fwd, dy, mask_in, mask_out, exact=False)
    out["dw2"] = grad_weight_mvue(np.asarray(dy, dtype=np.float64), fwd["a"], rng_seed, 1)
    out["dw_in"] = grad_weight_mvue(out["dz"], fwd["x"], rng_seed, 2)
    return out
