"""The reference's kernel-module interface (sparse24.backend.kernels,
backend.py:13-36, _core.pyx:26-250) implemented over the B200 C ABI.

A maintainer of the reference can inject it without editing the package,
because every call site resolves `kernels.<fn>` at call time
(sparsity.py:236/269/278, spmm.py:161/176/187, gated_ffn.py:162/223/267/373):

    import sparse24.backend, sparse24.sparsity, sparse24.gated_ffn
    from paper_2404_01847_b200 import reference_backend as rb
    for mod in (sparse24.sparsity, sparse24.gated_ffn, sparse24.spmm):
        mod.kernels = rb

Semantics per entry point:
  * pattern_scores   -- `best` is computed by K1 on the GPU and is bit-exact
                        (same float64 ascending-order scores, first max);
                        `scores` are the same sequential float64 sums,
                        evaluated on the GPU with torch in the same order.
  * spmm_colwise     -- the 2:4 tensor-core GEMM (bf16 operands, fp32
                        accumulation): toleranced, NOT bit-equal to the
                        float64 reference (the reference's own bitwise tests
                        of spmm vs dense_matmul do not apply).
  * gate_gelu        -- the fused gate kernel K6 (fp32 math, bf16 storage):
                        toleranced.
  * matmul_ref       -- the dense tcgen05 GEMM (bf16 operands, fp32 accumulation),
                        toleranced.
  * spmm_rowwise     -- the MVUE weight-gradient product: a row-wise 2:4 operand
                        on the 2:4 tensor cores (s24_pack24 + s24_flat_to_e +
                        s24_spmm_dw), toleranced.
  * prune_2of4_keep  -- s24_prune_2of4, bit-exact (ties to the lowest index).
  * greedy_masks     -- s24_greedy_search, bit-exact; RuntimeError when a block
                        cannot be completed, as the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _capi as C
from .matrix import ShapeError

BACKEND_NAME = "b200"


def _dev(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def pattern_scores(absblocks, positions):
    """(scores (nb, np) float64, best (nb,) int64) -- _core.pyx:83-110."""
    ab = np.ascontiguousarray(np.asarray(absblocks, dtype=np.float64))
    pos = np.asarray(positions)
    nb = ab.shape[0]
    from .sparsity import enumerate_patterns

    canon = enumerate_patterns().positions
    # K1 works on whole 4x4 blocks: lay the (nb, 16) rows out as a (4, 4*nb) matrix
    w = _dev(ab.reshape(nb, 4, 4).transpose(1, 0, 2).reshape(4, 4 * nb))
    best = torch.empty((1, nb), dtype=torch.uint8, device="cuda")
    if nb:
        C.call("s24_transposable_search", w.data_ptr(), C.S24_F64, 4, 4 * nb, best.data_ptr(), C.stream_of(w))
    blocks = _dev(ab)
    pos_d = torch.as_tensor(pos.astype(np.int64)).cuda()
    scores = blocks[:, pos_d[:, 0]].clone()
    for p in range(1, pos.shape[1]):
        scores = scores + blocks[:, pos_d[:, p]]  # sequential ascending adds, like _core.pyx:102-105
    best64 = best.reshape(-1).to(torch.int64)
    if pos.shape != canon.shape or not np.array_equal(pos, canon):
        best64 = torch.argmax(scores, dim=1)  # non-canonical table: first max of the given order
    return scores.cpu().numpy(), best64.cpu().numpy()


def spmm_colwise(a, values, pos):
    """C = A @ B, B column-wise 2:4 as (values, absolute row positions), F-order
    output (_core.pyx:63-80), via the tensor-core GEMM on W^T = B^T (toleranced)."""
    from .engine import CompressedOperand, compress_with_meta, spmm

    a = np.asarray(a, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    pos = np.asarray(pos)
    m, k = a.shape
    s, n = values.shape
    if 2 * s != k:
        raise ValueError("inner dimensions differ")
    bt = np.zeros((n, k))
    bt[np.arange(n)[None, :].repeat(s, 0), pos] = values  # dense W = B^T (n x k)
    pad = lambda v, q: (v + q - 1) // q * q  # noqa: E731
    N_, K_, M_ = pad(n, 128), pad(k, 128), pad(m, 64)
    w = torch.zeros((N_, K_), dtype=torch.bfloat16, device="cuda")
    w[:n, :k] = torch.as_tensor(bt).cuda().to(torch.bfloat16)
    from .sparsity import TransposableMask

    # mask of W = B^T; padded blocks take canonical pattern 0 (their values are 0)
    pat0 = torch.tensor([[0, 0, 1, 1], [0, 0, 1, 1], [1, 1, 0, 0], [1, 1, 0, 0]], dtype=torch.uint8)
    bits = pat0.repeat(N_ // 4, K_ // 4).cuda()
    bits[:n, :k] = torch.as_tensor(_kept(pos, n, k)).cuda().to(torch.uint8)
    mask = TransposableMask(bits=bits)
    mask.validate()  # the tensor-core operand needs a transposable (4x4-block) mask, as FST produces
    op = CompressedOperand.empty(N_, K_, "cuda")
    op.idx.copy_(mask.idx)
    compress_with_meta(w, op)
    x = torch.zeros((M_, K_), dtype=torch.bfloat16, device="cuda")
    x[:m, :k] = torch.as_tensor(a).cuda().to(torch.bfloat16)
    out = torch.empty((N_, M_), dtype=torch.bfloat16, device="cuda")
    spmm(op.fwd_vals, op.fwd_e, N_, K_, x, False, M_, out)
    return np.asfortranarray(out[:n, :m].t().double().cpu().numpy())


def _kept(pos, n, k):
    mask = np.zeros((n, k), dtype=bool)
    mask[np.arange(n)[None, :].repeat(pos.shape[0], 0), pos] = True
    return mask


def gate_gelu(z1, z2, row_order):
    """gelu(z1) * z2 into a column-major buffer (_core.pyx:222-250), K6 on the GPU."""
    z1 = np.asarray(z1, dtype=np.float64)
    z2 = np.asarray(z2, dtype=np.float64)
    if z1.shape != z2.shape:
        raise ValueError("gate operands differ in shape")
    m, n = z1.shape
    npad = (n + 7) // 8 * 8
    z = torch.zeros((m, 2 * npad), dtype=torch.bfloat16, device="cuda")  # token-major [z1 | z2]
    z[:, :n] = torch.as_tensor(z1).cuda().to(torch.bfloat16)
    z[:, npad:npad + n] = torch.as_tensor(z2).cuda().to(torch.bfloat16)
    a = torch.empty((m, npad), dtype=torch.bfloat16, device="cuda")
    if m and npad:
        C.call("s24_act_fwd", z.data_ptr(), 2 * npad, npad, m, C.ACT_GEGLU, a.data_ptr(), npad, C.stream_of(z))
    return np.asfortranarray(a[:, :n].double().cpu().numpy())


def _pad(v: int, q: int) -> int:
    return (v + q - 1) // q * q


def _out_dtype(*arrays):
    """The reference's fused `real` type: float32 in -> float32 out, else float64 (_core.pyx:21-23)."""
    return np.float32 if all(np.asarray(x).dtype == np.float32 for x in arrays) else np.float64


def matmul_ref(a, b):
    """C = A @ B (_core.pyx:26-41) on the dense tcgen05 GEMM (s24_gemm_dw: bf16 operands, fp32
    accumulation; toleranced, not the reference's ascending-k float64 sums)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("inner dimensions differ")
    m, k = a.shape
    n = b.shape[1]
    out_dt = _out_dtype(a, b)
    if m == 0 or n == 0 or k == 0:
        return np.zeros((m, n), dtype=out_dt)
    M_, N_, K_ = _pad(m, 128), _pad(n, 128), _pad(k, 64)
    ad = torch.zeros((M_, K_), dtype=torch.bfloat16, device="cuda")
    ad[:m, :k] = _dev(a.astype(np.float64)).to(torch.bfloat16)
    bd = torch.zeros((K_, N_), dtype=torch.bfloat16, device="cuda")  # stored k x n: B MN-major
    bd[:k, :n] = _dev(b.astype(np.float64)).to(torch.bfloat16)
    out = torch.empty((M_, N_), dtype=torch.float32, device="cuda")
    from .engine import gemm_dw

    gemm_dw(ad, False, bd, True, M_, N_, K_, out)
    return out[:m, :n].cpu().numpy().astype(out_dt)


def spmm_rowwise(values, pos, b):
    """C = A @ B with A given row-wise as kept values + absolute column positions
    (_core.pyx:44-60; the MVUE weight-gradient product of _grad_weight, gated_ffn.py:372-373).
    A 2:4 row-wise operand (at most two kept per aligned group of four, as mvue_slots_rowwise
    produces) runs on the 2:4 tensor cores: packed with s24_pack24, metadata to E tiles
    (s24_flat_to_e), then s24_spmm_dw.  Any other sparsity takes the dense GEMM.  Toleranced."""
    values = np.asarray(values)
    pos = np.asarray(pos, dtype=np.int64)
    b = np.asarray(b)
    m, s_ = values.shape
    k, n = b.shape
    out_dt = _out_dtype(values, b)
    if pos.shape != values.shape:
        raise ValueError("values and positions differ in shape")
    if m == 0 or n == 0 or s_ == 0:
        return np.zeros((m, n), dtype=out_dt)
    if pos.min() < 0 or pos.max() >= k:
        raise ValueError("position out of range")
    a = np.zeros((m, k))
    np.add.at(a, (np.repeat(np.arange(m), s_), pos.reshape(-1)), values.reshape(-1).astype(np.float64))
    kept = np.zeros((m, _pad(k, 4)), dtype=np.int32)
    np.add.at(kept, (np.repeat(np.arange(m), s_), pos.reshape(-1)), 1)
    per_group = kept.reshape(m, -1, 4).sum(axis=2)
    if per_group.max() > 2:
        return matmul_ref(a, b)
    M_, K_, N_ = _pad(m, 128), _pad(k, 128), _pad(n, 128)
    # complete every group to exactly two kept slots (zero-valued fillers at the lowest free
    # positions) so it is a valid 2:4 operand
    bits = np.zeros((M_, K_), dtype=np.uint8)
    bits[:m, :kept.shape[1]] = kept > 0
    g = bits.reshape(M_, K_ // 4, 4)
    for _ in range(2):
        need = g.sum(axis=2) < 2
        free = np.argmax(g == 0, axis=2)
        r, c = np.nonzero(need)
        g[r, c, free[r, c]] = 1
    wd = torch.zeros((M_, K_), dtype=torch.bfloat16, device="cuda")
    wd[:m, :k] = _dev(a).to(torch.bfloat16)
    bits_d = _dev(bits)
    vals = torch.empty((M_, K_ // 2), dtype=torch.bfloat16, device="cuda")
    meta = torch.empty((M_, K_ // 4), dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = C.stream_of(wd)
    C.call("s24_pack24", wd.data_ptr(), C.S24_BF16, bits_d.data_ptr(), M_, K_, 0, vals.data_ptr(), meta.data_ptr(),
           bad.data_ptr(), st)
    e = torch.empty((M_ // 128) * (K_ // 128) * 2048, dtype=torch.uint8, device="cuda")
    C.call("s24_flat_to_e", meta.data_ptr(), M_, K_, e.data_ptr(), st)
    bd = torch.zeros((K_, N_), dtype=torch.bfloat16, device="cuda")  # stored k x n: B MN-major
    bd[:k, :n] = _dev(b.astype(np.float64)).to(torch.bfloat16)
    out = torch.empty((M_, N_), dtype=torch.float32, device="cuda")
    from .engine import spmm_dw

    spmm_dw(vals, e, M_, K_, bd, True, N_, out)
    return out[:m, :n].cpu().numpy().astype(out_dt)


def prune_2of4_keep(groups):
    """Keep-mask (ng, 4) uint8 of the two largest |g| per group, ties to the lowest index
    (_core.pyx:113-136) -- s24_prune_2of4 on the (ng x 4) matrix, bit-exact."""
    g = np.ascontiguousarray(np.asarray(groups))
    if g.ndim != 2 or g.shape[1] != 4:
        raise ValueError("groups must be (ng, 4)")
    ng = g.shape[0]
    if ng == 0:
        return np.zeros((0, 4), dtype=np.uint8)
    dt = C.S24_F32 if g.dtype == np.float32 else C.S24_F64
    gd = _dev(g.astype(np.float32 if dt == C.S24_F32 else np.float64))
    # the kernel tiles rows in groups of 4: pad the group count to a multiple of 4 rows
    rows = _pad(ng, 4)
    if rows != ng:
        gd = torch.cat([gd, torch.zeros((rows - ng, 4), dtype=gd.dtype, device="cuda")])
    bits = torch.empty((rows, 4), dtype=torch.uint8, device="cuda")
    C.call("s24_prune_2of4", gd.data_ptr(), dt, rows, 4, 0, bits.data_ptr(), C.stream_of(gd))
    return bits[:ng].cpu().numpy()


def greedy_masks(absblocks):
    """Greedy transposable mask per 4x4 block (_core.pyx:139-219), bit-exact: s24_greedy_search
    on the blocks laid out as a (4, 4 nb) matrix.  RuntimeError when a block cannot be completed
    (the reference's failure, :215-216)."""
    ab = np.ascontiguousarray(np.asarray(absblocks))
    if ab.ndim != 2 or ab.shape[1] != 16:
        raise ValueError("absblocks must be (nb, 16)")
    nb = ab.shape[0]
    if nb == 0:
        return np.zeros((0, 16), dtype=np.uint8)
    dt = C.S24_F32 if ab.dtype == np.float32 else C.S24_F64
    w = _dev(ab.astype(np.float32 if dt == C.S24_F32 else np.float64).reshape(nb, 4, 4).transpose(1, 0, 2)
             .reshape(4, 4 * nb))
    idx = torch.empty((1, nb), dtype=torch.uint8, device="cuda")
    fails = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = C.stream_of(w)
    C.call("s24_greedy_search", w.data_ptr(), dt, 4, 4 * nb, idx.data_ptr(), fails.data_ptr(), st)
    if int(fails.item()):
        raise RuntimeError("greedy mask completion failed")
    bits = torch.empty((4, 4 * nb), dtype=torch.uint8, device="cuda")
    C.call("s24_idx_to_bits", idx.data_ptr(), 4, 4 * nb, bits.data_ptr(), st)
    return bits.reshape(4, nb, 4).permute(1, 0, 2).reshape(nb, 16).cpu().numpy()
