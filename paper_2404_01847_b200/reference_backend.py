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
  * matmul_ref, spmm_rowwise, prune_2of4_keep, greedy_masks -- not on the
                        B200 hot path: raise.
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


def _not_on_path(name):
    def f(*a, **k):
        raise NotImplementedError(f"{name} is not on the B200 hot path (SURVEY.md section 2.1)")

    return f


matmul_ref = _not_on_path("matmul_ref")
spmm_rowwise = _not_on_path("spmm_rowwise")
prune_2of4_keep = _not_on_path("prune_2of4_keep")
greedy_masks = _not_on_path("greedy_masks")
