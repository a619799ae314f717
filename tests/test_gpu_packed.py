"""The packed 2:4 route (Compressed24 / compress / decompress / mask_of / spmm / spmm_right /
dense_matmul, spmm.py:38-190), mvue_prune (sparsity.py:379-398) and block_flip_stats
(optim.py:164-192) on the GPU, against reference-generated goldens
(tests/golden/packed_golden.npz, tests/golden/make_golden.py packed_golden)."""
import os

import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
GD = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "packed_golden.npz")))


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


def _rel(got, want):
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


@pytest.mark.parametrize("name", ["a", "b", "c"])
@pytest.mark.parametrize("colwise", [False, True])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
def test_compress_decompress_mask_of_bit_exact(name, colwise, dtype):
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction

    d = "col" if colwise else "row"
    direction = Direction.COL_WISE if colwise else Direction.ROW_WISE
    w = _dev(GD[f"{name}.w"], dtype)
    est = P.prune_2of4(w, direction)
    assert np.array_equal(est.mask.bits.cpu().numpy(), GD[f"{name}.{d}.bits"])
    est.mask.validate()
    c = P.compress(est)
    assert c.values.dtype == dtype
    assert np.array_equal(c.values.double().cpu().numpy(), GD[f"{name}.{d}.values"])
    assert np.array_equal(c.meta.cpu().numpy(), GD[f"{name}.{d}.meta"])
    dense = P.decompress(c)
    assert np.array_equal(dense.double().cpu().numpy(), GD[f"{name}.{d}.dense"])
    assert dense.is_contiguous() != colwise  # column-wise comes back column-major, like Matrix.col_major
    assert torch.equal(P.mask_of(c).bits, est.mask.bits)
    i0, i1 = c.kept_indices()
    assert bool((i0 < i1).all())
    # compress_masked reads only the kept entries of the unmasked weight
    c2 = P.compress_masked(w, est.mask)
    assert torch.equal(c2.values, c.values) and torch.equal(c2.meta, c.meta)
    t = P.transpose_view(c)
    assert (t.rows, t.cols) == (c.cols, c.rows) and t.values.data_ptr() == c.values.data_ptr()
    assert torch.equal(P.decompress(t), dense.t())


def test_packed_format_errors():
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction, FormatError, ShapeError

    w = torch.randn(8, 16, device="cuda")
    bad = torch.zeros(8, 16, dtype=torch.uint8, device="cuda")
    bad[:, 0] = 1  # one kept entry per group
    with pytest.raises(FormatError):
        P.compress(P.SparseEstimate(w, P.Mask24(bad)))
    with pytest.raises(FormatError):
        P.Mask24(bad).validate()
    with pytest.raises(FormatError):
        P.Mask24(bad * 2 + 0).validate()  # non-0/1 bits
    with pytest.raises(ShapeError):
        P.Mask24(torch.zeros(8, 6, dtype=torch.uint8, device="cuda")).validate()
    c = P.compress(P.prune_2of4(w))
    meta = c.meta.clone()
    meta[3] = 0b0101  # i0 == i1
    broken = P.Compressed24(8, 16, Direction.ROW_WISE, c.values, meta)
    with pytest.raises(FormatError):
        P.decompress(broken)
    with pytest.raises(FormatError):
        broken.kept_indices()
    with pytest.raises(FormatError):
        P.Compressed24(8, 16, Direction.ROW_WISE, c.values[:-1], c.meta)
    with pytest.raises(FormatError):
        P.spmm(P.transpose_view(c), torch.randn(8, 4, device="cuda"))
    with pytest.raises(ShapeError):
        P.spmm(c, torch.randn(15, 4, device="cuda"))


def test_spmm_and_spmm_right_vs_reference():
    """The packed-route products on the 2:4 tensor cores (ragged 96 x 160 x 40: padded to the
    tile multiples) against the reference's float64 results; bf16 output, fp32 accumulation:
    normwise <= 5e-3."""
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction

    w = _dev(GD["b.w"], torch.bfloat16)
    a_c = P.compress(P.prune_2of4(w, Direction.ROW_WISE))
    out = P.spmm(a_c, _dev(GD["spmm.rhs"], torch.bfloat16))
    assert out.shape == (96, 40) and out.dtype == torch.bfloat16
    assert _rel(out.double().cpu().numpy(), GD["spmm.out"]) < 5e-3
    b_c = P.compress(P.prune_2of4(w.t().contiguous(), Direction.COL_WISE))
    out_r = P.spmm_right(_dev(GD["spmm_right.lhs"], torch.bfloat16), b_c)
    assert out_r.shape == (40, 96) and out_r.stride()[0] == 1  # column-major, like the reference
    assert _rel(out_r.double().cpu().numpy(), GD["spmm_right.out"]) < 5e-3
    # fp64 values are rounded to bf16 for the tensor cores: same result here (bf16-exact data)
    a64 = P.compress(P.prune_2of4(w.double(), Direction.ROW_WISE))
    assert torch.equal(P.spmm(a64, _dev(GD["spmm.rhs"], torch.float64)), out)


@pytest.mark.parametrize("m,k,n", [(96, 160, 40), (1024, 4096, 512), (256, 128, 1000)])
def test_spmm_matches_dense_matmul_of_decompressed(m, k, n):
    import paper_2404_01847_b200 as P

    g = torch.Generator(device="cpu").manual_seed(m + k + n)
    w = torch.randn(m, k, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(k, n, generator=g).to(torch.bfloat16).cuda()
    c = P.compress(P.SparseEstimate(w, P.transposable_search_conv(w).to_mask24(P.Direction.ROW_WISE)))
    got = P.spmm(c, b).double()
    ref = P.decompress(c).double() @ b.double()
    assert _rel(got.cpu().numpy(), ref.cpu().numpy()) < 5e-3
    dm = P.dense_matmul(P.decompress(c), b)
    assert dm.dtype == torch.float32
    assert _rel(dm.double().cpu().numpy(), ref.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("i", range(4))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float64])
def test_mvue_prune_bit_exact_vs_reference(i, dtype):
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.matrix import Direction

    g = _dev(GD[f"mvue{i}.g"], dtype)
    seed = int(GD[f"mvue{i}.seed"])
    for colwise in (False, True):
        d = "col" if colwise else "row"
        est = P.mvue_prune(g, Direction.COL_WISE if colwise else Direction.ROW_WISE, seed)
        assert est.values.dtype == torch.float64
        assert np.array_equal(est.values.cpu().numpy().view(np.uint64), GD[f"mvue{i}.{d}.values"].view(np.uint64))
        assert np.array_equal(est.mask.bits.cpu().numpy(), GD[f"mvue{i}.{d}.bits"])
        est.mask.validate()


def test_mvue_prune_large_matches_oracle_and_is_unbiased():
    """A 512 x 1024 bf16 gradient (131072 groups, many jump-ahead runs): bit-exact vs the
    oracle's float64 restatement, and the seed average converges to the input."""
    import paper_2404_01847_b200 as P

    gx = o.round_bf16(o.det_normal((512, 1024), seed=77))
    g = _dev(gx, torch.bfloat16)
    est = P.mvue_prune(g, rng_seed=123456789)
    vals, bits = o.mvue_prune(gx, False, 123456789)
    assert np.array_equal(est.values.cpu().numpy().view(np.uint64), vals.view(np.uint64))
    assert np.array_equal(est.mask.bits.cpu().numpy(), bits)
    acc = torch.zeros_like(est.values)
    for s in range(64):
        acc += P.mvue_prune(g, rng_seed=s).values
    err = (acc / 64 - g.double()).abs().mean() / g.double().abs().mean()
    assert float(err) < 0.12


def test_block_flip_stats_bit_exact_vs_reference():
    import paper_2404_01847_b200 as P

    snaps = [_dev(GD[f"flip3.w{c}"], torch.float64) for c in "abc"]
    tr = P.block_flip_stats(snaps)
    assert np.array_equal(tr.block_flips.cpu().numpy(), GD["flip3.block_flips"])
    assert np.array_equal(tr.block_gaps.cpu().numpy().view(np.uint64), GD["flip3.block_gaps"].view(np.uint64))
    ties = _dev(GD["ties.w"], torch.bfloat16)
    tt = P.block_flip_stats([ties, ties])
    assert int(tt.block_flips.sum()) == 0
    assert np.array_equal(tt.block_gaps.cpu().numpy(), GD["ties.block_gaps"])
    # bf16 / fp32 snapshots: gaps equal the oracle's on the same (exactly representable) values
    w = o.round_bf16(o.det_normal((256, 512), 5))
    w2 = o.round_bf16(w * 1.5)
    for dt in (torch.bfloat16, torch.float32):
        got = P.block_flip_stats([_dev(w, dt), _dev(w2, dt)]).block_gaps.cpu().numpy()
        assert np.array_equal(got, o.block_gaps(w2))


def test_srste_weight_decay_matches_reference_formula():
    import paper_2404_01847_b200 as P

    w0 = o.round_bf16(o.det_normal((64, 96), 700) * 0.05)
    base = o.det_normal((64, 96), 701) * 0.05
    wt = _dev(w0, torch.float32)
    m = P.transposable_search_conv(wt)
    got = P.srste_weight_decay(_dev(base, torch.float32), wt, m, 3e-3, 6e-2).double().cpu().numpy()
    want = o.srste_weight_decay(base.astype(np.float32).astype(np.float64), w0, m.bits.cpu().numpy(), 3e-3, 6e-2)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-9)


def test_compress_round_trip_at_c3_weight_size():
    """Size-independent property at the C3 first-weight shape (22016 x 4096, 90 M weights):
    compress -> decompress reproduces the masked weight bit for bit, and the packed values /
    nibbles equal the training path's compressed operand (the same value order)."""
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200 import engine as E

    w = torch.randn(22016, 4096, device="cuda").to(torch.bfloat16)
    mask = P.transposable_search_conv(w)
    c = P.compress_masked(w, mask.to_mask24(P.Direction.ROW_WISE))
    assert torch.equal(P.decompress(c), w * mask.bits.to(w.dtype))
    op = E.CompressedOperand.empty(22016, 4096, "cuda")
    E.search_compress(w, op)
    assert torch.equal(c.values.view(22016, 2048), op.fwd_vals.view(22016, 2048))
    assert torch.equal(c.meta.view(22016, 1024), mask.meta()[0])
