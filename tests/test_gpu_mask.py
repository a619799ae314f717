"""K1 / K2 parity on the GPU: mask search, compress, metadata -- bit-exact
against the reference's golden vectors and the oracle."""
import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from make_golden import mask_corpora
from gpu_util import bf16_bits_of, need_gpu, to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    need_gpu()


@pytest.fixture(scope="module")
def corpora():
    return mask_corpora()


def _dev(w: np.ndarray, tag: str) -> torch.Tensor:
    if tag == "bf16":
        return to_dev_bf16(w)
    if tag == "f32":
        return torch.from_numpy(w.astype(np.float32)).cuda()
    return torch.from_numpy(w).cuda()


@pytest.mark.parametrize("name", ["gauss_f64", "gauss_bf16", "int_ties", "kats", "c1_w1_f32", "c2_w1_bf16"])
def test_search_bit_exact_vs_reference_golden(name, corpora, mask_golden):
    from paper_2404_01847_b200 import transposable_search_conv

    w, tag = corpora[name]
    m = transposable_search_conv(_dev(w, tag))
    np.testing.assert_array_equal(m.idx.cpu().numpy(), mask_golden[f"{name}.idx"])
    bits = m.bits.cpu().numpy()
    np.testing.assert_array_equal(bits, o.idx_to_bits(mask_golden[f"{name}.idx"]))


@pytest.mark.parametrize("name", ["gauss_bf16", "int_ties", "kats"])
def test_compress_values_and_meta_bit_exact(name, corpora, mask_golden):
    import paper_2404_01847_b200._capi as C

    w, _ = corpora[name]
    wd = to_dev_bf16(w)
    rows, cols = w.shape
    idx = torch.empty((rows // 4, cols // 4), dtype=torch.uint8, device="cuda")
    fv = torch.empty((rows, cols // 2), dtype=torch.bfloat16, device="cuda")
    bv = torch.empty((cols, rows // 2), dtype=torch.bfloat16, device="cuda")
    C.call("s24_search_compress", wd.data_ptr(), C.S24_BF16, rows, cols, idx.data_ptr(), fv.data_ptr(), None,
           bv.data_ptr(), None, 0, C.stream_of(wd))
    np.testing.assert_array_equal(idx.cpu().numpy(), mask_golden[f"{name}.idx"])
    np.testing.assert_array_equal(bf16_bits_of(fv), mask_golden[f"{name}.fwd_values"])
    np.testing.assert_array_equal(bf16_bits_of(bv), mask_golden[f"{name}.bwd_values"])
    from paper_2404_01847_b200 import TransposableMask
    fm, bm = TransposableMask(idx, (rows, cols)).meta()
    np.testing.assert_array_equal(fm.cpu().numpy(), mask_golden[f"{name}.fwd_meta"])
    np.testing.assert_array_equal(bm.cpu().numpy(), mask_golden[f"{name}.bwd_meta"])
    # K2 from the cached mask reproduces the same values
    fv2, bv2 = torch.zeros_like(fv), torch.zeros_like(bv)
    C.call("s24_prune_compress", wd.data_ptr(), C.S24_BF16, rows, cols, idx.data_ptr(), fv2.data_ptr(), None,
           bv2.data_ptr(), None, 0, C.stream_of(wd))
    assert torch.equal(fv2.view(torch.int16), fv.view(torch.int16))
    assert torch.equal(bv2.view(torch.int16), bv.view(torch.int16))


@pytest.mark.parametrize("name", ["gauss_bf16", "int_ties", "c2_w1_bf16"])
def test_tensor_core_metadata_tiles_encode_reference_meta(name, corpora, mask_golden):
    """E tiles (both orientations) decode to the reference nibbles."""
    import paper_2404_01847_b200._capi as C
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress

    w, _ = corpora[name]
    rows, cols = w.shape
    op = CompressedOperand.empty(rows, cols, "cuda")
    search_compress(to_dev_bf16(w), op)
    idx = mask_golden[f"{name}.idx"]
    np.testing.assert_array_equal(op.idx.cpu().numpy(), idx)
    ref_bits = o.idx_to_bits(idx)
    _, fmeta = o.compress_rowwise(np.zeros(ref_bits.shape), ref_bits)
    _, bmeta = o.compress_rowwise(np.zeros(ref_bits.shape), np.ascontiguousarray(ref_bits.T))
    f = torch.empty((rows, cols // 4), dtype=torch.uint8, device="cuda")
    b = torch.empty((cols, rows // 4), dtype=torch.uint8, device="cuda")
    C.call("s24_e_to_flat", op.fwd_e.data_ptr(), rows, cols, f.data_ptr(), C.stream_of(f))
    C.call("s24_e_to_flat", op.bwd_e.data_ptr(), cols, rows, b.data_ptr(), C.stream_of(b))
    np.testing.assert_array_equal(f.cpu().numpy(), fmeta)
    np.testing.assert_array_equal(b.cpu().numpy(), bmeta)


@pytest.mark.parametrize("shape", [(4, 4), (8, 12), (132, 200), (260, 388), (4, 1032)])
@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
def test_ragged_shapes_vs_oracle(shape, dtype):
    from paper_2404_01847_b200 import transposable_search_conv

    w = o.det_normal(shape, seed=sum(shape))
    if dtype == "bf16":
        w = o.round_bf16(w)
    elif dtype == "f32":
        w = w.astype(np.float32).astype(np.float64)
    if dtype in ("f32", "f64") and shape[1] % 4:
        pytest.skip("alignment")
    m = transposable_search_conv(_dev(w, dtype))
    np.testing.assert_array_equal(m.idx.cpu().numpy(), o.search_pattern_idx(w))


def test_ties_and_exponent_spans_bf16():
    """Heavy ties + blocks whose exponent span forces the float64 slow path."""
    from paper_2404_01847_b200 import transposable_search_conv

    rng = np.random.default_rng(3)
    w = rng.integers(-3, 4, size=(256, 256)).astype(np.float64)
    w[::3] *= 2.0 ** 40
    w[1::5] *= 2.0 ** -50
    w[:, ::7] = 0.0
    w = o.round_bf16(w)
    m = transposable_search_conv(to_dev_bf16(w))
    np.testing.assert_array_equal(m.idx.cpu().numpy(), o.search_pattern_idx(w))


def test_shape_error_and_format_error():
    from paper_2404_01847_b200 import FormatError, ShapeError, TransposableMask, transposable_search_conv

    with pytest.raises(ShapeError):
        transposable_search_conv(torch.zeros((6, 8), device="cuda", dtype=torch.bfloat16))
    bad = torch.ones((4, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(FormatError):
        TransposableMask(bits=bad).validate()
    good = transposable_search_conv(torch.randn(16, 16, device="cuda").bfloat16())
    TransposableMask(bits=good.bits).validate()
    t = good.transpose()
    assert torch.equal(t.bits, good.bits.t().contiguous())


def test_masked_decay_kernel():
    from paper_2404_01847_b200 import masked_decay_gradient, transposable_search_conv

    w = torch.randn(64, 128, device="cuda").bfloat16()
    g = torch.randn(64, 128, device="cuda")
    m = transposable_search_conv(w)
    out = masked_decay_gradient(g, w, m, 6e-5)
    ref = o.masked_decay_gradient(g.cpu().double().numpy(), w.float().cpu().double().numpy(),
                                  m.bits.cpu().numpy(), 6e-5)
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-6, atol=1e-7)
    # kept weights untouched (test_optim.py:81-86)
    kept = m.bits.bool()
    assert torch.equal(out[kept], g[kept])


def test_reference_backend_shim_pattern_scores_bit_exact(mask_golden):
    """The reference-kernel-interface shim: pattern_scores(best) bit-exact on the
    reference acceptance-style corpus, scores equal to the sequential f64 sums."""
    from paper_2404_01847_b200 import reference_backend as rb

    w = mask_corpora()["gauss_f64"][0]
    absb = np.abs(o.blocks16(w))
    _, pos = o.pattern_table()
    scores, best = rb.pattern_scores(absb, pos)
    s_ref, b_ref = o.pattern_scores(absb, pos)
    assert scores.tobytes() == s_ref.tobytes()
    np.testing.assert_array_equal(best, b_ref)
    np.testing.assert_array_equal(best.reshape(-1), mask_golden["gauss_f64.idx"].reshape(-1))


def test_reference_backend_shim_spmm_and_gate_toleranced():
    from paper_2404_01847_b200 import reference_backend as rb

    rng = np.random.default_rng(1)
    w = o.round_bf16(rng.standard_normal((48, 40)))  # B^T (n x k) in the reference's column-wise spmm
    bits = o.transposable_search_conv(w)
    take, pos_t = o.gather_plan(bits, False)
    vals = w.ravel()[take].T
    a = o.round_bf16(rng.standard_normal((20, 40)))
    got = rb.spmm_colwise(a, vals, pos_t)
    ref = o.spmm_colwise(a, vals, pos_t)
    assert got.flags["F_CONTIGUOUS"]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-2
    z1, z2 = rng.standard_normal((9, 12)), rng.standard_normal((9, 12))
    g = rb.gate_gelu(z1, z2, False)
    assert np.linalg.norm(g - o.gate(z1, z2)) / np.linalg.norm(o.gate(z1, z2)) < 1e-2


def test_gated_interleave_masks_are_reference_masks_permuted():
    """u/v-interleaved compression of W_in = [u; v]: the mask (un-permuted) equals
    the reference mask of [u; v]; the interleaved kept values are the rows' values."""
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress

    d_ff, d = 256, 128
    w = o.round_bf16(o.det_normal((2 * d_ff, d), seed=77))
    op = CompressedOperand.empty(2 * d_ff, d, "cuda", perm_ff=d_ff)
    search_compress(to_dev_bf16(w), op)
    np.testing.assert_array_equal(op.mask_idx().cpu().numpy(), o.search_pattern_idx(w))
    p = np.arange(2 * d_ff)
    orig = np.where(p % 32 < 16, 16 * (p // 32) + p % 32, d_ff + 16 * (p // 32) + p % 32 - 16)
    kv, _ = o.compress_rowwise(w[orig], o.transposable_search_conv(w)[orig])
    np.testing.assert_array_equal(bf16_bits_of(op.fwd_vals), o.bf16_bits(kv))


@pytest.mark.parametrize("shape,perm_ff", [((256, 384), 0), ((512, 128), 256), ((384, 1024), 0)])
def test_k2_fast_prune_matches_oracle(shape, perm_ff):
    """K2 bf16 fast path (tile-aligned shapes, no metadata): both value
    orientations bit-equal to the oracle's compress of the cached mask, for the
    plain and the u/v-interleaved (gated) row order."""
    from paper_2404_01847_b200.engine import CompressedOperand, compress_values, search_compress

    rows, cols = shape
    w = o.round_bf16(o.det_normal(shape, seed=rows + 7 * cols))
    wd = to_dev_bf16(w)
    op = CompressedOperand.empty(rows, cols, "cuda", perm_ff=perm_ff)
    search_compress(wd, op)
    fv1, bv1 = op.fwd_vals.clone(), op.bwd_vals.clone()
    w2 = o.round_bf16(o.det_normal(shape, seed=rows + 7 * cols + 1))  # new values, same (cached) mask
    op.fwd_vals.zero_()
    op.bwd_vals.zero_()
    compress_values(to_dev_bf16(w2), op)
    bits = o.idx_to_bits(op.mask_idx().cpu().numpy())
    p = np.arange(rows)
    order = p if perm_ff == 0 else np.where(p % 32 < 16, 16 * (p // 32) + p % 32, perm_ff + 16 * (p // 32) + p % 32 - 16)
    kv, _ = o.compress_rowwise(w2[order], bits[order])
    np.testing.assert_array_equal(bf16_bits_of(op.fwd_vals), o.bf16_bits(kv))
    kb, _ = o.compress_rowwise(np.ascontiguousarray(w2[order].T), np.ascontiguousarray(bits[order].T))
    np.testing.assert_array_equal(bf16_bits_of(op.bwd_vals), o.bf16_bits(kb))
    # and K2 on the original values reproduces K1's fused compress
    compress_values(wd, op)
    assert torch.equal(op.fwd_vals.view(torch.int16), fv1.view(torch.int16))
    assert torch.equal(op.bwd_vals.view(torch.int16), bv1.view(torch.int16))


@pytest.mark.parametrize("shape,perm_ff", [((256, 384), 0), ((512, 128), 256)])
def test_k2_fp32_masters_fast_prune_matches_oracle(shape, perm_ff):
    """K2 on fp32 master weights (the module's per-step recompression): kept values rounded to
    bf16 (round-to-nearest-even, incl. exact ties and values beyond bf16 range) equal the
    oracle's compress of the bf16-rounded weights, and equal K1's fused compress of the same
    fp32 weights (the general tiled kernel's conversion)."""
    from paper_2404_01847_b200.engine import CompressedOperand, compress_values, search_compress

    rows, cols = shape
    w = o.det_normal(shape, seed=rows + 3 * cols).astype(np.float32)
    # bf16 rounding ties (exactly halfway, both parities) and huge / tiny magnitudes
    flat = w.reshape(-1)
    flat[::97] = np.float32(1.0 + 2.0 ** -8)           # tie -> round down to even
    flat[5::97] = np.float32(1.0 + 3 * 2.0 ** -8)      # tie -> round up to even
    flat[11::193] = np.float32(3.0e38)
    flat[17::193] = np.float32(-1.0e-40)
    wd = torch.from_numpy(w).cuda()
    op = CompressedOperand.empty(rows, cols, "cuda", perm_ff=perm_ff)
    search_compress(wd, op)
    fv1, bv1 = op.fwd_vals.clone(), op.bwd_vals.clone()
    op.fwd_vals.zero_()
    op.bwd_vals.zero_()
    compress_values(wd, op)
    assert torch.equal(op.fwd_vals.view(torch.int16), fv1.view(torch.int16))
    assert torch.equal(op.bwd_vals.view(torch.int16), bv1.view(torch.int16))
    bits = o.idx_to_bits(op.mask_idx().cpu().numpy())
    p = np.arange(rows)
    order = p if perm_ff == 0 else np.where(p % 32 < 16, 16 * (p // 32) + p % 32, perm_ff + 16 * (p // 32) + p % 32 - 16)
    wr = o.round_bf16(w)
    kv, _ = o.compress_rowwise(wr[order], bits[order])
    np.testing.assert_array_equal(bf16_bits_of(op.fwd_vals), o.bf16_bits(kv))
    kb, _ = o.compress_rowwise(np.ascontiguousarray(wr[order].T), np.ascontiguousarray(bits[order].T))
    np.testing.assert_array_equal(bf16_bits_of(op.bwd_vals), o.bf16_bits(kb))


@pytest.mark.parametrize("gated", [False, True])
def test_k2_pair_launch_equals_two_single_launches(gated):
    """s24_prune_compress_pair (both weights of a block in one launch) == two s24_prune_compress calls."""
    from paper_2404_01847_b200 import engine as E

    d, d_ff = 256, 384
    r_in = 2 * d_ff if gated else d_ff
    w_in = torch.randn(r_in, d, device="cuda").bfloat16()
    w2 = torch.randn(d, d_ff, device="cuda").bfloat16()
    ops = []
    for _ in range(2):
        a = E.CompressedOperand.empty(r_in, d, "cuda", perm_ff=d_ff if gated else 0)
        b = E.CompressedOperand.empty(d, d_ff, "cuda")
        E.search_compress(w_in, a)
        E.search_compress(w2, b)
        ops.append((a, b))
    w_in2, w22 = w_in * 1.5, w2 - 0.25  # new values under the cached masks
    E.compress_values(w_in2, ops[0][0])
    E.compress_values(w22, ops[0][1])
    E.compress_values_pair(w_in2, ops[1][0], w22, ops[1][1])
    for x, y in zip(ops[0], ops[1]):
        assert torch.equal(x.fwd_vals, y.fwd_vals) and torch.equal(x.bwd_vals, y.bwd_vals)


@pytest.mark.parametrize("gated,dtype", [(False, torch.bfloat16), (True, torch.bfloat16), (False, torch.float32)])
def test_k1_pair_launch_equals_two_single_launches(gated, dtype):
    """s24_search_compress_pair (the mask refresh of both weights of a block in one launch) ==
    two s24_search_compress calls: pattern indices, kept values and E tiles of both orientations."""
    from paper_2404_01847_b200 import engine as E

    d, d_ff = 256, 384
    r_in = 2 * d_ff if gated else d_ff
    torch.manual_seed(5)
    w_in = torch.randn(r_in, d, device="cuda").to(dtype)
    w2 = torch.randn(d, d_ff, device="cuda").to(dtype)
    ops = [(E.CompressedOperand.empty(r_in, d, "cuda", perm_ff=d_ff if gated else 0),
            E.CompressedOperand.empty(d, d_ff, "cuda")) for _ in range(2)]
    E.search_compress(w_in, ops[0][0])
    E.search_compress(w2, ops[0][1])
    E.search_compress_pair(w_in, ops[1][0], w2, ops[1][1])
    for x, y in zip(ops[0], ops[1]):
        assert torch.equal(x.idx, y.idx)
        assert torch.equal(x.fwd_vals, y.fwd_vals) and torch.equal(x.bwd_vals, y.bwd_vals)
        assert torch.equal(x.fwd_e, y.fwd_e) and torch.equal(x.bwd_e, y.bwd_e)


@pytest.mark.parametrize("shape", [(256, 512), (132, 136)])
def test_wide_exponent_span_bf16(shape):
    """bf16 blocks with exponent spans 10..40 around the integer path's limit (13), with heavy
    ties, zeros and subnormals: pattern indices equal the reference's float64 search
    (tile-aligned shape: the fused K1 kernel; ragged shape: the general tiled kernel)."""
    from paper_2404_01847_b200 import transposable_search_conv

    rng = np.random.default_rng(17)
    r, c = shape
    nb = (r // 4) * (c // 4)
    spans = rng.integers(10, 41, size=nb)
    blocks = []
    for s in spans:
        mant = rng.integers(1, 5, size=16).astype(np.float64)  # small integers: many exact ties
        ex = rng.integers(0, s + 1, size=16)
        ex[rng.integers(0, 16)] = 0
        ex[rng.integers(0, 16)] = s  # the block spans exactly s binades
        b = mant * 2.0 ** (ex.astype(np.float64) - rng.integers(0, 60))
        b[rng.random(16) < 0.15] = 0.0
        if rng.random() < 0.05:
            b[rng.integers(0, 16)] = 2.0 ** -130  # bf16 subnormal
        b *= np.where(rng.random(16) < 0.5, -1.0, 1.0)
        blocks.append(b.reshape(4, 4))
    w = np.zeros((r, c))
    k = 0
    for i in range(r // 4):
        for j in range(c // 4):
            w[4 * i:4 * i + 4, 4 * j:4 * j + 4] = blocks[k]
            k += 1
    w = o.round_bf16(w)
    m = transposable_search_conv(to_dev_bf16(w))
    np.testing.assert_array_equal(m.idx.cpu().numpy(), o.search_pattern_idx(w))
