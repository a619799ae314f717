"""Parity at the BASELINE.json configuration shapes (SURVEY.md 8(a) parity contract).

Bit-exact: the transposable mask (pattern index of every 4x4 block), the kept values of both
compressed orientations and the tensor-core metadata (E tiles decoded to the reference nibbles
i0 | i1 << 2) at the full weight shapes of C2 (W2), C3 (W_in = [u; v] 22016 x 4096, W2
4096 x 11008) and C4 (49152 x 12288, 12288 x 49152; the float64 oracle checks 10 block-row
bands of every C4 weight -- the search and compression are block-local, and the bands sit in
different 128 x 128 tiles, CTA pairs and waves of the grid, including the first and last).

Toleranced (normwise relative error <= 1e-2, bf16 storage + fp32 accumulation, against the
float64 oracle on identical bf16-valued inputs; exact=False is the oracle's BLAS route,
within 1e-12 of the reference's gather route): the full FFN block forward + backward --
z / a, y, dx, dW_in, dbias, dW2 with the masked decay lambda = 6e-5 fused --
at C1 (768 / 3072, 2048 tokens, GELU, both the API route and the fused training path), C2
(1024 / 4096, 16384 tokens, the fused training path of bench.py), C3 (4096 / 11008 at 4096
tokens, SwiGLU and GEGLU, fused gated epilogues on two-slab tiles) and C4 (12288 / 49152 at
256 tokens, K = 49152 two-slab GEMMs).  SwiGLU has no reference implementation
(gated_ffn.py:47-50): its oracle rows are a restatement (GEGLU with silu) -- parity
UNPINNED for SwiGLU; GEGLU at the same shape is the pinned check of the gated path.
"""
import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import bf16_bits_of, need_gpu, normwise_rel

pytestmark = pytest.mark.gpu
TOL = 1e-2
LAM = 6e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    need_gpu()


def _bf16(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


def _f64(t: torch.Tensor) -> np.ndarray:
    return t.double().cpu().numpy()


def _oracle_idx(w: np.ndarray) -> np.ndarray:
    """o.search_pattern_idx over row chunks (block-local, bounded memory)."""
    out = []
    for r0 in range(0, w.shape[0], 2048):
        out.append(o.search_pattern_idx(w[r0:r0 + 2048]))
    return np.concatenate(out)


def _compress_full(w: torch.Tensor):
    import paper_2404_01847_b200._capi as C
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress

    rows, cols = w.shape
    op = CompressedOperand.empty(rows, cols, w.device)
    search_compress(w, op)
    fm = torch.empty((rows, cols // 4), dtype=torch.uint8, device=w.device)
    bm = torch.empty((cols, rows // 4), dtype=torch.uint8, device=w.device)
    C.call("s24_e_to_flat", op.fwd_e.data_ptr(), rows, cols, fm.data_ptr(), C.stream_of(fm))
    C.call("s24_e_to_flat", op.bwd_e.data_ptr(), cols, rows, bm.data_ptr(), C.stream_of(bm))
    return op, fm, bm


def _check_band(w_band: np.ndarray, r0: int, op, fm, bm):
    """Oracle search + compress of rows [r0, r0 + h) vs the GPU outputs of the full weight."""
    h = w_band.shape[0]
    idx = o.search_pattern_idx(w_band)
    np.testing.assert_array_equal(op.idx[r0 // 4:(r0 + h) // 4].cpu().numpy(), idx)
    bits = o.idx_to_bits(idx)
    kv, km = o.compress_rowwise(w_band, bits)
    np.testing.assert_array_equal(bf16_bits_of(op.fwd_vals[r0:r0 + h]), o.bf16_bits(kv))
    np.testing.assert_array_equal(fm[r0:r0 + h].cpu().numpy(), km)
    kt, kmt = o.compress_rowwise(np.ascontiguousarray(w_band.T), np.ascontiguousarray(bits.T))
    np.testing.assert_array_equal(bf16_bits_of(op.bwd_vals[:, r0 // 2:(r0 + h) // 2]), o.bf16_bits(kt))
    np.testing.assert_array_equal(bm[:, r0 // 4:(r0 + h) // 4].cpu().numpy(), kmt)


WEIGHTS = {  # name: (shape, full oracle comparison of the pattern indices)
    "c2_w2": ((1024, 4096), True),
    "c3_w_in": ((22016, 4096), True),
    "c3_w2": ((4096, 11008), True),
    "c4_w_in": ((49152, 12288), False),
    "c4_w2": ((12288, 49152), False),
}


@pytest.mark.parametrize("name", sorted(WEIGHTS))
def test_mask_values_metadata_bit_exact_at_config_weight_shapes(name):
    (rows, cols), full = WEIGHTS[name]
    w = _bf16((rows, cols), seed=rows + cols, scale=1.0 / np.sqrt(cols))
    op, fm, bm = _compress_full(w)
    torch.cuda.synchronize()
    if full:
        np.testing.assert_array_equal(op.idx.cpu().numpy(), _oracle_idx(_f64(w)))
    # bands: first, last and 8 spread over the grid (64 rows each, 16 block rows)
    h = 64
    starts = sorted({0, rows - h, *[(k * rows // 9) // h * h for k in range(1, 9)]})
    for r0 in starts:
        _check_band(_f64(w[r0:r0 + h]), r0, op, fm, bm)


def test_gated_interleave_at_c3_shape():
    """The training path compresses C3's [u; v] u/v-interleaved (perm_ff = d_ff): the pattern
    indices are the reference masks with 4-row block rows permuted."""
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress

    d, d_ff = 4096, 11008
    w = _bf16((2 * d_ff, d), seed=77, scale=1.0 / np.sqrt(d))
    plain = CompressedOperand.empty(2 * d_ff, d, "cuda")
    inter = CompressedOperand.empty(2 * d_ff, d, "cuda", perm_ff=d_ff)
    search_compress(w, plain)
    search_compress(w, inter)
    assert torch.equal(inter.mask_idx(), plain.idx)


# ---------------------------------------------------------------------------
# FFN block fwd + bwd at the configuration shapes


def _layer(act, d, d_ff, n, seed):
    r_in = 2 * d_ff if act in ("geglu", "swiglu") else d_ff
    return dict(x=_bf16((n, d), seed + 1), w_in=_bf16((r_in, d), seed + 2, 1.0 / np.sqrt(d)),
                b=_bf16((r_in,), seed + 3, 0.125), w2=_bf16((d, d_ff), seed + 4, 1.0 / np.sqrt(d_ff)),
                dy=_bf16((n, d), seed + 5, 1.0 / np.sqrt(n * d)))


def _oracle_step(c, act, mi, mo, lam):
    lo = o.Layer(_f64(c["w_in"]), _f64(c["b"]), _f64(c["w2"]), act)
    fr = o.fst_forward(lo, _f64(c["x"]), mi, mo, exact=False)
    br = o.fst_backward(lo, fr, _f64(c["dy"]), mi, mo, exact=False)
    if mi is None:  # the dense route has no decay
        br["dw_in_decayed"], br["dw2_decayed"] = br["dw_in"], br["dw2"]
    else:
        br["dw_in_decayed"] = o.masked_decay_gradient(br["dw_in"], lo.w_in, mi, lam)
        br["dw2_decayed"] = o.masked_decay_gradient(br["dw2"], lo.w2, mo, lam)
    return fr, br


def _fused_step(c, act):
    """The bench.py training step: K1 (both weights, one launch), fused forward, backward with
    the decay in the dW epilogues."""
    from paper_2404_01847_b200 import engine as E

    d_ff = c["w2"].shape[1]
    op_in = E.CompressedOperand.empty(*c["w_in"].shape, "cuda", perm_ff=d_ff if act in E.GATED else 0)
    op_out = E.CompressedOperand.empty(*c["w2"].shape, "cuda")
    E.search_compress_pair(c["w_in"], op_in, c["w2"], op_out)
    st = E.ffn_forward(c["x"], op_in, c["b"], op_out, act, fused=True)
    g = E.ffn_backward(st, c["dy"], op_in, op_out, act, w_in_dense=c["w_in"], w2_dense=c["w2"], lam=LAM)
    torch.cuda.synchronize()
    mi = o.idx_to_bits(op_in.mask_idx().cpu().numpy())
    mo = o.idx_to_bits(op_out.idx.cpu().numpy())
    return st, g, mi, mo


def _assert_step(st, g, fr, br, gated_dims=None):
    checks = [("a", st.a, fr["a"]), ("y", st.y, fr["y"]), ("dx", g.dx, br["dx"]),
              ("dbias", g.dbias_in, br["dbias_in"]), ("dw_in", g.dw_in, br["dw_in_decayed"]),
              ("dw2", g.dw2, br["dw2_decayed"])]
    errs = {k: normwise_rel(_f64(v), r) for k, v, r in checks}
    assert all(e < TOL for e in errs.values()), errs
    return errs


def test_c1_shape_api_route_and_fused_path():
    """C1 (the CPU-reference configuration): d=768, d_ff=3072, 2048 tokens, GELU -- through the
    reference API (fst_forward / fst_backward, z / GELU(z) epilogue + K7) and the fused path."""
    import paper_2404_01847_b200 as P

    c = _layer("gelu", 768, 3072, 2048, seed=101)
    layer = P.FFNLayer(c["w_in"], c["b"], c["w2"], P.Activation.GELU)
    masks = P.search_layer_masks(layer)
    mi, mo = masks.w_in.bits.cpu().numpy(), masks.w_out.bits.cpu().numpy()
    np.testing.assert_array_equal(mi, o.transposable_search_conv(_f64(c["w_in"])))
    np.testing.assert_array_equal(mo, o.transposable_search_conv(_f64(c["w2"])))
    f = P.fst_forward(layer, c["x"], masks)
    g = P.fst_backward(f, c["dy"], mvue=False, decay_lambda=LAM)
    fr, br = _oracle_step(c, "gelu", mi, mo, LAM)
    for name, ours, ref in (("z", f.z, fr["z"]), ("a", f.a, fr["a"]), ("y", f.y, fr["y"]), ("dx", g.d_x, br["dx"]),
                            ("dw1", g.d_w1, br["dw_in_decayed"]), ("db", g.d_b, br["dbias_in"]),
                            ("dw2", g.d_w2, br["dw2_decayed"])):
        assert normwise_rel(_f64(ours), ref) < TOL, name
    st, g2, mi2, mo2 = _fused_step(c, "gelu")
    np.testing.assert_array_equal(mi2, mi)
    _assert_step(st, g2, fr, br)


def test_c2_shape_fused_training_step():
    """C2 (GPT-2 medium block, 16384 tokens): the bench.py step -- fused GELU / GELU' and dGELU +
    bias-gradient epilogues, the C2 dW schedule (wave-synchronised), decay fused."""
    c = _layer("gelu", 1024, 4096, 16384, seed=202)
    st, g, mi, mo = _fused_step(c, "gelu")
    fr, br = _oracle_step(c, "gelu", mi, mo, LAM)
    np.testing.assert_array_equal(mi, o.transposable_search_conv(_f64(c["w_in"])))
    np.testing.assert_array_equal(mo, o.transposable_search_conv(_f64(c["w2"])))
    _assert_step(st, g, fr, br)


@pytest.mark.parametrize("act", ["geglu", "swiglu"])
def test_c3_shape_fused_gated_step(act):
    """C3 (d=4096, d_ff=11008) at 4096 tokens: the gated forward on the u/v-interleaved operand
    (two-slab tiles at K=4096), the gated backward + [b; c] bias gradients, dW_in in [u; v]
    order with the decay.  SwiGLU: parity unpinned (restated oracle); GEGLU: pinned."""
    c = _layer(act, 4096, 11008, 4096, seed=303)
    st, g, mi, mo = _fused_step(c, act)
    np.testing.assert_array_equal(mi[:512], o.transposable_search_conv(_f64(c["w_in"][:512])))
    fr, br = _oracle_step(c, act, mi, mo, LAM)
    _assert_step(st, g, fr, br)


def test_c4_shape_fused_step_small_batch():
    """C4 (d=12288, d_ff=49152) at 256 tokens: K = 49152 two-slab sparse GEMMs and the K = 12288
    fused epilogue GEMMs at the largest weight shape."""
    c = _layer("gelu", 12288, 49152, 256, seed=404)
    st, g, mi, mo = _fused_step(c, "gelu")
    fr, br = _oracle_step(c, "gelu", mi, mo, LAM)
    _assert_step(st, g, fr, br)


# ---------------------------------------------------------------------------
# fp32 mode (<= 2e-3 for an fp32 parity mode; C1 is the fp32 configuration)

TOL32 = 2e-3


def _layer32(act, d, d_ff, n, seed):
    """fp32 inputs that are NOT bf16-representable (the reference's float32 fused type)."""
    r_in = 2 * d_ff if act in ("geglu", "swiglu") else d_ff

    def f(shape, s, scale=1.0):
        g = torch.Generator(device="cuda").manual_seed(s)
        return torch.randn(shape, generator=g, device="cuda") * scale

    return dict(x=f((n, d), seed + 1), w_in=f((r_in, d), seed + 2, 1.0 / np.sqrt(d)), b=f((r_in,), seed + 3, 0.125),
                w2=f((d, d_ff), seed + 4, 1.0 / np.sqrt(d_ff)), dy=f((n, d), seed + 5, 1.0 / np.sqrt(n * d)))


def _fp32_case(act, d, d_ff, n, seed, sparse=True, lam=LAM):
    import paper_2404_01847_b200 as P

    c = _layer32(act, d, d_ff, n, seed)
    layer = P.FFNLayer(c["w_in"], c["b"], c["w2"], P.Activation(act))
    masks = P.search_layer_masks(layer) if sparse else None
    f = P.fst_forward(layer, c["x"], masks)
    assert f.y.dtype == torch.float32 and f.y.shape == (n, d) and f.y.stride() == (1, n)  # column-major
    g = P.fst_backward(f, c["dy"], mvue=False, decay_lambda=lam)
    mi = masks.w_in.bits.cpu().numpy() if sparse else None
    mo = masks.w_out.bits.cpu().numpy() if sparse else None
    if sparse:  # the fp32 search is bit-exact (float64 scores in the reference's add order)
        np.testing.assert_array_equal(mi, o.transposable_search_conv(_f64(c["w_in"])))
        np.testing.assert_array_equal(mo, o.transposable_search_conv(_f64(c["w2"])))
    fr, br = _oracle_step(c, act, mi, mo, lam if sparse else 0.0)
    dw_in = torch.cat([g.d_u, g.d_v]) if layer.is_gated else g.d_w1
    db = torch.cat([g.d_b, g.d_c]) if layer.is_gated else g.d_b
    errs = {k: normwise_rel(_f64(v), r) for k, v, r in (
        ("z", f.z, fr["z"]), ("a", f.a, fr["a"]), ("y", f.y, fr["y"]), ("dx", g.d_x, br["dx"]),
        ("dw_in", dw_in, br["dw_in_decayed"]), ("dbias", db, br["dbias_in"]), ("dw2", g.d_w2, br["dw2_decayed"]))}
    assert all(e < TOL32 for e in errs.values()), errs
    return errs


def test_c1_fp32_mode():
    """C1 exactly: d=768, d_ff=3072, 2048 tokens, GELU, fp32 -- the fp32 mode (split-bf16 2:4
    products, fp32 accumulation and activations, exact-erf GELU) at <= 2e-3 normwise against
    the float64 oracle on the same fp32 values, with the masked decay; bit-exact masks."""
    errs = _fp32_case("gelu", 768, 3072, 2048, seed=505)
    assert max(errs.values()) < 1e-4, errs  # what the split products actually reach


@pytest.mark.parametrize("act", ["gelu", "geglu", "swiglu", "relu"])
@pytest.mark.parametrize("sparse", [True, False])
def test_fp32_mode_small(act, sparse):
    _fp32_case(act, 256, 384, 256, seed=606 + len(act), sparse=sparse)


def test_pair_launch_mixed_super_tiles_equals_single_launches():
    """K1 of a block's two weights in one launch with two-tile super-tiles for the weight whose tile
    columns are even and single tiles for the odd one (12288 x 3968: 31 tile columns), against two
    single-weight launches (below the pairing threshold: single tiles) -- every output bit-equal --
    and oracle bands of both weights."""
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress, search_compress_pair

    w0 = _bf16((12288, 3968), seed=11, scale=1.0 / np.sqrt(3968))
    w1 = _bf16((3968, 12288), seed=12, scale=1.0 / np.sqrt(12288))
    ops = [CompressedOperand.empty(*w.shape, w.device) for w in (w0, w1)]
    search_compress_pair(w0, ops[0], w1, ops[1])
    for w, op in zip((w0, w1), ops):
        ref = CompressedOperand.empty(*w.shape, w.device)
        search_compress(w, ref)
        for a in ("idx", "fwd_vals", "bwd_vals", "fwd_e", "bwd_e"):
            assert torch.equal(getattr(op, a), getattr(ref, a)), a
    op, w = ops[1], w1
    for r0 in (0, 1984, 3904):
        idx = o.search_pattern_idx(_f64(w[r0:r0 + 64]))
        np.testing.assert_array_equal(op.idx[r0 // 4:(r0 + 64) // 4].cpu().numpy(), idx)
