"""FFN block fwd + bwd on the GPU (fst_forward / fst_backward, mvue=False)
against the float64 oracle on identical bf16-valued inputs.

Tolerance (stated): normwise relative error <= 1e-2 for every activation and
gradient (bf16 storage of z / a / dA / dZ, fp32 tensor-core accumulation);
masks must match the oracle bit-exactly."""
import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import bf16_bits_of, need_gpu, normwise_rel, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    need_gpu()


def _case(act, d, d_ff, n, seed):
    r_in = 2 * d_ff if act in ("geglu", "swiglu") else d_ff
    return dict(
        x=o.round_bf16(o.det_normal((n, d), seed=seed + 1)),
        w_in=o.round_bf16(o.det_normal((r_in, d), seed=seed + 2) / np.sqrt(d)),
        bias_in=o.round_bf16(o.det_normal((r_in,), seed=seed + 3, scale_log2=-3)),
        w2=o.round_bf16(o.det_normal((d, d_ff), seed=seed + 4) / np.sqrt(d_ff)),
        dy=o.round_bf16(o.det_normal((n, d), seed=seed + 5, scale_log2=-4)),
    )


@pytest.mark.parametrize("act", ["gelu", "geglu", "relu", "swiglu"])
@pytest.mark.parametrize("d,d_ff,n", [(128, 256, 128), (256, 512, 192), (128, 256, 100), (128, 128, 4)])
def test_fst_fwd_bwd_vs_oracle(act, d, d_ff, n):
    """fst_forward / fst_backward vs the float64 oracle; token counts that are not multiples of 64
    (the reference takes any batch) run on zero-padded tokens."""
    import paper_2404_01847_b200 as P

    c = _case(act, d, d_ff, n, seed=d + d_ff + n)
    A = P.Activation(act)
    layer = P.FFNLayer(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), A)
    masks = P.search_layer_masks(layer)
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], act)
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    np.testing.assert_array_equal(masks.w_in.bits.cpu().numpy(), mi)
    np.testing.assert_array_equal(masks.w_out.bits.cpu().numpy(), mo)
    f = P.fst_forward(layer, to_dev_bf16(c["x"]), masks)
    g = P.fst_backward(f, to_dev_bf16(c["dy"]), mvue=False)
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    assert f.y.shape == (n, d) and f.y.stride() == (d, 1)  # token-major (reference: column-major, same values)
    for name, ours, ref in (("z", f.z, fr["z"]), ("a", f.a, fr["a"]), ("y", f.y, fr["y"]),
                            ("dx", g.d_x, br["dx"]), ("dw2", g.d_w2, br["dw2"])):
        err = normwise_rel(ours.float().cpu().numpy(), ref)
        assert err < TOL, (name, err)
    dw_in = torch.cat([g.d_u, g.d_v]) if layer.is_gated else g.d_w1
    db = torch.cat([g.d_b, g.d_c]) if layer.is_gated else g.d_b
    assert normwise_rel(dw_in.cpu().numpy(), br["dw_in"]) < TOL
    assert normwise_rel(db.cpu().numpy(), br["dbias_in"]) < TOL


@pytest.mark.parametrize("act,n", [("gelu", 100), ("geglu", 36)])
def test_fst_backward_mvue_ragged_batch_reference_draws(act, n):
    """fst_backward(mvue=True) (the reference default) at a batch that is not a multiple of 64:
    dW2 = MVUE(dY^T, the reference's draws for n tokens) A, on the zero-padded tensor-core path."""
    import paper_2404_01847_b200 as P

    d, d_ff = 128, 256
    c = _case(act, d, d_ff, n, seed=77 + n)
    layer = P.FFNLayer(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), P.Activation(act))
    masks = P.search_layer_masks(layer)
    f = P.fst_forward(layer, to_dev_bf16(c["x"]), masks)
    assert f.y.shape == (n, d) and f.a.shape == (n, d_ff)
    g = P.fst_backward(f, to_dev_bf16(c["dy"]), rng_seed=9, mvue=True)
    assert g.d_x.shape == (n, d)
    a = f.a.double().cpu().numpy()
    ref2 = o.round_bf16(_mvue_dense(np.ascontiguousarray(c["dy"].T), o.mvue_seed(9, 1))) @ a
    assert normwise_rel(g.d_w2.cpu().numpy(), ref2) < 5e-3


def test_fused_masked_decay_matches_oracle():
    import paper_2404_01847_b200 as P

    c = _case("geglu", 128, 256, 128, seed=99)
    layer = P.FFNLayer(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), P.Activation.GEGLU)
    masks = P.search_layer_masks(layer)
    f = P.fst_forward(layer, to_dev_bf16(c["x"]), masks)
    lam = 6e-2
    g = P.fst_backward(f, to_dev_bf16(c["dy"]), mvue=False, decay_lambda=lam)
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], "geglu")
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    ref_in = o.masked_decay_gradient(br["dw_in"], c["w_in"], mi, lam)
    ref_2 = o.masked_decay_gradient(br["dw2"], c["w2"], mo, lam)
    assert normwise_rel(torch.cat([g.d_u, g.d_v]).cpu().numpy(), ref_in) < TOL
    assert normwise_rel(g.d_w2.cpu().numpy(), ref_2) < TOL


def test_dense_path_and_mvue_flag():
    import paper_2404_01847_b200 as P

    c = _case("gelu", 128, 256, 128, seed=5)
    layer = P.FFNLayer(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), P.Activation.GELU)
    f = P.fst_forward(layer, to_dev_bf16(c["x"]), None)  # dense fine-tune path
    g = P.fst_backward(f, to_dev_bf16(c["dy"]))
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], "gelu")
    fr = o.fst_forward(lo, c["x"], None, None)
    br = o.fst_backward(lo, fr, c["dy"], None, None)
    assert normwise_rel(f.y.float().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(g.d_x.float().cpu().numpy(), br["dx"]) < TOL
    masks = P.search_layer_masks(layer)
    fs = P.fst_forward(layer, to_dev_bf16(c["x"]), masks)
    g = P.fst_backward(fs, to_dev_bf16(c["dy"]))  # mvue=True, the reference default: K8 path
    assert g.d_w1.shape == (256, 128) and torch.isfinite(g.d_w1).all()


@pytest.mark.parametrize("d,d_ff,n", [(128, 256, 128), (256, 512, 192), (256, 768, 448)])
def test_fused_training_path_vs_oracle(d, d_ff, n):
    """GEMM1 epilogue -> GELU(z), GELU'(z); GEMM3 epilogue -> dZ and the bias
    gradient (no separate activation-backward kernel)."""
    from paper_2404_01847_b200 import engine as E

    c = _case("gelu", d, d_ff, n, seed=7 * d + n)
    w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
    op_in, op_out = E.CompressedOperand.empty(d_ff, d, "cuda"), E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    st = E.ffn_forward(to_dev_bf16(c["x"]), op_in, b, op_out, "gelu", fused=True)
    assert st.z is None and st.g is not None
    g = E.ffn_backward(st, to_dev_bf16(c["dy"]), op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2)
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], "gelu")
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    assert normwise_rel(st.a.float().cpu().numpy(), fr["a"]) < TOL
    g_fm = E.aux_to_feature_major(st.g, d_ff, n)
    assert normwise_rel(g_fm.t().float().cpu().numpy(), o.gelu_grad(fr["z"])) < TOL
    assert normwise_rel(st.y.float().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(g.dx.float().cpu().numpy(), br["dx"]) < TOL
    assert normwise_rel(g.dbias_in.cpu().numpy(), br["dbias_in"]) < TOL
    assert normwise_rel(g.dw_in.cpu().numpy(), o.masked_decay_gradient(br["dw_in"], c["w_in"], mi, 1e-2)) < TOL
    assert normwise_rel(g.dw2.cpu().numpy(), o.masked_decay_gradient(br["dw2"], c["w2"], mo, 1e-2)) < TOL


@pytest.mark.parametrize("act,n", [("gelu", 128), ("swiglu", 128), ("gelu", 100), ("swiglu", 12)])
def test_sparse_ffn_module_autograd_vs_oracle(act, n):
    """The autograd module vs the float64 oracle, also at token counts that are not multiples of
    64 (zero-padded tokens, outputs / dX sliced)."""
    from paper_2404_01847_b200.module import SparseFFN

    d, d_ff = 128, 256
    c = _case(act, d, d_ff, n, seed=31)
    mod = SparseFFN.from_weights(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), act)
    x = to_dev_bf16(c["x"])
    y = mod(x)
    y.backward(to_dev_bf16(c["dy"]))
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], "swiglu" if act == "swiglu" else "gelu")
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    assert tuple(y.shape) == (n, d)
    assert normwise_rel(y.float().detach().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(mod.w_in.grad.cpu().numpy(), br["dw_in"]) < TOL
    assert normwise_rel(mod.bias_in.grad.cpu().numpy(), br["dbias_in"]) < TOL
    assert normwise_rel(mod.w2.grad.cpu().numpy(), br["dw2"]) < TOL
    assert mod.mask_searches == 2
    # refresh schedule: 40 optimizer steps -> one more search; forwards within one step
    # (gradient accumulation) neither recompress nor advance the schedule
    for _ in range(3):
        mod(x)
    assert mod.mask_searches == 2
    for _ in range(40):
        mod.mark_weights_updated()
        mod(x)
    assert mod.mask_searches == 4


@pytest.mark.parametrize("act", ["geglu", "swiglu"])
@pytest.mark.parametrize("d,d_ff,n", [(128, 256, 128), (256, 384, 192)])
def test_fused_gated_training_path_vs_oracle(act, d, d_ff, n):
    """Gate computed in GEMM1's epilogue on the u/v-interleaved operand; the gated
    backward + bias gradients in GEMM3's epilogue; dW_in returned in [u; v] order."""
    from paper_2404_01847_b200 import engine as E

    c = _case(act, d, d_ff, n, seed=3 * d + n)
    w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
    op_in = E.CompressedOperand.empty(2 * d_ff, d, "cuda", perm_ff=d_ff)
    op_out = E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    st = E.ffn_forward(to_dev_bf16(c["x"]), op_in, b, op_out, act, fused=True)
    g = E.ffn_backward(st, to_dev_bf16(c["dy"]), op_in, op_out, act, w_in_dense=w_in, w2_dense=w2, lam=1e-2)
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], act)
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    np.testing.assert_array_equal(o.idx_to_bits(op_in.mask_idx().cpu().numpy()), mi)
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    assert normwise_rel(st.a.float().cpu().numpy(), fr["a"]) < TOL
    assert normwise_rel(st.y.float().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(g.dx.float().cpu().numpy(), br["dx"]) < TOL
    assert normwise_rel(g.dbias_in.cpu().numpy(), br["dbias_in"]) < TOL
    assert normwise_rel(g.dw_in.cpu().numpy(), o.masked_decay_gradient(br["dw_in"], c["w_in"], mi, 1e-2)) < TOL
    assert normwise_rel(g.dw2.cpu().numpy(), o.masked_decay_gradient(br["dw2"], c["w2"], mo, 1e-2)) < TOL


def _mvue_dense(gt_bits_src: np.ndarray, seed: int) -> np.ndarray:
    """Oracle MVUE of the (features x tokens) matrix, as a dense sparsified matrix."""
    vals, pos = o.mvue_slots_rowwise(gt_bits_src, seed)
    dense = np.zeros_like(gt_bits_src)
    np.put_along_axis(dense, pos, vals, axis=1)
    return dense


@pytest.mark.parametrize("f,n,seed", [(256, 384, 0), (128, 256, 7), (384, 128, (12345 << 2) ^ 2),
                                      (256, 256, 2 ** 40 + 5)])
def test_mvue_kernel_bit_exact_vs_oracle(f, n, seed):
    """K8 on bf16 inputs: kept pairs, kept values (bf16) and metadata equal the
    reference MVUE (oracle pinned to reference goldens) bit-for-bit."""
    import paper_2404_01847_b200._capi as C
    from paper_2404_01847_b200 import engine as E

    x = o.det_normal((f, n), seed=f + n)
    u = (o._splitmix64(f * n, 3 + n) % np.uint64(10)).reshape(f, n)
    x = np.where(u < 2, 0.0, np.where(u == 9, x * 2.0 ** 10, x))
    x = o.round_bf16(x)  # features x tokens, zeros + dominant entries
    g = to_dev_bf16(np.ascontiguousarray(x.T))  # token-major input
    vals, e, pairs = E.mvue_compress(g, seed, want_pairs=True)
    rv, _, ridx = o.mvue_kept(x.reshape(-1, 4), seed)
    np.testing.assert_array_equal(pairs.cpu().numpy().reshape(-1), ridx)
    np.testing.assert_array_equal(bf16_bits_of(vals).reshape(-1), o.bf16_bits(o.round_bf16(rv.reshape(-1))))
    meta = torch.empty((f, n // 4), dtype=torch.uint8, device="cuda")
    C.call("s24_e_to_flat", e.data_ptr(), f, n, meta.data_ptr(), C.stream_of(meta))
    nib = np.array([4, 8, 12, 9, 13, 14], dtype=np.uint8)[ridx]
    np.testing.assert_array_equal(meta.cpu().numpy().reshape(-1), nib)


def test_mvue_sparse_dw_gemm_and_unbiasedness():
    """MVUE-sparse dW GEMM == the oracle's sparsified product on the same input;
    the estimator averages to the dense gradient (Monte Carlo, 4 sigma)."""
    from paper_2404_01847_b200 import engine as E

    f, n, dcols = 256, 512, 256
    gx = o.round_bf16(o.det_normal((n, f), seed=1))
    b = o.round_bf16(o.det_normal((n, dcols), seed=2))
    gd, bd = to_dev_bf16(gx), to_dev_bf16(b)
    out = torch.empty((f, dcols), dtype=torch.float32, device="cuda")
    vals, e, _ = E.mvue_compress(gd, 99)
    E.spmm_dw(vals, e, f, n, bd, True, dcols, out)
    ref = o.round_bf16(_mvue_dense(np.ascontiguousarray(gx.T), 99)) @ b
    assert normwise_rel(out.cpu().numpy(), ref) < 2e-3
    dense = gx.T @ b
    for exact in (True, False):
        _check_unbiased(E, gd, bd, f, n, dcols, out, dense, exact)


def _check_unbiased(E, gd, bd, f, n, dcols, out, dense, exact):
    acc = np.zeros_like(dense)
    acc2 = np.zeros_like(dense)
    trials = 48
    for s in range(trials):
        vals, e, _ = E.mvue_compress(gd, 1000 + s, exact=exact)
        E.spmm_dw(vals, e, f, n, bd, True, dcols, out)
        r = out.double().cpu().numpy()
        acc += r
        acc2 += r * r
    mean = acc / trials
    se = np.sqrt(np.maximum(acc2 / trials - mean ** 2, 0) / trials) + 1e-3 * np.abs(dense).mean()
    z = np.abs(mean - dense) / se
    assert np.mean(z < 4.0) > 0.995, np.mean(z < 4.0)


@pytest.mark.parametrize("f,n,seed,gff", [(256, 192, 3, 0), (128, 64, 11, 0), (256, 196, 2 ** 33 + 1, 0),
                                          (256, 320, 5, 128)])
def test_mvue_kernel_ragged_tokens_bit_exact(f, n, seed, gff):
    """Token counts that are not multiples of 128 (the reference takes any multiple of 4): the
    operand covers n rounded up to 128 tokens, the first n are the reference's draws for n tokens
    (stream index row * n/4 + group) bit-for-bit, the padded groups are zero; gated row order
    included."""
    from paper_2404_01847_b200 import engine as E

    x = o.round_bf16(o.det_normal((f, n), seed=f + n + 1))  # features x tokens
    g = to_dev_bf16(np.ascontiguousarray(x.T))
    vals, e, pairs = E.mvue_compress(g, seed, gate_ff=gff, want_pairs=True)
    n_pad = (n + 127) // 128 * 128
    assert tuple(vals.shape) == (f, n_pad // 2) and tuple(pairs.shape) == (f, n_pad // 4)
    if gff:  # feature p of the operand is row gate_row(p) of [u; v] for the draw
        p = np.arange(f)
        rows = np.where(p % 32 < 16, 16 * (p // 32) + p % 32, gff + 16 * (p // 32) + p % 32 - 16)
        src = np.empty_like(x)
        src[rows] = x
        rv, _, ridx = o.mvue_kept(src.reshape(-1, 4), seed)
        rv, ridx = rv.reshape(f, -1)[rows], ridx.reshape(f, -1)[rows]
    else:
        rv, _, ridx = o.mvue_kept(x.reshape(-1, 4), seed)
        rv, ridx = rv.reshape(f, -1), ridx.reshape(f, -1)
    np.testing.assert_array_equal(pairs.cpu().numpy()[:, : n // 4], ridx)
    np.testing.assert_array_equal(bf16_bits_of(vals[:, : n // 2].contiguous()).reshape(f, -1),
                                  o.bf16_bits(o.round_bf16(rv)).reshape(f, -1))
    assert not vals[:, n // 2:].float().abs().sum().item()
    # the padded operand through the 2:4 weight-gradient GEMM == the oracle product on n tokens
    b = o.round_bf16(o.det_normal((n, 128), seed=7))
    out = torch.empty((f, 128), dtype=torch.float32, device="cuda")
    E.spmm_dw(vals, e, f, n_pad, E.pad_tokens(to_dev_bf16(b)), True, 128, out)
    dense = _mvue_dense(src, seed)[rows] if gff else _mvue_dense(x, seed)
    ref = o.round_bf16(dense) @ b
    assert normwise_rel(out.cpu().numpy(), ref) < 2e-3


@pytest.mark.parametrize("act,n", [("gelu", 256), ("swiglu", 256), ("gelu", 192), ("swiglu", 64)])
def test_mvue_training_path_vs_oracle_on_same_gradients(act, n):
    """fst_backward(mvue=True) semantics on the fused training path: the dW
    outputs equal the oracle MVUE products of the GPU's own dY / dZ (identical
    inputs -> identical draws), with the decay fused; also for token counts that are not
    multiples of 128 (padded operands, the reference's draws for the real tokens)."""
    from paper_2404_01847_b200 import engine as E

    d, d_ff = 128, 256
    c = _case(act, d, d_ff, n, seed=5 + n)
    w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
    gated = act == "swiglu"
    op_in = E.CompressedOperand.empty(w_in.shape[0], d, "cuda", perm_ff=d_ff if gated else 0)
    op_out = E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    x, dy = to_dev_bf16(c["x"]), to_dev_bf16(c["dy"])
    st = E.ffn_forward(x, op_in, b, op_out, act, fused=True)
    g = E.ffn_backward(st, dy, op_in, op_out, act, w_in_dense=w_in, w2_dense=w2, lam=1e-2, mvue=True,
                       rng_seed=31)
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    # dW2 = MVUE(dY^T, salt 1) A
    a = st.a.double().cpu().numpy()
    ref2 = o.round_bf16(_mvue_dense(np.ascontiguousarray(c["dy"].T), o.mvue_seed(31, 1))) @ a
    ref2 = o.masked_decay_gradient(ref2, c["w2"], mo, 1e-2)
    assert normwise_rel(g.dw2.cpu().numpy(), ref2) < 5e-3
    # dW_in = MVUE(dZ^T, salt 2) X, dZ in [u; v] order for the draw
    dzp = _dz_from(st, dy, op_in, op_out, act)
    if gated:
        p = np.arange(2 * d_ff)
        orig = np.where(p % 32 < 16, 16 * (p // 32) + p % 32, d_ff + 16 * (p // 32) + p % 32 - 16)
        dz_orig = np.empty_like(dzp)
        dz_orig[:, orig] = dzp
    else:
        dz_orig = dzp
    ref1 = o.round_bf16(_mvue_dense(np.ascontiguousarray(dz_orig.T), o.mvue_seed(31, 2))) @ c["x"]
    ref1 = o.masked_decay_gradient(ref1, c["w_in"], mi, 1e-2)
    assert normwise_rel(g.dw_in.cpu().numpy(), ref1) < 5e-3


def _dz_from(st, dy, op_in, op_out, act):
    """The fused backward's dZ (token-major, interleaved for gated) recomputed by the same kernels."""
    import paper_2404_01847_b200._capi as C
    from paper_2404_01847_b200 import engine as E

    n, d_ff = st.a.shape
    r_in = op_in.rows
    dz = torch.empty((n, r_in), dtype=torch.bfloat16, device="cuda")
    db = torch.zeros(r_in, dtype=torch.float32, device="cuda")
    if st.g2 is not None:
        E.spmm(op_out.bwd_vals, op_out.bwd_e, d_ff, dy.shape[1], dy, False, n, dz, epi=C.EPI_DGATED, aux=st.g,
               aux2=st.g2, dbias=db, out_t=True, gate_ff=d_ff)
    else:
        E.spmm(op_out.bwd_vals, op_out.bwd_e, d_ff, dy.shape[1], dy, False, n, dz, epi=C.EPI_DGELU, aux=st.g,
               dbias=db, out_t=True)
    return dz.double().cpu().numpy()


def test_backward_bucket_views_and_grads_ready_hook():
    """ffn_backward writes dW_in / dbias / dW2 into caller views (the DP gradient bucket) and
    calls grads_ready() once all of them are enqueued, before dX (bench.py starts the
    all-reduce there); results equal the plain call."""
    from paper_2404_01847_b200 import engine as E

    d, d_ff, n = 128, 256, 128
    c = _case("gelu", d, d_ff, n, seed=5)
    w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
    op_in, op_out = E.CompressedOperand.empty(d_ff, d, "cuda"), E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    x, dy = to_dev_bf16(c["x"]), to_dev_bf16(c["dy"])
    st = E.ffn_forward(x, op_in, b, op_out, "gelu", fused=True)
    ref = E.ffn_backward(st, dy, op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2)
    bucket = torch.full((w_in.numel() + d_ff + w2.numel(),), float("nan"), device="cuda")
    dwi, db, dw2 = (bucket[:w_in.numel()].view(w_in.shape), bucket[w_in.numel():w_in.numel() + d_ff],
                    bucket[w_in.numel() + d_ff:].view(w2.shape))
    calls = []
    g = E.ffn_backward(st, dy, op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2, dw_in_out=dwi,
                       dw2_out=dw2, dbias_out=db, grads_ready=lambda: calls.append(1))
    torch.cuda.synchronize()
    assert calls == [1]
    assert g.dw_in.data_ptr() == dwi.data_ptr() and g.dbias_in.data_ptr() == db.data_ptr()
    assert torch.isfinite(bucket).all()
    assert torch.equal(dwi, ref.dw_in) and torch.equal(dw2, ref.dw2) and torch.equal(g.dx, ref.dx)
    assert torch.allclose(db, ref.dbias_in, rtol=1e-5, atol=1e-6)


def test_training_step_cuda_graph_capture_and_replay():
    """The C-ABI calls are stream-ordered and sync-free, so a whole step (K2, fused GEMMs,
    wave-synchronised dW GEMMs with their self-resetting counters) captures into a CUDA graph;
    replays reproduce the eager results bit for bit."""
    from paper_2404_01847_b200 import engine as E

    d, d_ff, n = 256, 512, 1024
    c = _case("gelu", d, d_ff, n, seed=11)
    w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
    x, dy = to_dev_bf16(c["x"]), to_dev_bf16(c["dy"])
    op_in, op_out = E.CompressedOperand.empty(d_ff, d, "cuda"), E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    dwi = torch.empty(d_ff, d, device="cuda")
    dw2 = torch.empty(d, d_ff, device="cuda")
    db = torch.empty(d_ff, device="cuda")

    def step():
        E.compress_values_pair(w_in, op_in, w2, op_out)
        st = E.ffn_forward(x, op_in, b, op_out, "gelu", fused=True)
        g = E.ffn_backward(st, dy, op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2, dw_in_out=dwi,
                           dw2_out=dw2, dbias_out=db)
        return st.y, g.dx

    y0, dx0 = step()
    ref = [t.clone() for t in (y0, dx0, dwi, dw2, db)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm the stream
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        yg, dxg = step()
    for _ in range(3):
        for t in (dwi, dw2, db):
            t.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        for got, want in zip((yg, dxg, dwi, dw2, db), ref):
            assert torch.equal(got, want) or torch.allclose(got, want, rtol=0, atol=1e-6)


@pytest.mark.parametrize("d,d_ff,n", [(256, 512, 1024), (1024, 4096, 2048)])
def test_dx_accumulate_into_residual_gradient(d, d_ff, n):
    """ffn_backward(dx_accumulate=dh): the dX GEMM add-reduces into the residual gradient
    (S24_EPI_STORE_ADD, one-slab and two-slab tiles), even when dh is the upstream dy itself:
    result == rn(dh + dX) of the plain path; the other gradients are unchanged."""
    from paper_2404_01847_b200 import engine as E
    from paper_2404_01847_b200 import _capi as C

    g = torch.Generator(device="cpu").manual_seed(d + n)
    w_in = (torch.randn(d_ff, d, generator=g) / d ** 0.5).to(torch.bfloat16).cuda()
    w2 = (torch.randn(d, d_ff, generator=g) / d_ff ** 0.5).to(torch.bfloat16).cuda()
    b = torch.zeros(d_ff, dtype=torch.bfloat16, device="cuda")
    x = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
    dy = torch.randn(n, d, generator=g).to(torch.bfloat16).cuda()
    op_in, op_out = E.CompressedOperand.empty(d_ff, d, "cuda"), E.CompressedOperand.empty(d, d_ff, "cuda")
    E.search_compress(w_in, op_in)
    E.search_compress(w2, op_out)
    st = E.ffn_forward(x, op_in, b, op_out, "gelu", fused=True)
    ref = E.ffn_backward(st, dy, op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2)
    want = (dy.float() + ref.dx.float()).to(torch.bfloat16)
    dh = dy.clone()
    got = E.ffn_backward(st, dh, op_in, op_out, "gelu", w_in_dense=w_in, w2_dense=w2, lam=1e-2, dx_accumulate=dh)
    torch.cuda.synchronize()
    assert got.dx.data_ptr() == dh.data_ptr()
    assert torch.equal(got.dw_in, ref.dw_in) and torch.equal(got.dw2, ref.dw2)
    diff = (dh.float() - want.float()).abs()
    ulp = want.float().abs() * 2.0 ** -7 + 1e-30
    assert bool((diff <= ulp).all()), float((diff / ulp).max())
    # the accumulate epilogue needs the token-major store
    with pytest.raises(RuntimeError):
        C.call("s24_spmm", op_in.bwd_vals.data_ptr(), op_in.bwd_e.data_ptr(), d, d_ff, st.a.data_ptr(), 0, d_ff,
               n, dh.data_ptr(), n, None, C.EPI_STORE_ADD, None, 0, None, None, 0, 0, None, 0, C.stream_of(dh))


def _mvue_corpus(f, n, kind, seed):
    """features x tokens bf16-valued corpora for the certificate: Gaussian, small integers (exact
    ties, clamp boundaries amax == rest, rounding midpoints of g / pi), wide exponent spans."""
    x = o.det_normal((f, n), seed=seed)
    if kind == "ints":
        x = np.floor(np.abs(x) * 1.7) * np.sign(x)  # {0, +-1, +-2, +-3, ...}
    elif kind == "span":
        sh = (o._splitmix64(f * n, seed + 11) % np.uint64(60)).astype(np.int64).reshape(f, n) - 30
        x = x * np.exp2(sh.astype(np.float64))
    elif kind == "pow2":
        sh = (o._splitmix64(f * n, seed + 13) % np.uint64(4)).astype(np.int64).reshape(f, n)
        x = np.sign(x) * np.exp2(sh.astype(np.float64)) * ((o._splitmix64(f * n, seed + 17) % np.uint64(3)) > 0
                                                            ).reshape(f, n)
    return o.round_bf16(x)


@pytest.mark.parametrize("kind", ["normal", "ints", "span", "pow2"])
@pytest.mark.parametrize("gate_ff", [0, 512])
def test_mvue_certified_fast_path_equals_float64_path(kind, gate_ff):
    """Exact mode's common case runs in fp32 under an error certificate and falls back to the
    float64 reference computation when a decision is within the bound; exact=2 forces float64 for
    every group.  Both must give identical kept pairs, values and metadata (2 M groups per corpus)."""
    from paper_2404_01847_b200 import engine as E

    f, n = 1024, 8192
    x = _mvue_corpus(f, n, kind, seed=len(kind) * 7 + gate_ff)
    g = to_dev_bf16(np.ascontiguousarray(x.T))
    outs = [E.mvue_compress(g, 4242, gate_ff=gate_ff, want_pairs=True, exact=mode) for mode in (1, 2)]
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                           b.view(torch.uint8) if b.dtype != torch.uint8 else b)


def test_mvue_gated_stream_bit_exact_vs_oracle():
    """Gated operand (u / v rows interleaved in 16-row groups): feature p of G draws from the
    stream of row gate_row(p) of [u; v] -- the per-CTA base states and row-table jumps."""
    from paper_2404_01847_b200 import engine as E

    ff, n, seed = 256, 512, 77
    f = 2 * ff
    x = _mvue_corpus(f, n, "normal", seed=5)  # interleaved feature order
    rows = np.array([16 * (p // 32) + (p % 32) if p % 32 < 16 else ff + 16 * (p // 32) + (p % 32) - 16
                     for p in range(f)])
    xr = np.empty_like(x)
    xr[rows] = x  # [u; v] order: row r holds feature p with gate_row(p) = r
    g = to_dev_bf16(np.ascontiguousarray(x.T))
    vals, e, pairs = E.mvue_compress(g, seed, gate_ff=ff, want_pairs=True)
    rv, _, ridx = o.mvue_kept(xr.reshape(-1, 4), seed)
    ridx = ridx.reshape(f, n // 4)[rows]
    rv = rv.reshape(f, n // 2)[rows]
    np.testing.assert_array_equal(pairs.cpu().numpy(), ridx)
    np.testing.assert_array_equal(bf16_bits_of(vals), o.bf16_bits(o.round_bf16(rv)))
