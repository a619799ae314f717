"""FFN block fwd + bwd on the GPU (fst_forward / fst_backward, mvue=False)
against the float64 oracle on identical bf16-valued inputs.

Tolerance (stated): normwise relative error <= 1e-2 for every activation and
gradient (bf16 storage of z / a / dA / dZ, fp32 tensor-core accumulation);
masks must match the oracle bit-exactly."""
import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import need_gpu, normwise_rel, to_dev_bf16

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
@pytest.mark.parametrize("d,d_ff,n", [(128, 256, 128), (256, 512, 192)])
def test_fst_fwd_bwd_vs_oracle(act, d, d_ff, n):
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

    c = _case("gelu", 128, 256, 64, seed=5)
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
    with pytest.raises(NotImplementedError):
        P.fst_backward(fs, to_dev_bf16(c["dy"]))  # mvue=True default: K8 not built


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
    assert normwise_rel(st.g.t().float().cpu().numpy(), o.gelu_grad(fr["z"])) < TOL
    assert normwise_rel(st.y.float().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(g.dx.float().cpu().numpy(), br["dx"]) < TOL
    assert normwise_rel(g.dbias_in.cpu().numpy(), br["dbias_in"]) < TOL
    assert normwise_rel(g.dw_in.cpu().numpy(), o.masked_decay_gradient(br["dw_in"], c["w_in"], mi, 1e-2)) < TOL
    assert normwise_rel(g.dw2.cpu().numpy(), o.masked_decay_gradient(br["dw2"], c["w2"], mo, 1e-2)) < TOL


@pytest.mark.parametrize("act", ["gelu", "swiglu"])
def test_sparse_ffn_module_autograd_vs_oracle(act):
    from paper_2404_01847_b200.module import SparseFFN

    d, d_ff, n = 128, 256, 128
    c = _case(act, d, d_ff, n, seed=31)
    mod = SparseFFN.from_weights(to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"]), act)
    x = to_dev_bf16(c["x"])
    y = mod(x)
    y.backward(to_dev_bf16(c["dy"]))
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], "swiglu" if act == "swiglu" else "gelu")
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    assert normwise_rel(y.float().detach().cpu().numpy(), fr["y"]) < TOL
    assert normwise_rel(mod.w_in.grad.cpu().numpy(), br["dw_in"]) < TOL
    assert normwise_rel(mod.bias_in.grad.cpu().numpy(), br["dbias_in"]) < TOL
    assert normwise_rel(mod.w2.grad.cpu().numpy(), br["dw2"]) < TOL
    assert mod.mask_searches == 2
    # refresh schedule: 40 training steps -> one more search
    for _ in range(40):
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
