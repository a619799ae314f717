"""Pin the CPU oracle (oracle/s24_oracle.py) against golden vectors that the
reference package itself produced (tests/golden/make_golden.py).  CPU only."""

import hashlib
import os

import numpy as np
import pytest

from oracle import s24_oracle as o
from make_golden import fst_cases, mask_corpora

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_pattern_table_matches_reference_golden():
    pats, pos = o.pattern_table()
    text = o.pattern_text(pats)
    assert len(pats) == 90
    assert hashlib.md5(text.encode()).hexdigest() == "313a02e787e3fa096f2727e789833468"
    assert text == open(os.path.join(GOLDEN, "patterns.txt")).read()
    # every row / column sums to two; closed under transpose
    assert (pats.sum(axis=1) == 2).all() and (pats.sum(axis=2) == 2).all()
    flat = {tuple(p.reshape(16)) for p in pats}
    assert all(tuple(p.T.reshape(16)) in flat for p in pats)
    assert list(pos[0]) == [2, 3, 6, 7, 8, 9, 12, 13]


@pytest.fixture(scope="module")
def corpora():
    return mask_corpora()


@pytest.mark.parametrize("name", ["gauss_f64", "gauss_bf16", "int_ties", "kats", "c1_w1_f32", "c2_w1_bf16"])
def test_search_idx_bit_exact(name, corpora, mask_golden):
    w, _ = corpora[name]
    idx = o.search_pattern_idx(w)
    assert idx.dtype == np.uint8
    np.testing.assert_array_equal(idx, mask_golden[f"{name}.idx"])
    bits = o.idx_to_bits(idx)
    o.validate_transposable(bits)
    o.validate_transposable(bits.T)


@pytest.mark.parametrize("name", ["gauss_bf16", "int_ties", "kats"])
def test_compress_both_orientations_bit_exact(name, corpora, mask_golden):
    w, _ = corpora[name]
    np.testing.assert_array_equal(o.bf16_bits(w), mask_golden[f"{name}.w_bf16"])
    bits = o.idx_to_bits(mask_golden[f"{name}.idx"])
    kv, meta = o.compress_rowwise(w, bits)
    np.testing.assert_array_equal(meta, mask_golden[f"{name}.fwd_meta"])
    np.testing.assert_array_equal(o.bf16_bits(kv), mask_golden[f"{name}.fwd_values"])
    kvt, metat = o.compress_rowwise(np.ascontiguousarray(w.T), np.ascontiguousarray(bits.T))
    np.testing.assert_array_equal(metat, mask_golden[f"{name}.bwd_meta"])
    np.testing.assert_array_equal(o.bf16_bits(kvt), mask_golden[f"{name}.bwd_values"])
    # round trip
    np.testing.assert_array_equal(o.decompress_rowwise(kv, meta, w.shape[1]), w * bits)


def test_kat_specifics(mask_golden):
    idx = mask_golden["kats.idx"]
    assert idx[0, 0] == 0  # all-equal block -> pattern 0 (first max)
    assert idx[0, 1] == 0  # all-zero block -> pattern 0
    assert idx[0, 2] == 37  # dominant pattern 37 (test_sparsity.py:129-134)
    assert idx[0, 3] == 5
    assert idx[0, 5] == 0  # sign does not matter


def test_meta_nibble_kat():
    # group [0, 5, 0, -3] -> values (5, -3), meta 1 | 3 << 2 = 13 (test_spmm.py:25-29)
    kv, meta = o.compress_rowwise(np.array([[0.0, 5.0, 0.0, -3.0]]), np.array([[0, 1, 0, 1]]))
    assert list(kv[0]) == [5.0, -3.0] and meta[0, 0] == 13
    with pytest.raises(o.FormatError):
        o.decompress_rowwise(np.zeros((1, 2)), np.array([[2 | (1 << 2)]], dtype=np.uint8), 4)


@pytest.mark.parametrize("act", ["gelu", "geglu", "relu"])
def test_fst_forward_backward_matches_reference(act, fst_golden):
    c = fst_cases()[act]
    g = {k.split(".", 1)[1]: v for k, v in fst_golden.items() if k.startswith(act + ".")}
    for k in ("x", "w_in", "bias_in", "w2", "dy"):
        np.testing.assert_array_equal(c[k], g[k])
    layer = o.Layer(c["w_in"], c["bias_in"], c["w2"], act)
    mi, mo = g["mask_in"], g["mask_out"]
    np.testing.assert_array_equal(mi, o.transposable_search_conv(c["w_in"]))
    for exact in (True, False):
        f = o.fst_forward(layer, c["x"], mi, mo, exact=exact)
        b = o.fst_backward(layer, f, c["dy"], mi, mo, exact=exact)
        tol = 0 if exact else 1e-12
        for ours, ref in ((f["z"], g["z"]), (f["a"], g["a"]), (f["y"], g["y"]), (b["dx"], g["dx"]),
                          (b["dw_in"], g["dw_in"]), (b["dbias_in"], g["dbias_in"]), (b["dw2"], g["dw2"])):
            np.testing.assert_allclose(ours, ref, rtol=tol, atol=1e-13 if exact else 1e-12)
    dec = o.masked_decay_gradient(b["dw_in"], c["w_in"], mi, 6e-5)
    np.testing.assert_allclose(dec, g["dw_in_decayed"], rtol=1e-12, atol=1e-14)
    fd = o.fst_forward(layer, c["x"], None, None)
    bd = o.fst_backward(layer, fd, c["dy"], None, None)
    np.testing.assert_allclose(fd["y"], g["dense_y"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(bd["dx"], g["dense_dx"], rtol=1e-12, atol=1e-13)


def test_geglu_gate(fst_golden):
    c = fst_cases()["geglu"]
    r = c["w2"].shape[1]
    z = c["x"] @ c["w_in"].T + c["bias_in"]
    out = o.gate(z[:, :r], z[:, r:])
    np.testing.assert_allclose(out, fst_golden["geglu_forward.out"], rtol=1e-12, atol=1e-13)


def test_switch_step_kat():
    assert o.switch_step(60000, 1 / 6) == 50000  # test_trainer.py:68-71


def test_ref_kernels_agree_with_restatement():
    k = o.ref_kernels()
    if k is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    _, pos = o.pattern_table()
    blocks = np.abs(rng.standard_normal((300, 16)))
    s1, b1 = k.pattern_scores(blocks, pos)
    s2, b2 = o.pattern_scores(blocks, pos)
    assert s1.tobytes() == s2.tobytes() and (b1 == b2).all()


def test_mvue_oracle_bit_exact_vs_reference():
    from make_golden import mvue_cases

    g = dict(np.load(os.path.join(GOLDEN, "mvue_golden.npz")))
    for i, (shape, seed) in enumerate(mvue_cases()):
        x = g[f"case{i}.x"]
        assert int(g[f"case{i}.seed"]) == seed
        pi = o.mvue_inclusion_probs(x.reshape(-1, 4))
        assert pi.tobytes() == g[f"case{i}.pi"].tobytes()
        assert o.mvue_pair_probs(pi).tobytes() == g[f"case{i}.pairs"].tobytes()
        vals, pos = o.mvue_slots_rowwise(x, seed)
        assert vals.tobytes() == g[f"case{i}.values"].tobytes()
        np.testing.assert_array_equal(pos, g[f"case{i}.pos"])
        # every group keeps exactly two entries; unbiased marginals sum to 2
        np.testing.assert_allclose(pi.sum(axis=1), 2.0, rtol=1e-12)


@pytest.mark.parametrize("act", ["gelu", "geglu", "relu"])
def test_fst_backward_mvue_matches_reference(act, fst_golden):
    g = dict(np.load(os.path.join(GOLDEN, "mvue_golden.npz")))
    c = fst_cases()[act]
    fg = {k.split(".", 1)[1]: v for k, v in fst_golden.items() if k.startswith(act + ".")}
    layer = o.Layer(c["w_in"], c["bias_in"], c["w2"], act)
    f = o.fst_forward(layer, c["x"], fg["mask_in"], fg["mask_out"], exact=True)
    for seed in (0, 12345):
        b = o.fst_backward_mvue(layer, f, c["dy"], fg["mask_in"], fg["mask_out"], rng_seed=seed)
        np.testing.assert_allclose(b["dw_in"], g[f"fst_{act}_{seed}.dw_in"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(b["dw2"], g[f"fst_{act}_{seed}.dw2"], rtol=1e-12, atol=1e-13)


def _optim_golden():
    return dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "optim_golden.npz")))


@pytest.mark.parametrize("mode", ["none", "on_gradients", "on_weights"])
def test_train_update_matches_reference_bit_exact(mode):
    """oracle Adam + masked decay (optim.py:105-147, trainer.py:438-447) == the reference, bitwise."""
    gd = _optim_golden()
    w, u, v = gd["w0"], np.zeros_like(gd["w0"]), np.zeros_like(gd["w0"])
    for t in range(3):
        w, u, v = o.train_update(w, u, v, t + 1, gd[f"g{t}"], gd["mask"], float(gd[f"{mode}.lam"]), mode, lr=3e-3)
    for k, a in (("w", w), ("u", u), ("v", v)):
        assert np.array_equal(a.view(np.uint64), gd[f"{mode}.{k}"].view(np.uint64)), k


def test_flip_statistics_match_reference():
    gd = _optim_golden()
    ma, mb = o.transposable_search_conv(gd["flip.wa"]), o.transposable_search_conv(gd["flip.wb"])
    assert o.flip_rate(ma, mb) == float(gd["flip.rate"])
    assert np.array_equal(o.block_flips(ma, mb), gd["flip.block_flips"])


@pytest.mark.parametrize("name", ["gauss_bf16", "int_ties", "kats"])
def test_greedy_and_prune2of4_oracle_match_reference(name):
    """oracle greedy search / prune_2of4 (_core.pyx:113-219) == the reference on the tie-heavy corpora."""
    gd = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "comparators_golden.npz")))
    w, _ = mask_corpora()[name]
    bits = o.transposable_search_greedy(w)
    o.validate_transposable(bits)
    pats, _ = o.pattern_table()
    assert np.array_equal(o.idx_to_bits(gd[f"{name}.greedy_idx"]), bits)
    assert np.array_equal(o.prune_2of4_bits(w), gd[f"{name}.prune_row"])
    assert np.array_equal(o.prune_2of4_bits(w, colwise=True), gd[f"{name}.prune_col"])


def _packed_golden():
    return dict(np.load(os.path.join(GOLDEN, "packed_golden.npz")))


@pytest.mark.parametrize("name", ["a", "b", "c"])
@pytest.mark.parametrize("colwise", [False, True])
def test_packed_format_oracle_matches_reference(name, colwise):
    """compress / decompress (spmm.py:92-129) restated == the reference in both directions."""
    gd = _packed_golden()
    d = "col" if colwise else "row"
    w, bits = gd[f"{name}.w"], gd[f"{name}.{d}.bits"]
    assert np.array_equal(o.prune_2of4_bits(w, colwise=colwise), bits)
    vals, meta = o.compress_groups(w * bits, bits, colwise)
    assert np.array_equal(vals, gd[f"{name}.{d}.values"]) and np.array_equal(meta, gd[f"{name}.{d}.meta"])
    assert np.array_equal(o.decompress_groups(vals, meta, w.shape, colwise), gd[f"{name}.{d}.dense"])


def test_packed_products_oracle_matches_reference():
    """spmm / spmm_right (spmm.py:165-190) are the dense products of the decompressed operands."""
    gd = _packed_golden()
    w, bits = gd["b.w"], gd["b.row.bits"]
    dense = o.decompress_groups(*o.compress_groups(w * bits, bits, False), w.shape, False)
    np.testing.assert_allclose(dense @ gd["spmm.rhs"], gd["spmm.out"], rtol=1e-12, atol=1e-12)
    bt = o.prune_2of4_bits(np.ascontiguousarray(w.T), colwise=True)
    np.testing.assert_allclose(gd["spmm_right.lhs"] @ (w.T * bt), gd["spmm_right.out"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("i", range(4))
def test_mvue_prune_oracle_bit_exact_vs_reference(i):
    gd = _packed_golden()
    for colwise in (False, True):
        d = "col" if colwise else "row"
        vals, bits = o.mvue_prune(gd[f"mvue{i}.g"], colwise, int(gd[f"mvue{i}.seed"]))
        assert np.array_equal(vals.view(np.uint64), gd[f"mvue{i}.{d}.values"].view(np.uint64))
        assert np.array_equal(bits, gd[f"mvue{i}.{d}.bits"])


def test_block_flip_stats_oracle_bit_exact_vs_reference():
    gd = _packed_golden()
    flips, gaps = o.block_flip_stats([gd["flip3.wa"], gd["flip3.wb"], gd["flip3.wc"]])
    assert np.array_equal(flips, gd["flip3.block_flips"])
    assert np.array_equal(gaps.view(np.uint64), gd["flip3.block_gaps"].view(np.uint64))
    assert np.array_equal(o.block_gaps(gd["ties.w"]), gd["ties.block_gaps"])
    assert (gd["ties.block_gaps"] == 0).any()  # the corpus exercises tied top-2 scores
