"""Generate golden vectors from the REFERENCE package itself.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py
It copies /root/reference/pkg to /tmp/refpkg_golden, builds the reference's
Cython core there (its own setup.py, -O3 -ffp-contract=off), imports
`sparse24` from that copy and records inputs + reference outputs as .npz
fixtures next to this script.  The fixtures are committed; the GPU box never
needs /root/reference.

Inputs are integer-generated (oracle.s24_oracle.det_normal) and rounded to
bf16 or fp32 where stated, so they are bit-reproducible everywhere.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
from oracle import s24_oracle as o  # noqa: E402

REF = "/root/reference/pkg"
BUILD = "/tmp/refpkg_golden"


def import_reference():
    if not os.path.isdir(os.path.join(BUILD, "src")):
        shutil.copytree(REF, BUILD)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=BUILD,
                       check=True, capture_output=True)
    sys.path.insert(0, os.path.join(BUILD, "src"))
    import sparse24  # noqa: F401

    assert sparse24.BACKEND == "cython", sparse24.BACKEND
    return sparse24


def ref_search(s24, w):
    """Reference mask, per-block idx and both compressed orientations."""
    from sparse24.matrix import Direction
    from sparse24.sparsity import Mask24, SparseEstimate, _blocks_16
    from sparse24.spmm import compress

    table = s24.enumerate_patterns()
    mask = s24.transposable_search_conv(w)
    blocks = _blocks_16(mask.bits).reshape(-1, 16)
    idx = np.array([table.index_of(b.reshape(4, 4)) for b in blocks], dtype=np.uint8)
    r, c = w.shape
    idx = idx.reshape(r // 4, c // 4)
    fwd = compress(SparseEstimate(w * mask.bits, Mask24(mask.bits, Direction.ROW_WISE)))
    wt, mt = np.ascontiguousarray(w.T), np.ascontiguousarray(mask.bits.T)
    bwd = compress(SparseEstimate(wt * mt, Mask24(mt, Direction.ROW_WISE)))
    return dict(
        bits=mask.bits,
        idx=idx,
        fwd_values=fwd.values.reshape(r, c // 2),
        fwd_meta=fwd.meta.reshape(r, c // 4),
        bwd_values=bwd.values.reshape(c, r // 2),
        bwd_meta=bwd.meta.reshape(c, r // 4),
    )


def mask_corpora():
    """name -> (input float64 array, storage dtype tag)."""
    out = {}
    # reference acceptance corpus style: 1000 Gaussian 16x16 blocks in f64
    out["gauss_f64"] = (o.det_normal((1000 * 16, 16), seed=2024), "f64")
    # bf16 N(0, 2^-6 ~ 0.0156): ~0.3% exact top-2 ties
    out["gauss_bf16"] = (o.round_bf16(o.det_normal((512, 512), seed=7, scale_log2=-6)), "bf16")
    # small-integer blocks: heavy ties (sparsity corpora, verify.py:193-214)
    ints = (o._splitmix64(256 * 256, 11) % np.uint64(5)).astype(np.float64) - 2.0
    out["int_ties"] = (ints.reshape(256, 256), "bf16")
    # all-equal, all-zero, dominant-pattern KATs (test_sparsity.py:129-165),
    # stuck-greedy block (test_sparsity.py:170-182), huge exponent spans
    pats, _ = o.pattern_table()
    kat = np.zeros((16, 64))
    kat[0:4, 0:4] = 1.0
    kat[0:4, 4:8] = 0.0
    kat[0:4, 8:12] = np.where(pats[37] > 0, 10.0, 1.0)
    kat[0:4, 12:16] = np.where(pats[5] > 0, 50.0, 1.0)
    kat[0:4, 16:20] = [[10, 10, 0.01, 0.3], [10, 10, 0.01, 0.3],
                       [0.02, 0.02, 10, 0.3], [0.4, 0.4, 10, 9]]
    kat[0:4, 20:24] = -1.0  # sign must not matter
    kat[4:8, :] = o.round_bf16(o.det_normal((4, 64), seed=3))
    # blocks mixing 2^60 and 2^-60 magnitudes: exponent span > 42 so the
    # reference's ascending f64 sum rounds (the GPU slow path must match)
    span = o.det_normal((8, 64), seed=5)
    span *= np.where((np.arange(8 * 64).reshape(8, 64) % 3) == 0, 2.0 ** 60, 2.0 ** -60)
    kat[8:16, :] = o.round_bf16(span)
    out["kats"] = (o.round_bf16(kat), "bf16")
    # fp32 weights at the C1 (CPU-oracle) shape, d=768 d_ff=3072
    out["c1_w1_f32"] = (o.det_normal((3072, 768), seed=101, scale_log2=-5).astype(np.float32).astype(np.float64), "f32")
    # bf16 weights at the C2 shape (GPT-2 medium FFN, w1 4096x1024)
    out["c2_w1_bf16"] = (o.round_bf16(o.det_normal((4096, 1024), seed=202, scale_log2=-5)), "bf16")
    return out


def fst_cases():
    """Small FFN layers (bf16-representable values) for fwd/bwd goldens."""
    cases = {}
    for act, d, d_ff, n in (("gelu", 32, 64, 48), ("geglu", 32, 64, 48), ("relu", 16, 32, 24)):
        seed = {"gelu": 1, "geglu": 2, "relu": 3}[act]
        r_in = 2 * d_ff if act == "geglu" else d_ff
        cases[act] = dict(
            x=o.round_bf16(o.det_normal((n, d), seed=seed * 10 + 1)),
            w_in=o.round_bf16(o.det_normal((r_in, d), seed=seed * 10 + 2, scale_log2=-2)),
            bias_in=o.round_bf16(o.det_normal((r_in,), seed=seed * 10 + 3, scale_log2=-3)),
            w2=o.round_bf16(o.det_normal((d, d_ff), seed=seed * 10 + 4, scale_log2=-3)),
            dy=o.round_bf16(o.det_normal((n, d), seed=seed * 10 + 5, scale_log2=-4)),
        )
    return cases


def main():
    s24 = import_reference()
    from sparse24.gated_ffn import Activation, FFNLayer, FFNMasks, fst_backward, fst_forward, geglu_forward
    from sparse24.optim import masked_decay_gradient

    table = s24.enumerate_patterns()
    text = table.to_text()
    md5 = hashlib.md5(text.encode()).hexdigest()
    assert md5 == "313a02e787e3fa096f2727e789833468", md5
    with open(os.path.join(HERE, "patterns.txt"), "w") as f:
        f.write(text)

    arrays = {}
    for name, (w, tag) in mask_corpora().items():
        res = ref_search(s24, w)
        arrays[f"{name}.idx"] = res["idx"]
        # large corpora are regenerated bit-exactly by tests from
        # mask_corpora() (integer-only generator); small ones store
        # inputs plus both compressed orientations
        if w.size <= 512 * 512 and name != "gauss_f64":
            arrays[f"{name}.w_bf16"] = o.bf16_bits(w)
            arrays[f"{name}.fwd_meta"] = res["fwd_meta"]
            arrays[f"{name}.bwd_meta"] = res["bwd_meta"]
            arrays[f"{name}.fwd_values"] = o.bf16_bits(res["fwd_values"])
            arrays[f"{name}.bwd_values"] = o.bf16_bits(res["bwd_values"])
        print(f"{name}: {w.shape} tag={tag}")
    np.savez_compressed(os.path.join(HERE, "mask_golden.npz"), **arrays)

    fst = {}
    for act, c in fst_cases().items():
        if act == "geglu":
            r = c["w2"].shape[1]
            layer = FFNLayer.gated(u=c["w_in"][:r], v=c["w_in"][r:], b=c["bias_in"][:r],
                                   c=c["bias_in"][r:], w2=c["w2"])
        else:
            layer = FFNLayer.plain(w1=c["w_in"], b=c["bias_in"], w2=c["w2"],
                                   activation=Activation(act))
        masks = FFNMasks(w_in=s24.transposable_search_conv(layer.w_in()),
                         w_out=s24.transposable_search_conv(layer.w2))
        f = fst_forward(layer, c["x"], masks)
        g = fst_backward(f, c["dy"], rng_seed=0, mvue=False)
        dw_in = np.concatenate([g.d_u, g.d_v]) if act == "geglu" else g.d_w1
        dbias = np.concatenate([g.d_b, g.d_c]) if act == "geglu" else g.d_b
        decayed = masked_decay_gradient(dw_in, layer.w_in(), masks.w_in.bits, 6e-5)
        # dense path (masks=None): the dense fine-tune switch target
        fd = fst_forward(layer, c["x"], None)
        gd = fst_backward(fd, c["dy"], rng_seed=0, mvue=False)
        for k, v in c.items():
            fst[f"{act}.{k}"] = v
        fst.update({
            f"{act}.mask_in": masks.w_in.bits, f"{act}.mask_out": masks.w_out.bits,
            f"{act}.z": np.asarray(f.z), f"{act}.a": np.asarray(f.a), f"{act}.y": np.asarray(f.y),
            f"{act}.dx": np.asarray(g.d_x), f"{act}.dw_in": dw_in, f"{act}.dbias_in": dbias,
            f"{act}.dw2": np.asarray(g.d_w2), f"{act}.dw_in_decayed": decayed,
            f"{act}.dense_y": np.asarray(fd.y), f"{act}.dense_dx": np.asarray(gd.d_x),
        })
        print(f"fst {act}: y {f.y.shape}")
    # standalone GEGLU gate (gated_ffn.py:208-224) on bf16-valued operands
    c = fst_cases()["geglu"]
    r = c["w2"].shape[1]
    gg = geglu_forward(c["x"], c["w_in"][:r], c["w_in"][r:], c["bias_in"][:r], c["bias_in"][r:])
    fst["geglu_forward.out"] = gg.to_array()
    np.savez_compressed(os.path.join(HERE, "fst_golden.npz"), **fst)

    # MVUE (sparsity.py:285-413) on bf16-valued inputs incl. zeros, single
    # nonzeros and one dominant entry per group; fst_backward(mvue=True), the
    # reference default (gated_ffn.py:308)
    from sparse24.sparsity import mvue_inclusion_probs, mvue_pair_probs, mvue_slots_rowwise

    mv = {}
    for i, (shape, seed) in enumerate(mvue_cases()):
        arr = mvue_input(shape, i)
        vals, pos = mvue_slots_rowwise(arr, seed)
        mv[f"case{i}.x"] = arr
        mv[f"case{i}.seed"] = np.array(seed, dtype=np.uint64)
        mv[f"case{i}.values"] = vals
        mv[f"case{i}.pos"] = pos.astype(np.int32)
        mv[f"case{i}.pi"] = mvue_inclusion_probs(arr.reshape(-1, 4))
        mv[f"case{i}.pairs"] = mvue_pair_probs(mv[f"case{i}.pi"])
    for act, c in fst_cases().items():
        if act == "geglu":
            r = c["w2"].shape[1]
            layer = FFNLayer.gated(u=c["w_in"][:r], v=c["w_in"][r:], b=c["bias_in"][:r],
                                   c=c["bias_in"][r:], w2=c["w2"])
        else:
            layer = FFNLayer.plain(w1=c["w_in"], b=c["bias_in"], w2=c["w2"], activation=Activation(act))
        masks = FFNMasks(w_in=s24.transposable_search_conv(layer.w_in()),
                         w_out=s24.transposable_search_conv(layer.w2))
        f = fst_forward(layer, c["x"], masks)
        for seed in (0, 12345):
            g = fst_backward(f, c["dy"], rng_seed=seed, mvue=True)
            mv[f"fst_{act}_{seed}.dw_in"] = np.concatenate([g.d_u, g.d_v]) if act == "geglu" else g.d_w1
            mv[f"fst_{act}_{seed}.dw2"] = np.asarray(g.d_w2)
    np.savez_compressed(os.path.join(HERE, "mvue_golden.npz"), **mv)
    print("wrote", os.listdir(HERE))


def optim_golden():
    """Adam + masked decay in both decay modes (trainer.py:438-447 with the reference's
    optim.adam_step / masked_decay_gradient / srste_weight_decay) and refresh flip
    statistics (flip_rate, block_flip_stats) -> optim_golden.npz."""
    s24 = import_reference()
    from sparse24.optim import (OptimizerState, adam_step, block_flip_stats, flip_rate, masked_decay_gradient,
                                srste_weight_decay)

    out = {}
    w0 = o.det_normal((64, 96), 700) * 0.05
    m = s24.transposable_search_conv(w0).bits
    grads = [o.det_normal((64, 96), 710 + t) * 2.0 ** -7 for t in range(3)]
    out["w0"], out["mask"] = w0, m
    for t, g in enumerate(grads):
        out[f"g{t}"] = g
    for mode, lam in (("none", 0.0), ("on_gradients", 6e-2), ("on_weights", 6e-2)):
        st = OptimizerState.init(w0.copy(), lr=3e-3)
        for g in grads:
            gg = masked_decay_gradient(g, st.w, m, lam) if mode == "on_gradients" else g
            w_before = st.w.copy()
            adam_step(st, gg)
            if mode == "on_weights":
                st.w[:] = srste_weight_decay(st.w, w_before, m, st.lr, lam)
        out[f"{mode}.w"], out[f"{mode}.u"], out[f"{mode}.v"] = st.w, st.u, st.v
        out[f"{mode}.lam"] = np.array(lam)
    # refresh statistics between two weight snapshots
    wa = o.det_normal((128, 64), 720)
    wb = wa + o.det_normal((128, 64), 721) * 0.3
    ma, mb = s24.transposable_search_conv(wa).bits, s24.transposable_search_conv(wb).bits
    out["flip.wa"], out["flip.wb"] = wa, wb
    out["flip.rate"] = np.array(flip_rate(ma, mb))
    out["flip.block_flips"] = block_flip_stats([wa, wb]).block_flips
    np.savez_compressed(os.path.join(HERE, "optim_golden.npz"), **out)
    print("optim golden:", {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


def comparator_golden():
    """Greedy transposable search and directional prune_2of4 of the reference (kernels
    greedy_masks / prune_2of4_keep) on the small mask corpora -> comparators_golden.npz."""
    s24 = import_reference()
    from sparse24.matrix import Direction
    from sparse24.sparsity import _blocks_16, prune_2of4, transposable_search_greedy

    table = s24.enumerate_patterns()
    out = {}
    for name, (w, tag) in mask_corpora().items():
        if name in ("c1_w1_f32", "c2_w1_bf16"):
            continue  # large corpora: the search goldens cover them
        g = transposable_search_greedy(w).bits
        blocks = _blocks_16(g).reshape(-1, 16)
        r, c = w.shape
        out[f"{name}.greedy_idx"] = np.array([table.index_of(b.reshape(4, 4)) for b in blocks],
                                             dtype=np.uint8).reshape(r // 4, c // 4)
        out[f"{name}.prune_row"] = prune_2of4(w, Direction.ROW_WISE).mask.bits.astype(np.uint8)
        out[f"{name}.prune_col"] = prune_2of4(w, Direction.COL_WISE).mask.bits.astype(np.uint8)
    np.savez_compressed(os.path.join(HERE, "comparators_golden.npz"), **out)
    print("comparator golden:", sorted(out))


TRAIN_CASES = {
    # name -> reference TrainConfig kwargs (tensor-core friendly dims: d, d_ff % 128, batch % 64)
    "geglu_ongrad": dict(d=128, d_ff=256, depth=2, batch=128, steps=36, lr=1e-2, mvue=False,
                         decay=dict(lambda_w=2e-4, mode="on_gradients", refresh_period=8)),
    "geglu_mvue_onweights": dict(d=128, d_ff=256, depth=2, batch=128, steps=36, lr=1e-2, mvue=True,
                                 decay=dict(lambda_w=2e-4, mode="on_weights", refresh_period=8)),
}


SEARCH_GRID = (2e-5, 2e-4, 2e-3, 2e-2)
SEARCH_WARMUP = 20


def train_golden():
    """Loss / flip-rate curves of the reference's run_training (trainer.py:387-480) ->
    train_golden.npz; the GPU trainer runs the same configs on the same data."""
    import_reference()
    from sparse24.optim import DecayConfig, DecayMode
    from sparse24.trainer import TrainConfig, run_training

    out = {}
    for name, kw in TRAIN_CASES.items():
        kw = dict(kw)
        dec = kw.pop("decay")
        cfg = TrainConfig(**kw, decay=DecayConfig(lambda_w=dec["lambda_w"], mode=DecayMode(dec["mode"]),
                                                  refresh_period=dec["refresh_period"]))
        art = run_training(cfg)
        out[f"{name}.losses"] = art.losses
        out[f"{name}.flips"] = art.flips
        out[f"{name}.eval"] = np.array(art.final_eval_loss)
        out[f"{name}.searches"] = np.array(art.mask_search_calls)
        print(name, art.losses[:3], art.losses[-3:], art.final_eval_loss)
    # decay-factor search on short warm-ups (optim.py:220-259 with trainer.make_warmup_runner)
    from sparse24.optim import decay_factor_search
    from sparse24.trainer import make_warmup_runner

    kw = dict(TRAIN_CASES["geglu_ongrad"])
    kw.pop("decay")
    kw["steps"] = 200
    base = TrainConfig(**kw)
    res = decay_factor_search(list(SEARCH_GRID), SEARCH_WARMUP, make_warmup_runner(base, SEARCH_WARMUP))
    out["search.mu"] = np.array([e.mu for e in res.entries])
    out["search.dense_ref"] = np.array(res.dense_reference)
    out["search.chosen"] = np.array(np.nan if res.chosen is None else res.chosen)
    print("search", out["search.mu"], res.chosen)
    np.savez_compressed(os.path.join(HERE, "train_golden.npz"), **out)


PACKED_SHAPES = {"a": (8, 16), "b": (96, 160), "c": (36, 44)}


def packed_golden():
    """The packed route of the reference (spmm.py: compress / decompress / mask_of / spmm /
    spmm_right), mvue_prune in both directions and block_flip_stats' gaps ->
    packed_golden.npz."""
    s24 = import_reference()
    from sparse24.matrix import Direction
    from sparse24.optim import block_flip_stats
    from sparse24.sparsity import mvue_prune, prune_2of4
    from sparse24.spmm import compress, decompress, mask_of, spmm, spmm_right

    out = {}
    for name, shape in PACKED_SHAPES.items():
        w = o.round_bf16(o.det_normal(shape, 800 + len(name) + shape[0]))
        out[f"{name}.w"] = w
        for dname, d in (("row", Direction.ROW_WISE), ("col", Direction.COL_WISE)):
            est = prune_2of4(w, d)
            c = compress(est)
            out[f"{name}.{dname}.bits"] = est.mask.bits.astype(np.uint8)
            out[f"{name}.{dname}.values"] = c.values
            out[f"{name}.{dname}.meta"] = c.meta
            out[f"{name}.{dname}.dense"] = decompress(c).data
            assert np.array_equal(mask_of(c).bits, est.mask.bits)
    # products through the packed route (A row-wise 96 x 160, B column-wise 160 x 96)
    w = out["b.w"]
    a_c = compress(prune_2of4(w, Direction.ROW_WISE))
    rhs = o.round_bf16(o.det_normal((160, 40), 811))
    out["spmm.rhs"] = rhs
    out["spmm.out"] = spmm(a_c, rhs).data
    lhs = o.round_bf16(o.det_normal((40, 160), 812))
    b_c = compress(prune_2of4(np.ascontiguousarray(w.T), Direction.COL_WISE))  # 160 x 96 column-wise
    out["spmm_right.lhs"] = lhs
    out["spmm_right.out"] = spmm_right(lhs, b_c).data
    # mvue_prune
    for i, (shape, seed) in enumerate(mvue_cases()):
        g = mvue_input(shape, i)
        out[f"mvue{i}.g"] = g
        out[f"mvue{i}.seed"] = np.array(seed, dtype=np.uint64)
        for dname, d in (("row", Direction.ROW_WISE), ("col", Direction.COL_WISE)):
            est = mvue_prune(g, d, seed)
            out[f"mvue{i}.{dname}.values"] = est.values
            out[f"mvue{i}.{dname}.bits"] = est.mask.bits.astype(np.uint8)
    # block_flip_stats over three snapshots, and the tie corpus' gaps
    wa = o.det_normal((64, 96), 830)
    wb = wa + o.det_normal((64, 96), 831) * 0.3
    wc = wb + o.det_normal((64, 96), 832) * 0.3
    tr = block_flip_stats([wa, wb, wc])
    out["flip3.wa"], out["flip3.wb"], out["flip3.wc"] = wa, wb, wc
    out["flip3.block_flips"], out["flip3.block_gaps"] = tr.block_flips, tr.block_gaps
    ties = (o._splitmix64(64 * 64, 833) % np.uint64(3)).astype(np.float64).reshape(64, 64)
    tt = block_flip_stats([ties, ties])
    out["ties.w"], out["ties.block_gaps"] = ties, tt.block_gaps
    np.savez_compressed(os.path.join(HERE, "packed_golden.npz"), **out)
    print("packed golden:", len(out), "arrays")


def mvue_cases():
    return [((16, 64), 0), ((32, 128), 7), ((8, 256), 2 ** 40 + 3), ((128, 64), (12345 << 2) ^ 2)]


def mvue_input(shape, i):
    a = o.det_normal(shape, seed=500 + i)
    u = (o._splitmix64(int(np.prod(shape)), 900 + i) % np.uint64(10)).reshape(shape)
    a = np.where(u < 2, 0.0, a)                       # zeros -> groups with < 2 nonzeros
    a = np.where(u == 9, a * 2.0 ** 12, a)            # dominant entries -> clamped pi
    return o.round_bf16(a)


if __name__ == "__main__":
    if sys.argv[1:] == ["optim"]:
        optim_golden()
    elif sys.argv[1:] == ["comparators"]:
        comparator_golden()
    elif sys.argv[1:] == ["train"]:
        train_golden()
    elif sys.argv[1:] == ["packed"]:
        packed_golden()
    else:
        main()
        optim_golden()
        comparator_golden()
        train_golden()
        packed_golden()
