"""GPU parity of the fused optimizer step and the mask-flip statistics
against the reference-generated golden vectors (tests/golden/optim_golden.npz)."""
import os

import numpy as np
import pytest
import torch

from oracle import s24_oracle as o
from gpu_util import need_gpu, normwise_rel

pytestmark = pytest.mark.gpu
GD = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "optim_golden.npz")))


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def _run(mode, dtype):
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.optim import DecayConfig, DecayMode, OptimizerState, adam_step

    w0 = torch.from_numpy(GD["w0"]).cuda()
    mask = P.transposable_search_conv(w0.to(torch.float64))
    assert np.array_equal(mask.bits.cpu().numpy(), GD["mask"])  # same mask as the reference
    st = OptimizerState.init(w0, lr=3e-3, dtype=dtype)
    cfg = DecayConfig(lambda_w=float(GD[f"{mode}.lam"]),
                      mode={"none": DecayMode.NONE, "on_gradients": DecayMode.ON_GRADIENTS,
                            "on_weights": DecayMode.ON_WEIGHTS}[mode])
    for t in range(3):
        adam_step(st, torch.from_numpy(GD[f"g{t}"]).cuda().to(dtype), mask, cfg)
    torch.cuda.synchronize()
    return st


@pytest.mark.parametrize("mode", ["none", "on_gradients", "on_weights"])
def test_adam_fused_decay_f64_bit_exact(mode):
    st = _run(mode, torch.float64)
    for k in ("w", "u", "v"):
        got = getattr(st, k).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), GD[f"{mode}.{k}"].view(np.uint64)), k


@pytest.mark.parametrize("mode", ["none", "on_gradients", "on_weights"])
def test_adam_fused_decay_fp32(mode):
    st = _run(mode, torch.float32)
    # fp32 master weights / moments: relative to the step size actually taken
    dw_ref = GD[f"{mode}.w"] - GD["w0"]
    dw = st.w.double().cpu().numpy() - GD["w0"].astype(np.float32).astype(np.float64)
    assert normwise_rel(dw, dw_ref) < 1e-4
    assert normwise_rel(st.v.cpu().numpy(), GD[f"{mode}.v"]) < 1e-5


def test_adam_flat_bias_vector_and_errors():
    from paper_2404_01847_b200.optim import OptimizerState, adam_step
    from paper_2404_01847_b200.matrix import ShapeError

    b = torch.from_numpy(GD["g0"][0, :37].copy()).cuda()  # odd length: vector tail path
    g = torch.from_numpy(GD["g1"][0, :37].copy()).cuda()
    st = OptimizerState.init(b, dtype=torch.float64)
    adam_step(st, g)
    w, u, v = o.adam_step(GD["g0"][0, :37], np.zeros(37), np.zeros(37), 1, GD["g1"][0, :37])
    assert np.array_equal(st.w.cpu().numpy().view(np.uint64), w.view(np.uint64))
    with pytest.raises(ShapeError):
        adam_step(st, g[:5])


def test_flip_rate_and_block_flips_bit_exact():
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.optim import flip_rate, mask_flips

    ma = P.transposable_search_conv(torch.from_numpy(GD["flip.wa"]).cuda())
    mb = P.transposable_search_conv(torch.from_numpy(GD["flip.wb"]).cuda())
    assert flip_rate(ma, mb) == float(GD["flip.rate"])
    blk = torch.zeros(ma.idx.numel(), dtype=torch.int32, device="cuda")
    n = mask_flips(ma, mb, blk)
    mask_flips(ma, mb, blk)  # accumulates
    assert int(n) == int(round(float(GD["flip.rate"]) * GD["flip.wa"].size))
    assert np.array_equal(blk.cpu().numpy(), 2 * GD["flip.block_flips"])


@pytest.mark.parametrize("mode", ["none", "on_gradients", "on_weights"])
@pytest.mark.parametrize("gated", [False, True])
def test_adam_fused_with_next_step_compression_bit_exact(mode, gated):
    """s24_adam_compress (the fp32 optimizer step fused with the next forward's prune/compress)
    equals s24_adam_step followed by K2 on the updated weight, bit for bit: w, u, v and the kept
    values of both orientations (gated: the u/v-interleaved operand of W_in)."""
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200 import engine as E
    from paper_2404_01847_b200.optim import DecayConfig, DecayMode, OptimizerState, adam_step

    rows, cols = (768, 256) if gated else (512, 384)
    ff = rows // 2 if gated else 0
    g0 = torch.Generator(device="cuda").manual_seed(rows + cols + len(mode))
    w = torch.randn(rows, cols, generator=g0, device="cuda") * 0.05
    op_a = E.CompressedOperand.empty(rows, cols, "cuda", perm_ff=ff)
    E.search_compress(w, op_a)
    op_b = E.CompressedOperand.empty(rows, cols, "cuda", perm_ff=ff)
    op_b.idx.copy_(op_a.idx)
    mask = P.TransposableMask(op_a.mask_idx(), (rows, cols))
    cfg = DecayConfig(lambda_w=0.02, mode={"none": DecayMode.NONE, "on_gradients": DecayMode.ON_GRADIENTS,
                                           "on_weights": DecayMode.ON_WEIGHTS}[mode])
    sa = OptimizerState.init(w, lr=3e-3, dtype=torch.float32)
    sb = OptimizerState.init(w, lr=3e-3, dtype=torch.float32)
    for t in range(3):
        g = torch.randn(rows, cols, generator=g0, device="cuda")
        adam_step(sa, g, mask, cfg)
        E.compress_values(sa.w, op_a)
        adam_step(sb, g, None, cfg, compress_into=op_b)
        torch.cuda.synchronize()
        for k in ("w", "u", "v"):
            assert torch.equal(getattr(sa, k), getattr(sb, k)), (t, k)
        assert torch.equal(op_a.fwd_vals.view(torch.int16), op_b.fwd_vals.view(torch.int16)), t
        assert torch.equal(op_a.bwd_vals.view(torch.int16), op_b.bwd_vals.view(torch.int16)), t
