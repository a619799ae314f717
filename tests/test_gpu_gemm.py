"""K3/K4 (2:4 sparse tcgen05) and K5 (dense dW + masked decay) GEMMs vs a
plain fp32 torch reference on the same bf16 operands.

Tolerance: outputs are bf16 (sparse) or fp32 (dW) from fp32 accumulation;
normwise relative error <= 1e-2 for bf16 outputs and <= 2e-3 for fp32 dW,
plus an elementwise bound of 3 bf16 ulps of the row scale."""
import os
import numpy as np
import pytest
import torch

from gpu_util import need_gpu, normwise_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    need_gpu()


def _operand(m, k, seed):
    from paper_2404_01847_b200.engine import CompressedOperand, search_compress

    g = torch.Generator(device="cuda").manual_seed(seed)
    w = (torch.randn(m, k, generator=g, device="cuda") / k ** 0.5).bfloat16()
    op = CompressedOperand.empty(m, k, "cuda")
    search_compress(w, op)
    from paper_2404_01847_b200 import TransposableMask
    bits = TransposableMask(op.idx, (m, k)).bits
    return w, op, bits


@pytest.mark.parametrize("m,k,n", [(128, 128, 128), (256, 512, 384), (384, 256, 96), (1024, 1024, 512)])
@pytest.mark.parametrize("b_mn", [False, True])
def test_sparse_gemm_fwd_orientation(m, k, n, b_mn):
    from paper_2404_01847_b200.engine import spmm

    w, op, bits = _operand(m, k, 1 + m + k)
    x = torch.randn(n, k, device="cuda").bfloat16()
    b = x.t().contiguous() if b_mn else x
    bias = torch.randn(m, device="cuda").bfloat16()
    out = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    spmm(op.fwd_vals, op.fwd_e, m, k, b, b_mn, n, out, bias)
    ref = (w.float() * bits.float()) @ x.float().t() + bias.float()[:, None]
    assert normwise_rel(out.float().cpu(), ref.cpu()) < 1e-2


@pytest.mark.parametrize("m,k,n", [(128, 256, 128), (512, 384, 256)])
def test_sparse_gemm_bwd_orientation_and_gelu_epilogue(m, k, n):
    """W^T operand from the same transposable mask; fused GELU aux output."""
    from paper_2404_01847_b200.engine import spmm

    w, op, bits = _operand(m, k, 7)
    dy = torch.randn(n, m, device="cuda").bfloat16()
    out = torch.empty((k, n), dtype=torch.bfloat16, device="cuda")
    spmm(op.bwd_vals, op.bwd_e, k, m, dy, False, n, out)
    ref = (w.float() * bits.float()).t() @ dy.float().t()
    assert normwise_rel(out.float().cpu(), ref.cpu()) < 1e-2
    x = torch.randn(n, k, device="cuda").bfloat16()
    z = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    a = torch.empty_like(z)
    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, z, None, gelu_aux=a)
    zr = (w.float() * bits.float()) @ x.float().t()
    ar = torch.nn.functional.gelu(zr)
    assert normwise_rel(z.float().cpu(), zr.cpu()) < 1e-2
    assert normwise_rel(a.float().cpu(), ar.cpu()) < 1e-2


@pytest.mark.parametrize("m,k,n,slabs", [(256, 256, 384, "0"), (512, 4096, 448, "1")])
def test_gelu_epilogue_wide_range_and_saturation(m, k, n, slabs):
    """The packed f32x2 GELU / GELU' epilogue (clamp on z^2) over pre-activations spanning
    |z| up to ~40: elementwise against the float64 exact-erf GELU, and exact saturation
    (GELU' = 1 / 0, GELU = z / 0) beyond |z| = 9.5; single- and two-slab tiles."""
    import subprocess
    import sys

    code = (
        "import torch, sys\n"
        "sys.path[:0] = [%r, %r]\n"
        "import paper_2404_01847_b200._capi as C\n"
        "from paper_2404_01847_b200.engine import spmm, aux_empty, aux_to_feature_major, CompressedOperand, search_compress\n"
        "from paper_2404_01847_b200 import TransposableMask\n"
        "m, k, n = %d, %d, %d\n"
        "g = torch.Generator(device='cuda').manual_seed(5)\n"
        "w = (torch.randn(m, k, generator=g, device='cuda') / k ** 0.5).bfloat16()\n"
        "op = CompressedOperand.empty(m, k, 'cuda'); search_compress(w, op)\n"
        "bits = TransposableMask(op.idx, (m, k)).bits\n"
        "x = (torch.randn(n, k, generator=g, device='cuda') * 14).bfloat16()\n"
        "out = torch.empty((n, m), dtype=torch.bfloat16, device='cuda')\n"
        "ga = aux_empty(m, n, 'cuda')\n"
        "spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, None, epi=C.EPI_GELU_GRAD, aux=ga, out_t=True)\n"
        "gd = aux_to_feature_major(ga, m, n).t().double().cpu()\n"
        "z = (x.double() @ (w.double() * bits.double()).t()).cpu()\n"
        "cdf = 0.5 * (1 + torch.erf(z / 2 ** 0.5))\n"
        "ref = z * cdf\n"
        "dref = cdf + z * torch.exp(-0.5 * z * z) / (2 * torch.pi) ** 0.5\n"
        "o = out.double().cpu()\n"
        "assert z.abs().max() > 20, float(z.abs().max())\n"
        # bf16 rounding of the stored value + tanh.approx (<= 2^-11 relative in t, i.e.
        # <= 2.5e-4 |z| in GELU and ~1e-3 |z| in GELU' where t is not saturated)
        "tol = 2 ** -8 * ref.abs() + 3e-4 * z.abs() + 1e-4\n"
        "assert torch.all((o - ref).abs() <= tol), float(((o - ref).abs() / tol).max())\n"
        "dtol = 2 ** -8 * dref.abs() + 1.2e-3 * z.abs().clamp(max=10) + 5e-4\n"
        "assert torch.all((gd - dref).abs() <= dtol), float(((gd - dref).abs() / dtol).max())\n"
        "hi, lo = z > 9.5, z < -9.5\n"
        "assert hi.sum() > 100 and lo.sum() > 100\n"
        "assert torch.all(gd[hi] == 1.0) and torch.all(gd[lo] == 0.0)\n"
        "assert torch.all(o[lo] == 0.0)\n"
        "assert ((o[hi] - z[hi]).abs() / z[hi].abs()).max() < 2 ** -7\n"
        "print('ok')\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)), m, k, n)
    env = dict(os.environ, S24_SLABS_EPI=slabs)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (256, 512, 320), (384, 256, 1024)])
def test_dense_dw_gemm(m, n, k, a_mn, b_mn):
    from paper_2404_01847_b200.engine import gemm_dw

    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    gemm_dw(a.t().contiguous() if a_mn else a, a_mn, b.t().contiguous() if b_mn else b, b_mn, m, n, k, out)
    ref = a.float() @ b.float().t()
    assert normwise_rel(out.cpu(), ref.cpu()) < 2e-3


def test_dense_dw_gemm_masked_decay_epilogue():
    from paper_2404_01847_b200.engine import gemm_dw
    from paper_2404_01847_b200 import transposable_search_conv

    m, n, k = 256, 512, 256
    w = torch.randn(m, n, device="cuda").bfloat16()
    mask = transposable_search_conv(w)
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(k, n, device="cuda").bfloat16()  # MN-major B
    lam = 0.25
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    gemm_dw(a, False, b, True, m, n, k, out, w, mask.idx, lam)
    ref = a.float() @ b.float() + lam * (1 - mask.bits.float()) * w.float()
    assert normwise_rel(out.cpu(), ref.cpu()) < 2e-3
    # kept entries carry no decay
    plain = torch.empty_like(out)
    gemm_dw(a, False, b, True, m, n, k, plain)
    kept = mask.bits.bool()
    assert torch.allclose(out[kept], plain[kept], rtol=0, atol=0)


def test_shape_errors():
    from paper_2404_01847_b200 import ShapeError
    from paper_2404_01847_b200.engine import CompressedOperand

    with pytest.raises(ShapeError):
        CompressedOperand.empty(100, 128, "cuda")


@pytest.mark.parametrize("m,k,n", [(256, 256, 128), (512, 384, 448), (128, 256, 96)])
@pytest.mark.parametrize("epi", ["store", "gelu_grad", "dgelu"])
def test_sparse_gemm_token_major_output_and_epilogues(m, k, n, epi):
    """out_t: D^T stored token-major (n x m); fused GELU/GELU' and dGELU+bias-grad epilogues."""
    import paper_2404_01847_b200._capi as C
    from paper_2404_01847_b200.engine import spmm

    w, op, bits = _operand(m, k, 11 + m + n)
    x = torch.randn(n, k, device="cuda").bfloat16()
    ref = x.float() @ (w.float() * bits.float()).t()  # (n, m)
    out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
    if epi == "store":
        bias = torch.randn(m, device="cuda").bfloat16()
        spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, bias, out_t=True)
        assert normwise_rel(out.float().cpu(), (ref + bias.float()).cpu()) < 1e-2
    elif epi == "gelu_grad":
        from paper_2404_01847_b200.engine import aux_empty, aux_to_feature_major

        g = aux_empty(m, n, "cuda")  # GELU'(z), blocked layout
        spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, None, epi=C.EPI_GELU_GRAD, aux=g, out_t=True)
        g = aux_to_feature_major(g, m, n).t()
        zr = ref.double()
        cdf = 0.5 * (1 + torch.erf(zr / 2 ** 0.5))
        assert normwise_rel(out.float().cpu(), (zr * cdf).cpu()) < 1e-2
        gd = cdf + zr * torch.exp(-0.5 * zr * zr) / (2 * torch.pi) ** 0.5
        assert normwise_rel(g.float().cpu(), gd.cpu()) < 1e-2
    else:
        gin = torch.rand(n, m, device="cuda").bfloat16()
        db = torch.zeros(m, dtype=torch.float32, device="cuda")
        from paper_2404_01847_b200.engine import aux_from_feature_major

        gfm = aux_from_feature_major(gin.t().contiguous())  # blocked GELU'(z) input
        spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, None, epi=C.EPI_DGELU, aux=gfm, dbias=db, out_t=True)
        dz = ref * gin.float()
        assert normwise_rel(out.float().cpu(), dz.cpu()) < 1e-2
        assert normwise_rel(db.cpu(), dz.sum(0).cpu()) < 1e-3


@pytest.mark.parametrize("gate_ff", [0, 512])
def test_dense_dw_gemm_c2_shape(gate_ff):
    """C2-shaped dW (64 whole tiles on 74 CTA pairs) with the masked decay, plain and gated
    (u/v-interleaved rows restored to [u; v] order)."""
    from paper_2404_01847_b200.engine import gemm_dw
    from paper_2404_01847_b200 import transposable_search_conv

    m, n, k = (1024, 1024, 16384) if gate_ff else (1024, 4096, 16384)
    w = torch.randn(m, n, device="cuda").bfloat16()
    mask = transposable_search_conv(w)
    a = torch.randn(k, m, device="cuda").bfloat16()  # token-major upstream gradient (MN-major A)
    b = torch.randn(k, n, device="cuda").bfloat16()
    lam = 0.5
    out = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    if gate_ff:
        # gated first weight: dW rows come out of the u/v interleave back in [u; v] order
        from paper_2404_01847_b200 import engine as E

        p = torch.arange(m, device="cuda")
        orig = torch.where(p % 32 < 16, 16 * (p // 32) + p % 32, gate_ff + 16 * (p // 32) + p % 32 - 16)
        a_perm = torch.empty_like(a)
        a_perm[:, :] = a[:, orig]
        op = E.CompressedOperand.empty(m, n, "cuda", perm_ff=gate_ff)
        E.search_compress(w, op)
        gemm_dw(a_perm, True, b, True, m, n, k, out, w, op.idx, lam, gate_ff=gate_ff)
    else:
        gemm_dw(a, True, b, True, m, n, k, out, w, mask.idx, lam)
    ref = a.float().t() @ b.float() + lam * (1 - mask.bits.float()) * w.float()
    assert torch.isfinite(out).all()
    assert normwise_rel(out.cpu(), ref.cpu()) < 2e-3


@pytest.mark.parametrize("m,k,n", [(512, 8192, 480), (1024, 8448, 224)])
def test_sparse_gemm_two_slab_tiles(m, k, n):
    """K >= 8192 plain token-major stores run on 512 x 224 two-slab pair tiles (one TMEM
    accumulator holding both A slabs against one B tile); partial last N tile included."""
    from paper_2404_01847_b200.engine import spmm

    w, op, bits = _operand(m, k, 77 + m)
    x = torch.randn(n, k, device="cuda").bfloat16()
    bias = torch.randn(m, device="cuda").bfloat16()
    out = torch.full((n, m), float("nan"), dtype=torch.bfloat16, device="cuda")
    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, bias, out_t=True)
    ref = x.float() @ (w.float() * bits.float()).t() + bias.float()
    assert torch.isfinite(out.float()).all()
    assert normwise_rel(out.float().cpu(), ref.cpu()) < 1e-2


def test_sparse_gemm_two_slab_forced_small_k():
    """S24_SLABS=1 forces the two-slab tiles on short K (subprocess: the knob is read once)."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from test_gpu_gemm import _operand\n"
        "from paper_2404_01847_b200.engine import spmm\n"
        "for m, k, n in [(512, 128, 32), (512, 1024, 448), (1536, 2048, 672), (768, 512, 224), (1280, 256, 96)]:\n"
        "    w, op, bits = _operand(m, k, 5 + k)\n"
        "    x = torch.randn(n, k, device='cuda').bfloat16()\n"
        "    out = torch.full((n, m), float('nan'), dtype=torch.bfloat16, device='cuda')\n"
        "    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, out_t=True)\n"
        "    ref = x.float() @ (w.float() * bits.float()).t()\n"
        "    e = float((out.float() - ref).norm() / ref.norm())\n"
        "    assert e < 1e-2, (m, k, n, e)\n"
        "print('ok')\n" % (os.path.abspath(os.path.join(os.path.dirname(__file__), "..")), os.path.dirname(__file__)))
    env = dict(os.environ, S24_SLABS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_dense_dw_two_slab_tiles_forced():
    """S24_DW_SLABS=1: 512 x 256 two-slab dense dW tiles (MN-major operands), with the masked
    decay and the gated row remap (subprocess: the knob is read once)."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2404_01847_b200.engine import gemm_dw, CompressedOperand, search_compress\n"
        "from paper_2404_01847_b200 import transposable_search_conv\n"
        "for m, n, k, gff in [(512, 256, 1024, 0), (1024, 768, 4096, 0), (1024, 512, 2048, 512)]:\n"
        "    w = torch.randn(m, n, device='cuda').bfloat16()\n"
        "    mask = transposable_search_conv(w)\n"
        "    a = torch.randn(k, m, device='cuda').bfloat16(); b = torch.randn(k, n, device='cuda').bfloat16()\n"
        "    out = torch.full((m, n), float('nan'), device='cuda')\n"
        "    if gff:\n"
        "        p = torch.arange(m, device='cuda')\n"
        "        orig = torch.where(p %% 32 < 16, 16 * (p // 32) + p %% 32, gff + 16 * (p // 32) + p %% 32 - 16)\n"
        "        op = CompressedOperand.empty(m, n, 'cuda', perm_ff=gff); search_compress(w, op)\n"
        "        gemm_dw(a[:, orig].contiguous(), True, b, True, m, n, k, out, w, op.idx, 0.5, gate_ff=gff)\n"
        "    else:\n"
        "        gemm_dw(a, True, b, True, m, n, k, out, w, mask.idx, 0.5)\n"
        "    ref = a.float().t() @ b.float() + 0.5 * (1 - mask.bits.float()) * w.float()\n"
        "    e = float((out - ref).norm() / ref.norm())\n"
        "    assert torch.isfinite(out).all() and e < 2e-3, (m, n, k, gff, e)\n"
        "print('ok')\n" % os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    env = dict(os.environ, S24_DW_SLABS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_fused_epilogues_two_slab_tiles_forced():
    """S24_SLABS_EPI=1: GELU/GELU' and dGELU + bias-gradient epilogues on two-slab tiles, including
    a ragged last tile whose second slab lies beyond m (m = 768)."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from test_gpu_gemm import _operand\n"
        "from paper_2404_01847_b200.engine import spmm, aux_empty, aux_to_feature_major\n"
        "import paper_2404_01847_b200._capi as C\n"
        "for m, k, n in [(512, 256, 224), (768, 512, 448), (1280, 1024, 96)]:\n"
        "    w, op, bits = _operand(m, k, 3 + m + k)\n"
        "    x = torch.randn(n, k, device='cuda').bfloat16()\n"
        "    ref = x.float() @ (w.float() * bits.float()).t()\n"
        "    out = torch.full((n, m), float('nan'), dtype=torch.bfloat16, device='cuda')\n"
        "    g = aux_empty(m, n, 'cuda')\n"
        "    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, None, epi=C.EPI_GELU_GRAD, aux=g, out_t=True)\n"
        "    zr = ref.double(); cdf = 0.5 * (1 + torch.erf(zr / 2 ** 0.5))\n"
        "    e = float((out.double() - zr * cdf).norm() / (zr * cdf).norm()); assert e < 1e-2, ('gelu', m, k, n, e)\n"
        "    db = torch.zeros(m, device='cuda')\n"
        "    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, out, None, epi=C.EPI_DGELU, aux=g, dbias=db, out_t=True)\n"
        "    gd = aux_to_feature_major(g, m, n).t().float()\n"
        "    e = float((out.float() - ref * gd).norm() / (ref * gd).norm()); assert e < 1e-2, ('dgelu', m, k, n, e)\n"
        "    e = float((db - (ref * gd).sum(0)).norm() / (ref * gd).sum(0).norm()); assert e < 1e-2, ('dbias', e)\n"
        "print('ok')\n" % (os.path.abspath(os.path.join(os.path.dirname(__file__), "..")), os.path.dirname(__file__)))
    env = dict(os.environ, S24_SLABS_EPI="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_reserved_sms_leave_results_unchanged():
    """The per-call reserved_sms argument shrinks the persistent grids (DP overlap); results are
    unchanged."""
    from paper_2404_01847_b200.engine import reserved_sms, spmm

    m, k, n = 1024, 1024, 2048
    w, op, bits = _operand(m, k, 21)
    x = torch.randn(n, k, device="cuda").bfloat16()
    full = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
    spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, full, out_t=True)
    part = torch.empty_like(full)
    with reserved_sms(100):
        spmm(op.fwd_vals, op.fwd_e, m, k, x, False, n, part, out_t=True)
    assert torch.equal(full, part)


@pytest.mark.parametrize("gate_ff", [0, 1280])
def test_dense_dw_gemm_c5_shape_lockstep_splitk(gate_ff):
    """C5-shaped dW (100 tiles on 74 CTA pairs): the lockstep split-K schedule (two K halves
    add-reduced into the zeroed output, the decay added once) against fp32, and bit-identical
    across repeated launches (two addends onto zero: order-independent)."""
    from paper_2404_01847_b200 import engine as E
    from paper_2404_01847_b200.engine import gemm_dw
    from paper_2404_01847_b200 import transposable_search_conv

    m, n, k = (2560, 1280, 16384) if gate_ff else (1280, 5120, 16384)
    w = torch.randn(m, n, device="cuda").bfloat16()
    mask = transposable_search_conv(w)
    a = torch.randn(k, m, device="cuda").bfloat16()
    b = torch.randn(k, n, device="cuda").bfloat16()
    lam = 0.5
    outs = []
    for _ in range(2):
        out = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
        if gate_ff:
            p = torch.arange(m, device="cuda")
            orig = torch.where(p % 32 < 16, 16 * (p // 32) + p % 32, gate_ff + 16 * (p // 32) + p % 32 - 16)
            a_perm = a[:, orig].contiguous()
            op = E.CompressedOperand.empty(m, n, "cuda", perm_ff=gate_ff)
            E.search_compress(w, op)
            gemm_dw(a_perm, True, b, True, m, n, k, out, w, op.idx, lam, gate_ff=gate_ff)
        else:
            gemm_dw(a, True, b, True, m, n, k, out, w, mask.idx, lam)
        outs.append(out)
    ref = a.float().t() @ b.float() + lam * (1 - mask.bits.float()) * w.float()
    assert torch.isfinite(outs[0]).all()
    assert normwise_rel(outs[0].cpu(), ref.cpu()) < 2e-3
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("splits", ["2", "3", "8"])
def test_dw_gemms_splitk_forced_small_shapes(splits):
    """S24_SPLITK=N forces the lockstep split-K schedule on every dW GEMM (dense and the MVUE
    sparse-A one), including uneven K ranges and the decay; N >= 3 reduces the partial tiles in
    split order, so repeated launches are bit-identical."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2404_01847_b200 import engine as E, transposable_search_conv, _capi as C\n"
        "for m, n, k in [(128, 128, 512), (256, 512, 640), (384, 256, 1216), (512, 768, 4096)]:\n"
        "    w = torch.randn(m, n, device='cuda').bfloat16(); mk = transposable_search_conv(w)\n"
        "    a = torch.randn(k, m, device='cuda').bfloat16(); b = torch.randn(k, n, device='cuda').bfloat16()\n"
        "    out = torch.full((m, n), float('nan'), device='cuda')\n"
        "    E.gemm_dw(a, True, b, True, m, n, k, out, w, mk.idx, 0.5)\n"
        "    ref = a.float().t() @ b.float() + 0.5 * (1 - mk.bits.float()) * w.float()\n"
        "    e = float((out - ref).norm() / ref.norm())\n"
        "    assert e < 2e-3, (m, n, k, e)\n"
        "    for _ in range(3):\n"
        "        o2 = torch.full((m, n), float('nan'), device='cuda')\n"
        "        E.gemm_dw(a, True, b, True, m, n, k, o2, w, mk.idx, 0.5)\n"
        "        assert torch.equal(o2, out), (m, n, k)\n"
        "for f, n, d in [(256, 1024, 128), (512, 2048, 256)]:\n"
        "    g = torch.randn(n, f, device='cuda').bfloat16(); bd = torch.randn(n, d, device='cuda').bfloat16()\n"
        "    vals, e_, _ = E.mvue_compress(g, 7, exact=False)\n"
        "    out = torch.full((f, d), float('nan'), device='cuda')\n"
        "    E.spmm_dw(vals, e_, f, n, bd, True, d, out)\n"
        "    meta = torch.empty((f, n // 4), dtype=torch.uint8, device='cuda')\n"
        "    C.call('s24_e_to_flat', e_.data_ptr(), f, n, meta.data_ptr(), C.stream_of(meta))\n"
        "    sp = torch.empty((f, n), dtype=torch.bfloat16, device='cuda'); bad = torch.zeros(1, dtype=torch.int32, device='cuda')\n"
        "    C.call('s24_unpack24', vals.data_ptr(), 0, meta.data_ptr(), f, n, 0, sp.data_ptr(), 0, bad.data_ptr(), C.stream_of(meta))\n"
        "    dense = sp.float() @ bd.float()\n"
        "    e = float((out - dense).norm() / dense.norm())\n"
        "    assert e < 2e-3, (f, n, d, e)\n"
        "print('ok')\n" % os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    env = dict(os.environ, S24_SPLITK=splits)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_ordered_splitk_under_sm_contention_is_deterministic_or_reported():
    """Hardening of the persistent dW GEMMs: the ordered split-K reduce (S24_SPLITK=4, partial
    tiles add-reduced in split order through the caller's workspace counters) is launched while a
    side-stream kernel holds SMs, so its CTAs are not co-resident.  The bounded waits either keep
    the order (result bit-identical to a solo launch) or give up and say so in the workspace's
    timeout counter (engine.gemm_timeouts) -- never a hang, never a silent change.  The workspace
    is left zeroed apart from that counter."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2404_01847_b200 import engine as E, transposable_search_conv, _capi as C\n"
        "m, n, k = 1024, 2048, 8192\n"
        "w = torch.randn(m, n, device='cuda').bfloat16(); mk = transposable_search_conv(w)\n"
        "a = torch.randn(k, m, device='cuda').bfloat16(); b = torch.randn(k, n, device='cuda').bfloat16()\n"
        "solo = torch.empty((m, n), device='cuda')\n"
        "E.gemm_dw(a, True, b, True, m, n, k, solo, w, mk.idx, 0.5)\n"
        "torch.cuda.synchronize()\n"
        "side = torch.cuda.Stream(); big = torch.randn(8192, 8192, device='cuda').bfloat16()\n"
        "same = 0; runs = 6\n"
        "for i in range(runs):\n"
        "    out = torch.empty((m, n), device='cuda')\n"
        "    with torch.cuda.stream(side):\n"
        "        for _ in range(3): big @ big\n"
        "    E.gemm_dw(a, True, b, True, m, n, k, out, w, mk.idx, 0.5)\n"
        "    torch.cuda.synchronize()\n"
        "    same += int(torch.equal(out, solo))\n"
        "    ref = a.float().t() @ b.float() + 0.5 * (1 - mk.bits.float()) * w.float()\n"
        "    assert float((out - ref).norm() / ref.norm()) < 2e-3\n"
        "t = E.gemm_timeouts()\n"
        "ws = E.gemm_workspace(solo).clone(); ws[C.GEMM_WS_TIMEOUTS_WORD] = 0\n"
        "assert int(ws.abs().sum()) == 0, 'workspace not left zeroed'\n"
        "assert same == runs or t > 0, (same, runs, t)\n"
        "print('ok', same, runs, t)\n" % (os.path.abspath(os.path.join(os.path.dirname(__file__), "..")),))
    env = dict(os.environ, S24_SPLITK="4")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_sparse_dw_two_slab_tiles_forced():
    """S24_SDW_SLABS=1: the 2:4 weight-gradient GEMM (MVUE operand, K = tokens) on 512 x 224
    two-slab tiles with a K-major B (the repo's transpose of the token-major operand) equals the
    256 x 256 single-slab GEMM on the MN-major operand, with the masked decay and the gated row
    remap, ragged last N tile included (subprocess: the knob is read once)."""
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2404_01847_b200 import engine as E\n"
        "for m, n, k, ff in [(1024, 384, 4096, 0), (1536, 640, 2048, 0), (1024, 896, 1024, 512)]:\n"
        "    g = (torch.randn(k, m, device='cuda') * 0.1).bfloat16()\n"
        "    b = torch.randn(k, n, device='cuda').bfloat16()\n"
        "    w = (torch.randn(m, n, device='cuda') * 0.05).bfloat16()\n"
        "    op = E.CompressedOperand.empty(m, n, 'cuda')\n"
        "    E.search_compress(w, op)\n"
        "    vals, e, _ = E.mvue_compress(g, 5, gate_ff=ff)\n"
        "    ref = torch.empty(m, n, device='cuda')\n"
        "    out = torch.full((m, n), float('nan'), device='cuda')\n"
        "    E.spmm_dw(vals, e, m, k, b, True, n, ref, w, op.idx, 0.01, ff)\n"
        "    E.spmm_dw(vals, e, m, k, E.transpose_bf16(b), False, n, out, w, op.idx, 0.01, ff)\n"
        "    err = float((out - ref).norm() / ref.norm())\n"
        "    assert err < 1e-5, (m, n, k, ff, err)\n"
        "x = torch.randn(328, 200, device='cuda').bfloat16()\n"
        "assert torch.equal(E.transpose_bf16(x), x.t().contiguous())\n"
        "print('ok')\n" % os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    env = dict(os.environ, S24_SDW_SLABS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
