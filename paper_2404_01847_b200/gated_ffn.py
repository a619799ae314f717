"""Gated activations and the fully sparse FFN layer on the B200 -- the
reference API of sparse24.gated_ffn (gated_ffn.py:1-373) over CUDA tensors.

Differences from the reference that are deliberate and visible:
  * tensors are torch CUDA tensors; compute is bf16 with fp32 accumulation
    (the reference is float64); tolerances are stated in tests/;
  * z, a, y, d_x are token-major (row-major N x features) torch tensors; the
    reference's sparse route returns the same values in column-major numpy
    arrays (gated_ffn.py:162);
  * weight gradients are fp32;
  * mvue=True (the reference default, gated_ffn.py:308) runs K8: the MVUE
    draw of the reference (same PCG64 stream, same float64 selection) on the
    GPU's bf16 upstream gradients, then 2:4 tensor-core weight-gradient GEMMs;
  * Activation.SWIGLU is an extension (not in the reference enum).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import torch

from . import _capi as C
from . import engine as E
from .matrix import Layout, ShapeError
from .sparsity import TransposableMask, transposable_search_conv

__all__ = [
    "Activation", "Traversal", "FFNLayer", "FFNMasks", "LayerGrads", "FstActivations",
    "gelu", "gelu_grad", "geglu_forward", "geglu_backward", "fst_forward", "fst_backward",
]


class Activation(Enum):
    RELU = "relu"
    GELU = "gelu"
    GEGLU = "geglu"
    SWIGLU = "swiglu"  # extension


class Traversal(Enum):
    """Accepted for API compatibility: on the GPU the gate always streams the
    contiguous (token) axis; values never depend on traversal (test_gated_ffn.py:96-103)."""

    ROW_ORDER = "row_order"
    COL_ORDER = "col_order"


def gelu(x: torch.Tensor) -> torch.Tensor:
    """Exact GELU (gated_ffn.py:58-62); elementwise helper in torch, not a hot path."""
    return 0.5 * x * (1.0 + torch.erf(x * 0.7071067811865476))


def gelu_grad(x: torch.Tensor) -> torch.Tensor:
    return 0.5 * (1.0 + torch.erf(x * 0.7071067811865476)) + x * 0.3989422804014327 * torch.exp(-0.5 * x * x)


@dataclass
class FFNLayer:
    """One FFN layer (gated_ffn.py:77-128).  The gated first weight is stored
    concatenated as w_in = [u; v] (r_in = 2 d_ff) with bias_in = [b; c], which
    is how the trainer lays it out (trainer.py:166) and what the single
    transposable mask covers."""

    w_in_cat: torch.Tensor  # (r_in, d)
    bias_in_cat: torch.Tensor  # (r_in,)
    w2: torch.Tensor  # (d, d_ff)
    activation: Activation

    def __post_init__(self) -> None:
        d, d_ff = self.w2.shape
        if d % 4 or d_ff % 4:
            raise ShapeError(f"layer widths must be divisible by 4, got d={d}, d_ff={d_ff}")
        r_in = 2 * d_ff if self.is_gated else d_ff
        if tuple(self.w_in_cat.shape) != (r_in, d):
            raise ShapeError(f"w_in shape {tuple(self.w_in_cat.shape)} != {(r_in, d)}")

    @property
    def is_gated(self) -> bool:
        return self.activation in (Activation.GEGLU, Activation.SWIGLU)

    @property
    def d(self) -> int:
        return self.w2.shape[0]

    @property
    def d_ff(self) -> int:
        return self.w2.shape[1]

    def w_in(self) -> torch.Tensor:
        return self.w_in_cat

    def bias_in(self) -> torch.Tensor:
        return self.bias_in_cat

    @property
    def w1(self):
        return None if self.is_gated else self.w_in_cat

    @property
    def u(self):
        return self.w_in_cat[: self.d_ff] if self.is_gated else None

    @property
    def v(self):
        return self.w_in_cat[self.d_ff:] if self.is_gated else None

    @classmethod
    def gated(cls, u, v, b, c, w2, activation: Activation = Activation.GEGLU) -> "FFNLayer":
        return cls(torch.cat([u, v], 0).contiguous(), torch.cat([b, c]).contiguous(), w2, activation)

    @classmethod
    def plain(cls, w1, b, w2, activation: Activation = Activation.GELU) -> "FFNLayer":
        return cls(w1.contiguous(), b.contiguous(), w2, activation)


@dataclass
class FFNMasks:
    """Transposable masks for w_in and w2 (gated_ffn.py:165-188).  `plans()`
    validates once and builds the tensor-core metadata (E tiles) for both
    orientations; per-step values are recompressed from the current weights
    on every forward (the reference re-gathers them the same way,
    gated_ffn.py:159-162)."""

    w_in: TransposableMask
    w_out: TransposableMask
    _ops: dict = field(default_factory=dict, repr=False, compare=False)
    _ops_f32: dict = field(default_factory=dict, repr=False, compare=False)

    def plans_f32(self, layer: FFNLayer) -> dict:
        """The fp32 mode's operands: both weights as SplitOperands (hi / lo values of both
        orientations sharing the E tiles), validated once."""
        if not self._ops_f32:
            self.w_in.validate()
            self.w_out.validate()
            for name, mask, w in (("in", self.w_in, layer.w_in_cat), ("out", self.w_out, layer.w2)):
                op = E.SplitOperand.empty(mask.shape[0], mask.shape[1], w.device)
                op.hi.idx.copy_(mask.idx)
                op.compress(w, with_meta=True)
                self._ops_f32[name] = op
        return self._ops_f32

    def plans(self, layer: FFNLayer | None = None) -> dict:
        if not self._ops:
            self.w_in.validate()
            self.w_out.validate()
            if layer is None:
                return self._ops
            for name, mask, w in (("in", self.w_in, layer.w_in_cat), ("out", self.w_out, layer.w2)):
                op = E.CompressedOperand.empty(mask.shape[0], mask.shape[1], w.device)
                op.idx.copy_(mask.idx)
                E.compress_with_meta(w, op)
                self._ops[name] = op
        return self._ops


@dataclass
class LayerGrads:
    d_x: torch.Tensor
    d_w2: torch.Tensor | None = None
    d_b: torch.Tensor | None = None
    d_w1: torch.Tensor | None = None
    d_u: torch.Tensor | None = None
    d_v: torch.Tensor | None = None
    d_c: torch.Tensor | None = None


@dataclass
class FstActivations:
    """Everything the backward needs from one forward (gated_ffn.py:251-261)."""

    layer: FFNLayer
    x: torch.Tensor
    z: torch.Tensor  # (N, r_in)
    a: torch.Tensor  # (N, d_ff)
    y: torch.Tensor  # (N, d)
    masks: FFNMasks | None
    w_in_cat: torch.Tensor
    state: "E.FwdState | E.FwdStateF32 | None" = None


def _pad_tokens64(t: torch.Tensor) -> torch.Tensor:
    """Zero token rows up to the tensor-core path's 64-token granule (E.pad_tokens)."""
    return E.pad_tokens(t, 64)


def _head(t, n: int):
    """The first n token rows of a (possibly padded) activation, or t itself (None included)."""
    return t if t is None or t.shape[0] == n else t[:n]


def _as_bf16(t: torch.Tensor) -> torch.Tensor:
    C.require_cuda(t)
    return t if t.dtype == torch.bfloat16 else t.to(torch.bfloat16)


def _fp32_mode(x: torch.Tensor, precision: str | None) -> bool:
    if precision is None:  # the reference computes in its input's float type (_core.pyx:21-23)
        return x.dtype in (torch.float32, torch.float64)
    if precision not in ("bf16", "fp32"):
        raise ValueError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
    return precision == "fp32"


def _fst_forward_f32(layer: FFNLayer, x: torch.Tensor, masks: FFNMasks | None) -> FstActivations:
    """fp32 mode: split-bf16 products on the tensor cores, fp32 accumulation and activations
    (include/sparse24_b200.h, s24_fp32.cu); outputs are the feature-major fp32 results viewed as
    (tokens x features), i.e. the reference's column-major layout."""
    C.require_cuda(x)
    if masks is None:
        w_in, w2 = E.DenseSplitOperand.of(layer.w_in_cat), E.DenseSplitOperand.of(layer.w2)
    else:
        ops = masks.plans_f32(layer)
        ops["in"].compress(layer.w_in_cat)
        ops["out"].compress(layer.w2)
        w_in, w2 = ops["in"], ops["out"]
    st = E.ffn_forward_f32(x.float(), w_in, layer.bias_in_cat, w2, layer.activation.value)
    return FstActivations(layer, x, st.zt.t(), st.at.t(), st.yt.t(), masks, layer.w_in_cat, st)


def fst_forward(layer: FFNLayer, x: torch.Tensor, masks: FFNMasks | None,
                traversal: Traversal = Traversal.COL_ORDER, precision: str | None = None) -> FstActivations:
    """Forward (gated_ffn.py:273-301).  masks=None is the dense path (dense
    fine-tuning, gated_ffn.py:286-289): the same tensor-core kernels on the
    dense weights (s24_gemm_act) with the activation kernel K6.

    precision: None follows the input like the reference's fused float type -- bf16 input runs
    the bf16 path, float32 / float64 input the fp32 mode (split-bf16 products with fp32
    accumulation, fp32 activations); 'bf16' / 'fp32' force one."""
    if x.dim() != 2 or x.shape[1] != layer.d:
        raise ShapeError(f"x shape {tuple(x.shape)} does not match layer width {layer.d}")
    if _fp32_mode(x, precision):
        return _fst_forward_f32(layer, x, masks)
    x = _as_bf16(x)
    if x.dim() != 2 or x.shape[1] != layer.d:
        raise ShapeError(f"x shape {tuple(x.shape)} does not match layer width {layer.d}")
    n = x.shape[0]
    xp = _pad_tokens64(x)

    def bundle(st, m):
        return FstActivations(layer, x, _head(st.z, n), _head(st.a, n), _head(st.y, n), m, layer.w_in_cat, st)

    if masks is None:
        w_in, w2 = _dense_ops(layer)
        return bundle(E.ffn_forward(xp, w_in, _as_bf16(layer.bias_in_cat), w2, layer.activation.value), None)
    if masks.w_in.shape != tuple(layer.w_in_cat.shape) or masks.w_out.shape != tuple(layer.w2.shape):
        raise ShapeError("mask shapes do not match layer weights")
    ops = masks.plans(layer)
    E.compress_values(layer.w_in_cat, ops["in"])
    E.compress_values(layer.w2, ops["out"])
    return bundle(E.ffn_forward(xp, ops["in"], _as_bf16(layer.bias_in_cat), ops["out"], layer.activation.value),
                  masks)


def fst_backward(bundle: FstActivations, upstream: torch.Tensor, rng_seed: int = 0, mvue: bool = True,
                 decay_lambda: float = 0.0) -> LayerGrads:
    """Backward (gated_ffn.py:304-364) with the straight-through weight
    gradients reported against the dense weights.  `decay_lambda` (extension)
    fuses masked_decay_gradient (optim.py:105-114) into the dW epilogue."""
    layer = bundle.layer
    if isinstance(bundle.state, E.FwdStateF32):
        # fp32 mode: dense weight gradients (with mvue=True: the MVUE estimator's expectation)
        C.require_cuda(upstream)
        if tuple(upstream.shape) != tuple(bundle.y.shape):
            raise ShapeError(f"upstream shape {tuple(upstream.shape)} != output shape {tuple(bundle.y.shape)}")
        if bundle.masks is None:
            w_in, w2 = E.DenseSplitOperand.of(layer.w_in_cat), E.DenseSplitOperand.of(layer.w2)
            lam = 0.0
        else:
            ops = bundle.masks.plans_f32(layer)
            w_in, w2, lam = ops["in"], ops["out"], decay_lambda
        g = E.ffn_backward_f32(bundle.state, upstream.float(), w_in, w2, layer.activation.value,
                               w_in_dense=layer.w_in_cat.float(), w2_dense=layer.w2.float(), lam=lam)
        return _pack_grads(layer, g.dxt.t(), g.dw_in, g.dbias_in, g.dw2)
    up = _as_bf16(upstream)
    if tuple(up.shape) != tuple(bundle.y.shape):
        raise ShapeError(f"upstream shape {tuple(up.shape)} != output shape {tuple(bundle.y.shape)}")
    n = up.shape[0]
    up = _pad_tokens64(up)  # zero upstream rows for the padded tokens (fst_forward)
    if bundle.masks is None:
        return _dense_backward(bundle, up, n)
    ops = bundle.masks.plans(layer)
    g = E.ffn_backward(bundle.state, up, ops["in"], ops["out"], layer.activation.value,
                       w_in_dense=layer.w_in_cat, w2_dense=layer.w2, lam=decay_lambda, mvue=mvue,
                       rng_seed=rng_seed, n_valid=n)
    return _pack_grads(layer, _head(g.dx, n), g.dw_in, g.dbias_in, g.dw2)


def _pack_grads(layer, dx, dw_in, dbias, dw2) -> LayerGrads:
    grads = LayerGrads(d_x=dx, d_w2=dw2)
    if layer.is_gated:
        r = layer.d_ff
        grads.d_u, grads.d_v = dw_in[:r], dw_in[r:]
        grads.d_b, grads.d_c = dbias[:r], dbias[r:]
    else:
        grads.d_w1, grads.d_b = dw_in, dbias
    return grads


def _dense_ops(layer: FFNLayer):
    return (E.DenseOperand.of(_as_bf16(layer.w_in_cat).contiguous()),
            E.DenseOperand.of(_as_bf16(layer.w2).contiguous()))


def _dense_backward(bundle: FstActivations, up: torch.Tensor, n: int) -> LayerGrads:
    """masks=None backward (gated_ffn.py:304-364 on the dense route): dense tensor-core dA / dX
    GEMMs, K7 for the activation and bias gradients, the dense dW GEMMs (no decay)."""
    layer = bundle.layer
    w_in, w2 = _dense_ops(layer)
    g = E.ffn_backward(bundle.state, up, w_in, w2, layer.activation.value)
    return _pack_grads(layer, _head(g.dx, n), g.dw_in, g.dbias_in, g.dw2)


def geglu_forward(x, u, v, b, c, traversal: Traversal = Traversal.COL_ORDER) -> torch.Tensor:
    """gelu(x u^T + b) * (x v^T + c) (gated_ffn.py:208-224): the dense tensor-core GEMM on the
    concatenated [u; v] (s24_gemm_act, bias fused), then the gate kernel K6.  Returns (N x d_ff)."""
    x = _as_bf16(x).contiguous()
    w_cat = torch.cat([u, v], 0).to(torch.bfloat16).contiguous()
    b_cat = torch.cat([b, c]).to(torch.bfloat16)
    if x.shape[1] != w_cat.shape[1]:
        raise ShapeError(f"x cols {x.shape[1]} != weight cols {w_cat.shape[1]}")
    n, r = x.shape[0], u.shape[0]
    z = torch.empty((n, 2 * r), dtype=torch.bfloat16, device=x.device)  # (N, 2r) token-major
    E._mm(E.DenseOperand.of(w_cat), False, x, n, z, "geglu_fwd", bias=b_cat)
    a = torch.empty((n, r), dtype=torch.bfloat16, device=x.device)
    C.call("s24_act_fwd", z.data_ptr(), 2 * r, r, n, C.ACT_GEGLU, a.data_ptr(), r, C.stream_of(z))
    return a


def geglu_backward(x, u, v, b, c, upstream) -> LayerGrads:
    """Analytic GEGLU gradients (gated_ffn.py:227-244): the gate part by K7, dX by the dense
    tensor-core GEMM on [u; v]^T, dW by the dense dW GEMM."""
    x = _as_bf16(x).contiguous()
    up = _as_bf16(upstream).contiguous()
    w_cat = torch.cat([u, v], 0).to(torch.bfloat16).contiguous()
    b_cat = torch.cat([b, c]).to(torch.bfloat16)
    n, r = x.shape[0], u.shape[0]
    d = x.shape[1]
    if tuple(up.shape) != (n, r):
        raise ShapeError(f"upstream shape {tuple(up.shape)} != output shape {(n, r)}")
    op = E.DenseOperand.of(w_cat)
    z = torch.empty((n, 2 * r), dtype=torch.bfloat16, device=x.device)
    E._mm(op, False, x, n, z, "geglu_fwd", bias=b_cat)
    dz = torch.empty_like(z)
    dbias = torch.empty(2 * r, dtype=torch.float32, device=x.device)
    C.call("s24_act_bwd", z.data_ptr(), 2 * r, up.data_ptr(), r, r, n, C.ACT_GEGLU, dz.data_ptr(), 2 * r,
           dbias.data_ptr(), C.stream_of(z))
    dx = torch.empty((n, d), dtype=torch.bfloat16, device=x.device)
    E._mm(op, True, dz, n, dx, "geglu_bwd")
    dw = torch.empty((2 * r, d), dtype=torch.float32, device=x.device)
    E.gemm_dw(dz, True, x, True, 2 * r, d, n, dw)
    return LayerGrads(d_x=dx, d_u=dw[:r], d_v=dw[r:], d_b=dbias[:r], d_c=dbias[r:])


def search_layer_masks(layer: FFNLayer) -> FFNMasks:
    """Masks for both weights (trainer.py:212-219) via K1."""
    return FFNMasks(w_in=transposable_search_conv(layer.w_in_cat), w_out=transposable_search_conv(layer.w2))


LAYOUT_OF_OUTPUTS = Layout.COL_MAJOR
