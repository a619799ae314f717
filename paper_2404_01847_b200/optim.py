"""Masked decay and the schedule pieces on the path (optim.py:51-114 of the reference)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch

from . import _capi as C
from .matrix import ShapeError
from .sparsity import TransposableMask


class DecayMode(Enum):
    NONE = "none"
    ON_WEIGHTS = "on_weights"
    ON_GRADIENTS = "on_gradients"


@dataclass
class DecayConfig:
    """optim.py:51-61: lambda_w, mode, refresh_period (mask search every l steps)."""

    lambda_w: float = 0.0
    mode: DecayMode = DecayMode.NONE
    refresh_period: int = 40

    def __post_init__(self) -> None:
        if self.lambda_w < 0:
            raise ValueError("lambda_w must be nonnegative")
        if self.refresh_period < 1:
            raise ValueError("refresh_period must be >= 1")


def masked_decay_gradient(g: torch.Tensor, w: torch.Tensor, m, lambda_w: float) -> torch.Tensor:
    """g + lambda_w * (1 - m) * w (optim.py:105-114), computed by the
    s24_masked_decay kernel on an fp32 copy of g.  `m` is a TransposableMask
    (the hot-path form; the fused dW epilogue does the same in the GEMM) or a
    0/1 tensor of w's shape."""
    C.require_cuda(g, w)
    if isinstance(m, TransposableMask):
        if m.shape != tuple(g.shape) or tuple(w.shape) != tuple(g.shape):
            raise ShapeError("gradient, weights and mask must have equal shapes")
        out = g.to(torch.float32).contiguous().clone()
        wc = w.contiguous()
        C.call("s24_masked_decay", out.data_ptr(), wc.data_ptr(), C.dtype_code(wc), m.idx.data_ptr(),
               g.shape[0], g.shape[1], float(lambda_w), C.stream_of(out))
        return out
    m = torch.as_tensor(m, device=g.device)
    if not (g.shape == w.shape == m.shape):
        raise ShapeError("gradient, weights and mask must have equal shapes")
    return g.to(torch.float32) + lambda_w * ((1 - m.to(torch.float32)) * w.to(torch.float32))
