"""nn.Module / autograd wrapper of the 2:4 FFN hot path, with the reference's
training-schedule semantics for one FFN block:

  * mask refresh every `refresh_period` optimizer steps while sparse
    (trainer.py:422-432; DecayConfig.refresh_period = 40, optim.py:55): K1
    searches the new transposable masks and compresses both orientations;
    other steps run K2 (per-step prune/compress of the current weights);
  * masked decay on the gradient (DecayMode.ON_GRADIENTS, trainer.py:439-441)
    fused into the dW epilogue (K5);
  * dense fine-tune switch: `sparse = False` runs plain dense bf16 GEMMs
    (fst_forward with masks=None, gated_ffn.py:286-289);
  * data parallelism: `allreduce_grads()` sums [dW_in, dbias, dW2] in one
    NCCL all-reduce; the decay is pre-scaled by 1/world so it is applied once.

Parameters are fp32 master weights; the kernels read them directly and round
the kept values to bf16 while compressing.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from . import dp
from . import engine as E


class _SparseFFNFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_in, bias_in, w2, mod):
        xb = x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)
        st = E.ffn_forward(xb, mod.op_in, bias_in.to(torch.bfloat16), mod.op_out, mod.act, fused=True)
        ctx.mod = mod
        ctx.st = st
        ctx.save_for_backward(w_in, w2)
        return st.y

    @staticmethod
    def backward(ctx, dy):
        w_in, w2 = ctx.saved_tensors
        mod = ctx.mod
        g = E.ffn_backward(ctx.st, dy.to(torch.bfloat16), mod.op_in, mod.op_out, mod.act, w_in_dense=w_in,
                           w2_dense=w2, lam=mod.decay_lambda, mvue=mod.mvue, rng_seed=mod.mvue_seed,
                           mvue_exact=mod.mvue_exact)
        ctx.st = None
        return g.dx, g.dw_in, g.dbias_in, g.dw2, None


class SparseFFN(torch.nn.Module):
    def __init__(self, d: int, d_ff: int, act: str = "gelu", refresh_period: int = 40, decay_lambda: float = 0.0,
                 device=None):
        super().__init__()
        r_in = 2 * d_ff if act in E.GATED else d_ff
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.w_in = torch.nn.Parameter(torch.randn(r_in, d, device=dev) / d ** 0.5)  # trainer.py:180-191
        self.bias_in = torch.nn.Parameter(torch.zeros(r_in, device=dev))
        self.w2 = torch.nn.Parameter(torch.randn(d, d_ff, device=dev) / d_ff ** 0.5)
        self.act = act
        self.refresh_period = refresh_period
        self.decay_lambda = decay_lambda
        self.sparse = True
        self.op_in = E.CompressedOperand.empty(r_in, d, dev, perm_ff=d_ff if act in E.GATED else 0)
        self.op_out = E.CompressedOperand.empty(d, d_ff, dev)
        self.steps_since_refresh = None  # None -> search on first use
        self.mask_searches = 0
        # MVUE-sparsified weight gradients (fst_backward(mvue=True), gated_ffn.py:304-373): the
        # caller sets the per-step layer seed (trainer.py:245-247) before backward
        self.mvue = False
        self.mvue_seed = 0
        self.mvue_exact = True

    @classmethod
    def from_weights(cls, w_in, bias_in, w2, act, refresh_period=40, decay_lambda=0.0) -> "SparseFFN":
        d_ff = w2.shape[1]
        m = cls(w2.shape[0], d_ff, act, refresh_period, decay_lambda, device=w_in.device)
        with torch.no_grad():
            m.w_in.copy_(w_in.float())
            m.bias_in.copy_(bias_in.float())
            m.w2.copy_(w2.float())
        return m

    def refresh_masks(self) -> None:
        """K1: new transposable masks + both compressed orientations."""
        E.search_compress_pair(self.w_in.detach(), self.op_in, self.w2.detach(), self.op_out)
        self.steps_since_refresh = 0
        self.mask_searches += 2

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.sparse:
            return self._dense(x)
        if self.steps_since_refresh is None or self.steps_since_refresh >= self.refresh_period:
            self.refresh_masks()
        else:
            E.compress_values_pair(self.w_in.detach(), self.op_in, self.w2.detach(), self.op_out)
        if self.training:
            self.steps_since_refresh += 1
        return _SparseFFNFn.apply(x, self.w_in, self.bias_in, self.w2, self)

    def _dense(self, x):
        xb = x.to(torch.bfloat16)
        z = F.linear(xb, self.w_in.to(torch.bfloat16), self.bias_in.to(torch.bfloat16))
        r = self.w2.shape[1]
        if self.act == "gelu":
            a = F.gelu(z)
        elif self.act == "relu":
            a = F.relu(z)
        elif self.act == "swiglu":
            a = F.silu(z[:, :r]) * z[:, r:]
        else:
            a = F.gelu(z[:, :r]) * z[:, r:]
        return F.linear(a, self.w2.to(torch.bfloat16))

    def allreduce_grads(self, group=None) -> None:
        """One NCCL all-reduce of the concatenated gradients (SUM: the
        per-rank loss is a per-rank sum/mean and the decay is pre-scaled)."""
        dp.allreduce_grads([p.grad for p in (self.w_in, self.bias_in, self.w2)], group)

    @property
    def masks_idx(self):
        return self.op_in.idx, self.op_out.idx
