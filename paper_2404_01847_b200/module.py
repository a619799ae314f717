"""nn.Module / autograd wrapper of the 2:4 FFN hot path, with the reference's
training-schedule semantics for one FFN block:

  * mask refresh every `refresh_period` OPTIMIZER steps while sparse
    (trainer.py:422-432; DecayConfig.refresh_period = 40, optim.py:55).  An
    optimizer step is detected as a change of the parameters' in-place version
    counters (every torch optimizer updates parameters in place; call
    `mark_weights_updated()` after writing `.data` directly).  The first forward
    after a step recompresses the current weights (K2), or, once the period is
    reached, searches new transposable masks and compresses both orientations
    (K1).  Further forwards of the same step (gradient accumulation, recompute)
    reuse the operands;
  * masked decay on the gradient (DecayMode.ON_GRADIENTS, trainer.py:439-441)
    fused into the dW epilogue (K5);
  * dense fine-tune switch: `sparse = False` runs the same tensor-core kernels
    on the dense weights (fst_forward with masks=None, gated_ffn.py:286-289,
    trainer.py:111-114): dense GEMMs with the fused activation / bias-gradient
    epilogues and the dense dW GEMM, no decay (trainer.py:435-441);
  * data parallelism: `allreduce_grads()` sums [dW_in, dbias, dW2] in one
    NCCL all-reduce of a preallocated bucket the backward writes into; the decay
    is pre-scaled by 1/world so it is applied once.

Parameters are fp32 master weights; the sparse kernels read them directly and
round the kept values to bf16 while compressing.  A backward whose forward ran
on a different mask than the current one (a refresh in between) raises.
"""

from __future__ import annotations

import torch

from . import dp
from . import engine as E


class _SparseFFNFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_in, bias_in, w2, mod, dense_ops):
        xb = x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)
        op_in, op_out = dense_ops if dense_ops is not None else (mod.op_in, mod.op_out)
        n = xb.shape[0]  # any token count: zero-padded to the 64-token granule, outputs sliced
        st = E.ffn_forward(E.pad_tokens(xb, 64), op_in, bias_in.to(torch.bfloat16), op_out, mod.act, fused=True)
        ctx.n = n
        ctx.mod = mod
        ctx.st = st
        ctx.ops = (op_in, op_out)
        ctx.mask_version = mod.mask_version
        ctx.save_for_backward(w_in, w2)
        return st.y if st.y.shape[0] == n else st.y[:n]

    @staticmethod
    def backward(ctx, dy):
        w_in, w2 = ctx.saved_tensors
        mod = ctx.mod
        op_in, op_out = ctx.ops
        dense = isinstance(op_in, E.DenseOperand)
        if not dense and mod.mask_version != ctx.mask_version:
            raise RuntimeError("SparseFFN: the masks were refreshed between this forward and its backward; "
                               "the weight gradient would use a mask that did not produce the activations")
        params = (mod.w_in, mod.bias_in, mod.w2)
        # first gradient of the step: the dW GEMMs / bias epilogue write straight into the
        # preallocated all-reduce bucket, whose views become the parameters' .grad; with
        # gradient accumulation (.grad already set) autograd adds the fresh gradients in place
        direct = all(p.grad is None for p in params)
        b = mod.grad_bucket() if direct else None
        n = ctx.n
        g = E.ffn_backward(ctx.st, E.pad_tokens(dy.to(torch.bfloat16), 64), op_in, op_out, mod.act, w_in_dense=w_in,
                           w2_dense=w2, lam=0.0 if dense else mod.decay_lambda, mvue=mod.mvue and not dense,
                           rng_seed=mod.mvue_seed, mvue_exact=mod.mvue_exact,
                           dw_in_out=b.views[0] if direct else None, dbias_out=b.views[1] if direct else None,
                           dw2_out=b.views[2] if direct else None, n_valid=n)
        ctx.st = None
        dx = g.dx if g.dx.shape[0] == n else g.dx[:n]
        if direct:
            for p, v in zip(params, b.views):
                p.grad = v
            return dx, None, None, None, None, None
        return dx, g.dw_in, g.dbias_in, g.dw2, None, None


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
        self.mask_version = 0  # bumped by every refresh (K1)
        self._seen_version = None  # parameter versions the operands were built from
        self._dirty_steps = 0  # declared optimizer steps not yet seen by a forward
        self._fresh = False  # the last declared step left the operands current (fused compression)
        self._dense_cache = None  # (versions, DenseOperand pair) of the dense phase
        self._bucket = None
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

    def _versions(self):
        return (self.w_in._version, self.w2._version)

    def mark_weights_updated(self, compressed: bool = False) -> None:
        """Declare an optimizer step that bypassed the in-place version counters (e.g. writes
        through `.data`): the next forward advances the refresh schedule and recompresses --
        unless `compressed`, i.e. the step ran the fused optimizer + compression
        (optim.adam_step(compress_into=op_in / op_out)), which already left the current kept
        values in both operands (no K2 launch)."""
        self._dirty_steps += 1
        self._fresh = compressed
        self._dense_cache = None

    def refresh_masks(self) -> None:
        """K1: new transposable masks + both compressed orientations."""
        E.search_compress_pair(self.w_in.detach(), self.op_in, self.w2.detach(), self.op_out)
        self.steps_since_refresh = 0
        self._dirty_steps, self._fresh = 0, False
        self.mask_searches += 2
        self.mask_version += 1
        self._seen_version = self._versions()

    def _prepare_sparse(self) -> None:
        v = self._versions()
        if self.steps_since_refresh is None:
            self.refresh_masks()
            return
        # optimizer steps since the operands were built: declared ones, or one detected through
        # the parameters' version counters (an in-place torch optimizer step)
        steps = self._dirty_steps or (1 if v != self._seen_version else 0)
        if steps == 0:
            return  # same optimizer step (gradient accumulation, recompute): operands are current
        fresh, self._dirty_steps, self._fresh = self._fresh, 0, False
        self.steps_since_refresh += steps
        if self.steps_since_refresh >= self.refresh_period:
            self.refresh_masks()
        else:
            if not fresh:
                E.compress_values_pair(self.w_in.detach(), self.op_in, self.w2.detach(), self.op_out)
            self._seen_version = v

    def _dense_ops(self):
        v = self._versions()
        if self._dense_cache is None or self._dense_cache[0] != v:
            w_in = self.w_in.detach().to(torch.bfloat16).contiguous()
            w2 = self.w2.detach().to(torch.bfloat16).contiguous()
            ff = self.w2.shape[1] if self.act in E.GATED else 0
            self._dense_cache = (v, (E.DenseOperand.of(w_in, ff), E.DenseOperand.of(w2)))
        return self._dense_cache[1]

    def next_forward_refreshes(self) -> bool:
        """Whether the next sparse forward searches new masks (after one more optimizer step)."""
        return self.steps_since_refresh is None or self.steps_since_refresh + self._dirty_steps + 1 \
            >= self.refresh_period

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.sparse:
            return _SparseFFNFn.apply(x, self.w_in, self.bias_in, self.w2, self, self._dense_ops())
        self._prepare_sparse()
        return _SparseFFNFn.apply(x, self.w_in, self.bias_in, self.w2, self, None)

    def grad_bucket(self) -> "dp.GradBucket":
        """The preallocated fp32 [dW_in | dbias | dW2] bucket the backward writes into (one
        all-reduce per step, no packing copies)."""
        if self._bucket is None:
            self._bucket = dp.GradBucket.for_params([self.w_in, self.bias_in, self.w2])
        return self._bucket

    def allreduce_grads(self, group=None) -> None:
        """One NCCL all-reduce of the gradient bucket (SUM: the per-rank loss is a per-rank
        sum/mean and the decay is pre-scaled).  The parameters' .grad are views of the bucket
        when the last backward wrote them there; otherwise they are packed first."""
        params = (self.w_in, self.bias_in, self.w2)
        b = self.grad_bucket()
        if all(p.grad is not None and b.owns(p.grad, i) for i, p in enumerate(params)):
            dp.allreduce_bucket(b, group)
        else:
            dp.allreduce_grads([p.grad for p in params], group)

    @property
    def masks_idx(self):
        return self.op_in.idx, self.op_out.idx
