"""Token-batch data parallelism for the FFN block.

Weights, masks and compressed operands are replicated: every rank runs the
same K1 search on the same weights and gets the same masks bit-for-bit, so
no collective is needed for them.  Each rank runs fwd + bwd on its own token
shard; the only exchange is one SUM all-reduce of the flat gradient bucket
[dW_in | dbias_in | dW2] per step (NCCL over NVLink on the GPU box, gloo in
the CPU tests).  The masked decay (optim.py:105-114) is applied once in total:
each rank fuses lambda / world into its dW epilogue.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, rank: int, world: int) -> slice:
    """Contiguous token shard of rank `rank` (strong-scaling split of n tokens)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


def decay_share(lambda_w: float, world: int) -> float:
    """Per-rank decay so the summed gradient carries lambda_w exactly once."""
    return lambda_w / world


def allreduce_grads(tensors, group=None) -> None:
    """SUM-all-reduce a list of gradient tensors as ONE flat bucket (one
    collective per step), in place."""
    tensors = [t for t in tensors if t is not None]
    if not tensors:
        return
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for t in tensors:
        t.copy_(flat[off:off + t.numel()].view_as(t))
        off += t.numel()


class GradBucket:
    """Preallocated flat fp32 bucket whose views are the gradient outputs of
    the dW GEMMs, so the all-reduce needs no packing copy."""

    def __init__(self, shapes, device):
        sizes = [int(torch.Size(s).numel()) for s in shapes]
        self.flat = torch.empty(sum(sizes), dtype=torch.float32, device=device)
        self.views = []
        off = 0
        for s, n in zip(shapes, sizes):
            self.views.append(self.flat[off:off + n].view(s))
            off += n

    @classmethod
    def for_params(cls, params) -> "GradBucket":
        return cls([p.shape for p in params], params[0].device)

    def owns(self, t: torch.Tensor, i: int) -> bool:
        """True when `t` is view i of this bucket (the backward wrote the gradient in place)."""
        v = self.views[i]
        return t.data_ptr() == v.data_ptr() and t.shape == v.shape and t.dtype == v.dtype

    def allreduce(self, group=None, async_op: bool = False):
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def allreduce_bucket(bucket: GradBucket, group=None) -> None:
    """The one SUM all-reduce of a step when the gradients already live in `bucket`."""
    bucket.allreduce(group)
