"""Token-batch data parallelism on the GPU.

Two ranks share cuda:0 over a gloo process group (the sandbox has one GPU; NCCL refuses two
ranks on one device, the all-reduce itself is the same one-bucket SUM).  Each rank runs its
half of the tokens through

* the public module path: `SparseFFN` forward/backward writing the preallocated
  [dW_in | dbias | dW2] bucket, then `SparseFFN.allreduce_grads()` (dp.allreduce_bucket);
* the bench's training step (`bench.SparseStep`): the async all-reduce issued from the
  backward's `grads_ready` hook while the dX GEMM still runs (reserved SMs).

Oracle: linearity -- the summed bucket equals the full-batch float64 gradient
(oracle.fst_backward, exact=False) with the masked decay applied ONCE (each rank carries
lambda / world), normwise <= 1e-2 (bf16 operands, fp32 accumulation); and the K1 masks
(pattern indices) are bit-identical on both ranks (their equality with the oracle's search
is pinned in test_gpu_mask.py / test_gpu_parity_configs.py).
"""
import multiprocessing as mp
import os
import socket
import sys

import numpy as np
import pytest

from oracle import s24_oracle as o
from gpu_util import need_gpu, normwise_rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def _worker(rank, world, port, path, act, d, d_ff, n, lam, q):
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
        import torch
        import torch.distributed as dist

        from gpu_util import to_dev_bf16
        from paper_2404_01847_b200 import dp
        from paper_2404_01847_b200.module import SparseFFN

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        c = _case(act, d, d_ff, n, seed=11)
        sl = dp.shard_rows(n, rank, world)
        w_in, b, w2 = to_dev_bf16(c["w_in"]), to_dev_bf16(c["bias_in"]), to_dev_bf16(c["w2"])
        x, dy = to_dev_bf16(c["x"][sl]), to_dev_bf16(c["dy"][sl])
        if path == "module":
            mod = SparseFFN.from_weights(w_in, b, w2, act, decay_lambda=dp.decay_share(lam, world))
            mod(x).backward(dy)
            mod.allreduce_grads()
            grads = [mod.w_in.grad, mod.bias_in.grad, mod.w2.grad]
            idx = list(mod.masks_idx)
        else:
            import bench

            bench.LAMBDA = lam
            step = bench.SparseStep(w_in, b, w2, act, world, pg=None)
            step(x, dy)
            grads = [step.dw_in, step.dbias, step.dw2]
            idx = [step.op_in.idx, step.op_out.idx]
        torch.cuda.synchronize()
        # masks identical on every rank: gather rank 1's pattern indices to rank 0
        same = True
        for t in idx:
            g = [torch.empty_like(t.cpu()) for _ in range(world)]
            dist.all_gather(g, t.cpu().contiguous())
            same = same and all(torch.equal(g[0], gi) for gi in g[1:])
        if rank == 0:
            q.put(("ok", [g.double().cpu().numpy() for g in grads], same))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001 -- surfaced through the queue
        import traceback

        q.put(("err", f"rank {rank}: {e!r}\n{traceback.format_exc()}", False))
        raise


@pytest.mark.parametrize("path", ["module", "bench_step"])
@pytest.mark.parametrize("act,d,d_ff,n", [("gelu", 256, 512, 512), ("geglu", 256, 384, 512)])
def test_two_ranks_one_bucket_allreduce(path, act, d, d_ff, n):
    world = 2
    c = _case(act, d, d_ff, n, seed=11)
    lo = o.Layer(c["w_in"], c["bias_in"], c["w2"], act)
    mi, mo = o.transposable_search_conv(c["w_in"]), o.transposable_search_conv(c["w2"])
    fr = o.fst_forward(lo, c["x"], mi, mo, exact=False)
    br = o.fst_backward(lo, fr, c["dy"], mi, mo, exact=False)
    # lambda sized so the decay term is 10% of dW_in: a decay applied twice (each rank the
    # full lambda) or never is then ~10x outside the tolerance
    lam = 0.1 * float(np.linalg.norm(br["dw_in"]) / np.linalg.norm(c["w_in"] * (mi == 0)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, path, act, d, d_ff, n, lam, q)) for r in range(world)]
    for p in ps:
        p.start()
    status, payload, same = q.get(timeout=300)
    for p in ps:
        p.join(120)
    assert status == "ok", payload
    assert all(p.exitcode == 0 for p in ps)
    assert same, "ranks disagree on the K1 masks"

    ref = [o.masked_decay_gradient(br["dw_in"], c["w_in"], mi, lam), br["dbias_in"],
           o.masked_decay_gradient(br["dw2"], c["w2"], mo, lam)]
    dw_in, dbias, dw2 = payload
    for name, ours, r in (("dw_in", dw_in, ref[0]), ("dbias", dbias, ref[1]), ("dw2", dw2, ref[2])):
        assert normwise_rel(ours, r) < 1e-2, (name, normwise_rel(ours, r))
    twice = o.masked_decay_gradient(ref[0], c["w_in"], mi, lam)
    assert normwise_rel(dw_in, twice) > 5e-2  # the test would see a decay applied twice
