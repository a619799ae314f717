"""bench.py --config c5: the GPT-2 large 2:4 pre-training step (BASELINE.json configs[4]).

The measured unit is one training step of the residual FFN stack of the reference's
_FFNStack (trainer.py:159-262): h_{l+1} = h_l + FFN_l(h_l) over 36 blocks of
d=1280, d_ff=5120, GELU, 16384 tokens per rank, forward then backward through every
block (dh_l = dh_{l+1} + dX_l, accumulated by the dX GEMM's add-reduce store).  Each block runs the same kernels as the single-block
bench (K2 prune/compress of both weights, or K1 search every 40th step; fused
GEMM+GELU, GEMM; dGELU-fused dA, dW2 and dW_in with the masked decay, dX), and each
block's gradient bucket [dW_in | dbias | dW2] is all-reduced asynchronously as soon as
its dW GEMMs are enqueued, so the collective of block l overlaps the backward of
blocks l-1 .. 0.  The last few SMs are left to NCCL while any
all-reduce can be in flight (the GEMMs' reserved_sms argument, engine.RESERVED_SMS).  Same JSON contract as bench.py."""
from __future__ import annotations

import os

import bench as B


class StackStep:
    def __init__(self, layers, act, world, pg=None):
        import torch
        from paper_2404_01847_b200 import _capi
        from paper_2404_01847_b200 import engine as E

        self.E, self.torch, self.C = E, torch, _capi
        self.layers, self.act, self.world, self.pg = layers, act, world, pg
        self.ops, self.buckets = [], []
        for w_in, bias, w2 in layers:
            dev = w_in.device
            op_in = E.CompressedOperand.empty(w_in.shape[0], w_in.shape[1], dev,
                                              perm_ff=w2.shape[1] if act in E.GATED else 0)
            op_out = E.CompressedOperand.empty(w2.shape[0], w2.shape[1], dev)
            n_in, n_b, n_2 = w_in.numel(), w_in.shape[0], w2.numel()
            bucket = torch.empty(n_in + n_b + n_2, dtype=torch.float32, device=dev)
            views = (bucket[:n_in].view(w_in.shape), bucket[n_in:n_in + n_b], bucket[n_in + n_b:].view(w2.shape))
            self.ops.append((op_in, op_out))
            self.buckets.append((bucket, views))
        self.t = 0
        self.dh = None
        self.launches_per_step = len(layers) * (1 + 2 + 4)

    def __call__(self, x, dy):
        E, torch = self.E, self.torch
        refresh = self.t % B.REFRESH == 0
        if self.dh is None or self.dh.shape != dy.shape:
            self.dh = torch.empty_like(dy)
        states = []
        h = x
        for (w_in, bias, w2), (op_in, op_out) in zip(self.layers, self.ops):
            if refresh:
                E.search_compress_pair(w_in, op_in, w2, op_out)
            else:
                E.compress_values_pair(w_in, op_in, w2, op_out)
            st = E.ffn_forward(h, op_in, bias, op_out, self.act, fused=True)
            states.append(st)
            h = h + st.y
        work = []
        # the residual gradient dh_l = dh_{l+1} + dX_l accumulates in one buffer: each block's
        # dX GEMM add-reduces into it (S24_EPI_STORE_ADD) after the block's dA / dW2 GEMMs read it
        dh = self.dh
        dh.copy_(dy)
        for l in reversed(range(len(self.layers))):
            w_in, bias, w2 = self.layers[l]
            op_in, op_out = self.ops[l]
            bucket, (dwi, db, dw2) = self.buckets[l]

            def grads_ready(bucket=bucket):
                if self.world > 1:
                    work.append(torch.distributed.all_reduce(bucket, group=self.pg, async_op=True))
                    E.RESERVED_SMS = B.DP_RESERVED_SMS

            g = E.ffn_backward(states[l], dh, op_in, op_out, self.act, w_in_dense=w_in, w2_dense=w2,
                               lam=B.LAMBDA / self.world, dw_in_out=dwi, dw2_out=dw2, dbias_out=db,
                               grads_ready=grads_ready, dx_accumulate=dh)
            states[l] = None
        E.RESERVED_SMS = 0
        for w in work:
            w.wait()
        self.t += 1
        return h, dh


def make_stack(cfg, device, seed):
    import torch

    layers = []
    for l in range(cfg["layers"]):
        w_in, bias, w2, x, dy = B.make_problem(dict(cfg, tokens=64), device, seed * 1000 + l)
        layers.append((w_in, bias, w2))
    g = torch.Generator(device="cpu").manual_seed(seed)
    n, d = cfg["tokens"], cfg["d"]
    x = torch.randn(n, d, generator=g).to(torch.bfloat16).to(device)
    dy = (torch.randn(n, d, generator=g) / (n * d) ** 0.5).to(torch.bfloat16).to(device)
    return layers, x, dy


def dense_stack_factory(layers, act):
    import torch
    import torch.nn.functional as F

    params = [(w.clone().requires_grad_(True), b.clone().requires_grad_(True), w2.clone().requires_grad_(True))
              for w, b, w2 in layers]

    def step(x, dy):
        h = x.detach().requires_grad_(True)
        out = h
        for w, b, w2 in params:
            out = out + F.linear(F.gelu(F.linear(out, w, b)), w2)
        out.backward(dy)
        for p in params:
            for q in p:
                q.grad = None

    return step


class DenseFusedStack:
    """The dense residual stack on the SAME tensor-core kernels and fused epilogues as the 2:4
    stack (bench.DenseFusedStep per block: bias + GELU / GELU' in GEMM1, dGELU + bias gradient in
    GEMM3, the dense dW GEMMs, dX add-reduced into the residual gradient): the fair dense
    comparator of the stack, beside eager autograd."""

    def __init__(self, layers, act):
        import torch
        from paper_2404_01847_b200 import engine as E

        self.E, self.torch, self.act = E, torch, act
        self.blocks = []
        for w_in, bias, w2 in layers:
            self.blocks.append((E.DenseOperand.of(w_in, 0), bias, E.DenseOperand.of(w2),
                                torch.empty(w_in.shape, dtype=torch.float32, device=w_in.device),
                                torch.empty(w_in.shape[0], dtype=torch.float32, device=w_in.device),
                                torch.empty(w2.shape, dtype=torch.float32, device=w2.device)))
        self.dh = None

    def __call__(self, x, dy):
        E = self.E
        if self.dh is None or self.dh.shape != dy.shape:
            self.dh = self.torch.empty_like(dy)
        states, h = [], x
        for op_in, bias, op_out, _, _, _ in self.blocks:
            st = E.ffn_forward(h, op_in, bias, op_out, self.act, fused=True)
            states.append(st)
            h = h + st.y
        dh = self.dh
        dh.copy_(dy)
        for l in reversed(range(len(self.blocks))):
            op_in, _, op_out, dwi, db, dw2 = self.blocks[l]
            E.ffn_backward(states[l], dh, op_in, op_out, self.act, dw_in_out=dwi, dw2_out=dw2, dbias_out=db,
                           dx_accumulate=dh)
            states[l] = None
        return h, dh


def run_stack(a, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    shared = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    backend = "gloo" if shared else "nccl"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    from paper_2404_01847_b200 import _capi as C
    from paper_2404_01847_b200 import engine as E

    C.load()
    C.call("s24_device_check")
    if cfg["act"] != "gelu":
        raise SystemExit("the stack bench is GELU-only (GPT-2 large)")
    n_tok, n_layers = cfg["tokens"], cfg["layers"]
    # the same weights on every rank (replicated model), a different token shard per rank
    layers, x, dy = make_stack(cfg, dev, seed=1234)
    g = torch.Generator(device="cpu").manual_seed(99 + rank)
    x = torch.randn(x.shape, generator=g).to(torch.bfloat16).to(dev)
    step = StackStep(layers, cfg["act"], world, pg)
    steps = max(4, a.steps // 20)  # a stack step is ~36 single-block steps

    ms, clocks = B.time_loop(lambda: step(x, dy), steps, max(3, a.warmup // 4), dist if world > 1 else None,
                             local, True)
    t0 = max(3, a.warmup // 4)
    # refresh steps: one K1 launch (both weights of a block) in place of the block's K2 launch
    launches_timed = steps * step.launches_per_step
    ms_step = ms / steps
    value = n_tok * world / (ms_step / 1000.0)

    dense = dense_fused = None
    if not a.no_dense:
        dstep = dense_stack_factory(layers, cfg["act"])
        dsteps = max(3, steps // 2)
        dms, _ = B.time_loop(lambda: dstep(x, dy), dsteps, 3, dist if world > 1 else None)
        dense = n_tok * world / (dms / dsteps / 1000.0)
        del dstep
        fstep = DenseFusedStack(layers, cfg["act"])
        fms, _ = B.time_loop(lambda: fstep(x, dy), dsteps, 3, dist if world > 1 else None)
        dense_fused = n_tok * world / (fms / dsteps / 1000.0)
        del fstep

    # per-kernel attribution over one refresh period's worth of steps is too long for a
    # 36-block stack: 4 steps (one of them a refresh step only if t hits a multiple of 40)
    timer = B.EventTimer()
    E.TIMER = timer
    kt_steps = 4
    for _ in range(kt_steps):
        step(x, dy)
    totals = timer.totals()
    E.TIMER = E._NoTimer()
    per_kernel = {k: {"ms_per_launch": v[0] / v[1], "launches": v[1], "ms_per_step": v[0] / kt_steps}
                  for k, v in sorted(totals.items())}
    peaks, peaks_src = B.load_peaks()
    w_in0, _, w20 = layers[0]
    d, d_ff, r_in = cfg["d"], cfg["d_ff"], w_in0.shape[0]
    flops = {
        "k3_spmm_fwd_in": 2.0 * r_in * n_tok * d, "k3_spmm_fwd_out": 2.0 * d * n_tok * d_ff,
        "k4_spmm_bwd_out": 2.0 * d_ff * n_tok * d, "k4_spmm_bwd_in": 2.0 * d * n_tok * r_in,
        "k5_gemm_dw2": 2.0 * d * d_ff * n_tok, "k5_gemm_dw_in": 2.0 * r_in * d * n_tok,
    }
    sustained = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    for k, f in flops.items():
        if k in per_kernel:
            sp = k.startswith(("k3", "k4"))
            per_kernel[k]["tflops_dense_equiv"] = f / (per_kernel[k]["ms_per_launch"] * 1e-3) / 1e12
            per_kernel[k]["frac_of_peak"] = per_kernel[k]["tflops_dense_equiv"] / (sustained * (2.0 if sp else 1.0))
    dom = max((k for k in per_kernel if k in flops), key=lambda k: per_kernel[k]["ms_per_step"])
    sparse = dom.startswith(("k3", "k4"))
    achieved = per_kernel[dom]["tflops_dense_equiv"]
    peak = sustained * (2.0 if sparse else 1.0)
    roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": B.ncu_traffic("c5", dom),
            "note": ("dense-equivalent 2MNK / t vs 2x measured sustained dense bf16 peak (2:4 pipe)" if sparse
                     else "2MNK / t vs measured sustained dense bf16 peak") + f" ({peaks_src})"}

    e2e = run_stack_e2e(a, cfg, layers, dev, world, dist if world > 1 else None)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            from oracle.ref_step import time_reference

            toks = 32
            per, info = time_reference(d, d_ff, cfg["act"], toks, steps=3, warmup=1, refresh=B.REFRESH, budget_s=20)
            cpu = {"value": toks / per / n_layers, "unit": "tokens/s", "cores": info["cores"], "kind": info["kind"],
                   "sample": f"{toks} tokens x {info['steps']} steps of ONE d={d} d_ff={d_ff} block (fwd+bwd "
                             f"mvue=False, masked decay, mask search /{B.REFRESH}), reference Cython kernels on 1 "
                             f"core; tokens/s divided by the {n_layers} blocks of the stack"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port", "sample": f"failed: {exc!r}"}

    if rank == 0:
        import json

        line = {
            "metric": B.METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": steps,
            "warmup": t0, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference init N(0,1)/sqrt(fan_in) weights, N(0,1) tokens)",
            "config": B.config_dict(dict(cfg, tokens=n_tok, layers=n_layers), world),
            "dp_backend": backend + (" (ranks share GPUs: functional test only)" if shared else ""),
            "allreduce": "one fp32 bucket [dW_in|dbias|dW2] per block, async, overlapped with the backward of the "
                         "blocks below",
            "working_set": "~15 GB per step > 126 MB L2 (no flush)",
            "roofline": roof, "kernels": per_kernel, "e2e": e2e, "gpu_launches": launches_timed,
            "clocks": clocks, "cpu_baseline": cpu,
            # speed-ups last: the driver keeps the tail of the line
            "dense_tokens_per_s": dense, "dense_fused_tokens_per_s": dense_fused,
            "speedup_vs_dense": (value / dense) if dense else None,
            "speedup_vs_dense_fused": (value / dense_fused) if dense_fused else None,
            "speedup_vs_best_dense": (value / max(dense, dense_fused)) if dense and dense_fused else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_stack_e2e(a, cfg, layers, dev, world, dist):
    """The stack through the public API: one SparseFFN module per block (autograd over the
    C ABI), tokens copied host->device every step from pinned memory, loss read back."""
    import torch
    from paper_2404_01847_b200.module import SparseFFN

    mods = [SparseFFN.from_weights(w, b, w2, cfg["act"], refresh_period=B.REFRESH, decay_lambda=B.LAMBDA / world)
            for w, b, w2 in layers]
    n, d = cfg["tokens"], cfg["d"]
    host_x = torch.randn(n, d).to(torch.bfloat16).pin_memory()
    host_loss = torch.empty(1, dtype=torch.float32).pin_memory()
    dev_x = torch.empty(n, d, dtype=torch.bfloat16, device=dev)

    def one():
        dev_x.copy_(host_x, non_blocking=True)
        h = dev_x
        for m in mods:
            h = h + m(h)
        with torch.no_grad():
            loss = torch.linalg.vector_norm(h, dtype=torch.float32).square() * (0.5 / n)
            dy = h * (1.0 / n)
        h.backward(dy)
        if world > 1:
            for m in mods:
                m.allreduce_grads()
        host_loss.copy_(loss.detach().reshape(1), non_blocking=True)
        for m in mods:
            m.zero_grad(set_to_none=True)

    steps = max(3, a.steps // 40)
    ms, _ = B.time_loop(one, steps, 3, dist)
    per = ms / steps
    return {"value": n * world / (per / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": n * d * 2,
            "d2h_bytes_per_step": 4, "ms_per_step": per,
            "api": f"{len(mods)} paper_2404_01847_b200.module.SparseFFN blocks (autograd over the C ABI), residual, "
                   "loss 0.5|h|^2/N",
            "h2d": "pinned host tokens, one copy per step on the compute stream"}
