"""Diagnose the e2e loop: CPU time per step vs GPU time per step, and raw H2D copy rates."""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
import bench
from paper_2404_01847_b200.module import SparseFFN

cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda")
w_in, bias, w2, x, dy = bench.make_problem(cfg, dev, 1)
mod = SparseFFN.from_weights(w_in, bias, w2, cfg["act"], refresh_period=40, decay_lambda=6e-5)
n, d = cfg["tokens"], cfg["d"]
xd = x.clone()
def step_dev():
    y = mod(xd)
    loss = 0.5 * y.float().pow(2).sum() / n
    loss.backward()
    mod.zero_grad(set_to_none=True)
for _ in range(5):
    step_dev()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    step_dev()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"module step (device-resident x): CPU enqueue {1e3*(t1-t0)/50:.3f} ms/step, wall {1e3*(t2-t0)/50:.3f} ms/step")
h = torch.empty(n, d, dtype=torch.bfloat16).pin_memory()
dd = torch.empty(n, d, dtype=torch.bfloat16, device=dev)
for chunks in (1, 2, 4, 8):
    for _ in range(3):
        dd.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        for c in range(chunks):
            sl = slice(c * n // chunks, (c + 1) * n // chunks)
            dd[sl].copy_(h[sl], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H2D 32 MB in {chunks} chunks: {ms:.3f} ms = {n*d*2/ms/1e6:.1f} GB/s")
