"""Isolated C4 dense dW GEMM with the masked decay (dW_in = dZ^T X + lam (1 - M) W, K = 16384
tokens), CUDA-event timed (10 launches after 2 warm-ups).  python tools/experiments/exp_dw_iso.py"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
from paper_2404_01847_b200 import engine as E

dev = torch.device("cuda")
torch.manual_seed(0)
m, n, k = 49152, 12288, 16384
w = (torch.randn(m, n, device=dev) / n ** 0.5).to(torch.bfloat16)
op = E.CompressedOperand.empty(m, n, dev)
E.search_compress(w, op)
dz = torch.randn(k, m, device=dev).to(torch.bfloat16)
x = torch.randn(k, n, device=dev).to(torch.bfloat16)
dw = torch.empty(m, n, device=dev)
f = lambda: E.gemm_dw(dz, True, x, True, m, n, k, dw, w, op.idx, 6e-5)
for _ in range(2):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
print(f"dw_in c4 {e0.elapsed_time(e1) / 10:.3f} ms  ({2.0 * m * n * k / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12:.0f} TFLOP/s)")
