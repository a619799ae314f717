"""Isolated sparse / dense GEMMs at C3 shapes (for ncu per-clock efficiency studies).
python tools/experiments/exp_gemm_iso.py [reps]"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
from paper_2404_01847_b200 import engine as E

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda")
torch.manual_seed(0)
n = 32768
shapes = [(4096, 22016), (4096, 11008)]  # (m, k): bwd_in-like, fwd_out-like
for m, k in shapes:
    w = (torch.randn(m, k, device=dev) / k ** 0.5).to(torch.bfloat16)
    op = E.CompressedOperand.empty(m, k, dev)
    E.search_compress(w, op)
    b = torch.randn(n, k, device=dev).to(torch.bfloat16)
    out = torch.empty(n, m, device=dev, dtype=torch.bfloat16)
    for _ in range(reps):
        E.spmm(op.fwd_vals, op.fwd_e, m, k, b, False, n, out, out_t=True)
    del w, op, b, out
# dense dW-like: dW[4096, 11008] = dY^T A, K = 32768 tokens
a = torch.randn(n, 4096, device=dev).to(torch.bfloat16)
bb = torch.randn(n, 11008, device=dev).to(torch.bfloat16)
dw = torch.empty(4096, 11008, device=dev)
for _ in range(reps):
    E.gemm_dw(a, True, bb, True, 4096, 11008, n, dw)
torch.cuda.synchronize()
print("ok")
