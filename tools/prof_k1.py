"""K1 (fused search + compress) on the C3 first weight, a few launches (for ncu)."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E
rows, cols = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (22016, 4096)))
w = (torch.randn(rows, cols, device="cuda") / cols ** 0.5).bfloat16()
op = E.CompressedOperand.empty(rows, cols, "cuda")
for _ in range(3):
    E.search_compress(w, op)
torch.cuda.synchronize()
