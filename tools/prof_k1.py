"""K1 (fused search + compress) on one weight, or with `pair` on the weight and its transpose
shape in one launch (the refresh of a block's two weights), a few launches (for ncu).
python tools/prof_k1.py [rows cols [pair]]"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E
rows, cols = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (22016, 4096)))
pair = len(sys.argv) > 3 and sys.argv[3] == "pair"
w = (torch.randn(rows, cols, device="cuda") / cols ** 0.5).bfloat16()
op = E.CompressedOperand.empty(rows, cols, "cuda")
if pair:
    w2 = (torch.randn(cols, rows, device="cuda") / rows ** 0.5).bfloat16()
    op2 = E.CompressedOperand.empty(cols, rows, "cuda")
for _ in range(3):
    if pair:
        E.search_compress_pair(w, op, w2, op2)
    else:
        E.search_compress(w, op)
torch.cuda.synchronize()
