"""K8 MVUE sparsifier (fast / exact) on C3's dZ (32768 x 22016), for ncu."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E
exact = len(sys.argv) > 1 and sys.argv[1] == "exact"
g = (torch.randn(32768, 22016, device="cuda") * 1e-3).bfloat16()
for i in range(3):
    E.mvue_compress(g, 12345 + i, exact=exact)
torch.cuda.synchronize()
