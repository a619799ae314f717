"""K1 (search + compress) timing and ncu target: C3 W_in (22016 x 4096, gated)."""
import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E

rows, cols, ff = 22016, 4096, 11008
w = torch.randn(rows, cols, device="cuda").bfloat16()
op = E.CompressedOperand.empty(rows, cols, "cuda", perm_ff=ff)
E.search_compress(w, op)
for _ in range(3):
    E.search_compress(w, op)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
algo = rows * cols * (2 * 2 + 0.3125)
torch.cuda._sleep(1_000_000)
e0.record()
for _ in range(20):
    E.search_compress(w, op)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("K1", round(ms, 4), "ms", round(algo / ms / 1e6, 1), "GB/s")
