"""Standalone K8 (MVUE compress) timing on a 16384 x 4096 bf16 gradient."""
import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E

g = torch.randn(16384, 4096, device="cuda").bfloat16()
for ex in (False, True):
    for _ in range(3):
        E.mvue_compress(g, 5, exact=ex)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
algo = g.numel() * 2 * 1.5 + g.numel() // 4 * 0.125 * 8 / 8  # read G, write G/2 values + E
for ex in (False, True):
    torch.cuda._sleep(2_000_000)  # queue ahead so host launch overhead is hidden
    e0.record()
    for _ in range(20):
        E.mvue_compress(g, 5, exact=ex)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("MVUE exact" if ex else "MVUE fast", round(ms, 4), "ms", round(algo / ms / 1e6, 1), "GB/s")
