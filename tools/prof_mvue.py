import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E
g = torch.randn(16384, 4096, device="cuda").bfloat16()
for ex in (False, True):
    for _ in range(2):
        E.mvue_compress(g, 5, exact=ex)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for ex in (False, True):
    e0.record(); E.mvue_compress(g, 5, exact=ex); e1.record(); torch.cuda.synchronize()
    print("exact" if ex else "fast", e0.elapsed_time(e1), "ms")
