"""s24_transpose_bf16 GB/s at the MVUE token-operand shapes.  python tools/time_transpose.py"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E
for r, c in [(16384, 12288), (16384, 49152), (32768, 4096), (32768, 11008)]:
    x = torch.randn(r, c, device="cuda").bfloat16()
    E.transpose_bf16(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        E.transpose_bf16(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{r}x{c}: {ms:.3f} ms {4 * r * c / ms / 1e6:.0f} GB/s", flush=True)
