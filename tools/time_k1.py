"""K1 (search + compress of a block's two weights in one launch) and K2 GB/s at the config
weight shapes, CUDA-event timed (20 launches after a warm-up), algorithmic bytes of
SURVEY.md section 8(d).  python tools/time_k1.py"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E

SHAPES = {"c2": (4096, 1024, 0), "c3": (22016, 4096, 11008), "c4": (49152, 12288, 0), "c5": (5120, 1280, 0)}
torch.manual_seed(0)
for name, (r, c, ff) in SHAPES.items():
    w_in = (torch.randn(r, c, device="cuda") / c ** 0.5).bfloat16()
    w2 = (torch.randn(c, ff or r, device="cuda") / (ff or r) ** 0.5).bfloat16()
    op_in = E.CompressedOperand.empty(r, c, "cuda", perm_ff=ff)
    op_out = E.CompressedOperand.empty(c, ff or r, "cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def t(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    el = w_in.numel() + w2.numel()
    k1 = t(lambda: E.search_compress_pair(w_in, op_in, w2, op_out))
    k2 = t(lambda: E.compress_values_pair(w_in, op_in, w2, op_out))
    print(f"{name}: K1 {k1 * 1e3:8.1f} us {el * 4.3125 / k1 / 1e6:7.0f} GB/s | K2 {k2 * 1e3:8.1f} us "
          f"{el * 4.0625 / k2 / 1e6:7.0f} GB/s", flush=True)
    del w_in, w2, op_in, op_out
    torch.cuda.empty_cache()
