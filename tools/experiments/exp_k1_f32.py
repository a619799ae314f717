"""K1 (search + compress of both weights of a block) on fp32 master weights -- the module's
mask refresh every 40 optimizer steps -- vs the bf16 fast path, CUDA-event timed.
python tools/experiments/exp_k1_f32.py"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
from paper_2404_01847_b200 import engine as E

for name, (r, c) in {"c4": (49152, 12288), "c3": (11008, 4096), "c2": (4096, 1024)}.items():
    for dt in (torch.float32, torch.bfloat16):
        w_in = (torch.randn(r, c, device="cuda") / c ** 0.5).to(dt)
        w2 = (torch.randn(c, r, device="cuda") / r ** 0.5).to(dt)
        a = E.CompressedOperand.empty(r, c, "cuda"); b = E.CompressedOperand.empty(c, r, "cuda")
        f = lambda: E.search_compress_pair(w_in, a, w2, b)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{name} {str(dt)[6:]} K1 pair {ms:.3f} ms", flush=True)
        del w_in, w2, a, b; torch.cuda.empty_cache()
