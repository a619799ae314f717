"""K8 (MVUE sparsifier) per-launch time at the config gradient shapes, exact (certified) vs
exact=2 (float64 everywhere) vs fast.  python tools/time_k8.py"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2404_01847_b200 import engine as E

SHAPES = {"c2": (16384, 4096, 0), "c3": (32768, 22016, 11008), "c4": (16384, 49152, 0)}
for name, (n, f, ff) in SHAPES.items():
    g = (torch.randn(n, f, device="cuda") * 0.01).bfloat16()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for mode in (1, 2, 0):
        E.mvue_compress(g, 7, gate_ff=ff, exact=mode)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            E.mvue_compress(g, 7, gate_ff=ff, exact=mode)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 5
    gb = n * f * 2 * 1.5625 / 1e9  # read G + write values (half) + E tiles
    print(f"{name}: exact {res[1]:.3f} ms | float64-only {res[2]:.3f} ms | fast {res[0]:.3f} ms "
          f"({gb / res[1] * 1e3:.0f} / {gb / res[0] * 1e3:.0f} GB/s)", flush=True)
    del g
    torch.cuda.empty_cache()
