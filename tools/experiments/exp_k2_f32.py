import sys, torch
sys.path.insert(0, ".")
from paper_2404_01847_b200 import engine as E
for name, (r, c) in {"c4": (49152, 12288), "c3": (11008, 4096), "c2": (4096, 1024)}.items():
    w_in = (torch.randn(r, c, device="cuda") / c ** 0.5)
    w2 = (torch.randn(c, r, device="cuda") / r ** 0.5)
    a = E.CompressedOperand.empty(r, c, "cuda"); b = E.CompressedOperand.empty(c, r, "cuda")
    E.search_compress_pair(w_in, a, w2, b)
    f = lambda: E.compress_values_pair(w_in, a, w2, b)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    el = w_in.numel() + w2.numel()
    print(f"{name} fp32 K2 pair {ms:.3f} ms  {el * (4 + 2 + 1/16) / ms / 1e6:.0f} GB/s")
    del w_in, w2, a, b; torch.cuda.empty_cache()
