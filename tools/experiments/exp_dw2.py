"""dW GEMM (dZ^T X, MN-major operands) at C3-like shapes for ncu DRAM/drift studies."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
from paper_2404_01847_b200 import engine as E
n = 32768
for m in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048,8192,22016").split(",")]:
    a = torch.randn(n, m, device="cuda").bfloat16()
    b = torch.randn(n, 4096, device="cuda").bfloat16()
    out = torch.empty(m, 4096, device="cuda")
    for _ in range(2):
        E.gemm_dw(a, True, b, True, m, 4096, n, out)
    del a, b, out
torch.cuda.synchronize()
