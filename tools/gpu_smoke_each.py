"""Run each kernel family once with a synchronize after it; report which fails."""
import sys, os, traceback
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2404_01847_b200._capi as C
from paper_2404_01847_b200 import engine as E, transposable_search_conv

C.load(); C.call("s24_device_check")
def step(name, fn):
    try:
        fn(); torch.cuda.synchronize(); print("OK  ", name, flush=True)
    except Exception as e:
        print("FAIL", name, repr(e)[:300], flush=True); sys.exit(1)

w = torch.randn(256, 256, device="cuda").bfloat16()
op = E.CompressedOperand.empty(256, 256, "cuda")
step("search", lambda: transposable_search_conv(w))
step("search_compress", lambda: E.search_compress(w, op))
z = torch.randn(512, 128, device="cuda").bfloat16(); a = torch.empty(256, 128, device="cuda").bfloat16()
step("act_fwd", lambda: C.call("s24_act_fwd", z.data_ptr(), 128, 256, 128, 2, a.data_ptr(), 128, C.stream_of(z)))
dz = torch.empty_like(z); db = torch.empty(512, device="cuda")
step("act_bwd", lambda: C.call("s24_act_bwd", z.data_ptr(), 128, a.data_ptr(), 128, 256, 128, 2, dz.data_ptr(), 128, db.data_ptr(), C.stream_of(z)))
A = torch.randn(128, 64, device="cuda").bfloat16(); B = torch.randn(128, 64, device="cuda").bfloat16()
out = torch.empty(128, 128, device="cuda")
step("gemm_dw KK", lambda: E.gemm_dw(A, False, B, False, 128, 128, 64, out))
x = torch.randn(128, 256, device="cuda").bfloat16(); o = torch.empty(256, 128, device="cuda").bfloat16()
step("spmm K", lambda: E.spmm(op.fwd_vals, op.fwd_e, 256, 256, x, False, 128, o))
xt = x.t().contiguous()
step("spmm MN", lambda: E.spmm(op.fwd_vals, op.fwd_e, 256, 256, xt, True, 128, o))
print("ALL OK")
