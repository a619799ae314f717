"""Decode how the sm_100a sparse MMA interprets our (values, E-tile) operand.

With B = identity (n == k), D[m, k] = A_hw[m, k]: the decompressed A as the
tensor core sees it.  Two runs with stored values = row id and = slot id tell,
for every (m, k), which stored (row, slot) landed there.  Prints a summary of
mismatches vs the intended decompression.  Also runs a dense GEMM sanity check.
"""
import sys, os, json
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2404_01847_b200._capi as C
from paper_2404_01847_b200.engine import CompressedOperand, spmm, gemm_dw, compress_with_meta
from paper_2404_01847_b200 import TransposableMask

C.load(); C.call("s24_device_check")
report = {}
# dense sanity
a = torch.randn(128, 64, device="cuda").bfloat16(); b = torch.randn(128, 64, device="cuda").bfloat16()
out = torch.empty(128, 128, device="cuda")
gemm_dw(a, False, b, False, 128, 128, 64, out)
ref = a.float() @ b.float().t()
report["dense_rel"] = float((out - ref).norm() / ref.norm())
M = K = 128
w = torch.randn(M, K, device="cuda").bfloat16()
op = CompressedOperand.empty(M, K, "cuda")
from paper_2404_01847_b200.engine import search_compress
search_compress(w, op)
bits = TransposableMask(op.idx, (M, K)).bits
eye = torch.eye(K, device="cuda").bfloat16()  # B[n, k] = 1 iff n == k
res = {}
for name, fill in (("row", lambda r, s: r + 1), ("slot", lambda r, s: s + 1)):
    vals = torch.empty(M, K // 2, device="cuda")
    rr = torch.arange(M, device="cuda")[:, None].float().expand(M, K // 2)
    ss = torch.arange(K // 2, device="cuda")[None, :].float().expand(M, K // 2)
    vals = fill(rr, ss).bfloat16().contiguous()
    d = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    spmm(vals, op.fwd_e, M, K, eye, False, K, d)
    res[name] = d.float().cpu()
torch.cuda.synchronize()
# intended: position (m, k) kept -> row m, slot = rank of k among kept in row m
bits_c = bits.cpu()
slot_of = torch.cumsum(bits_c.long(), dim=1) - 1
want_row = torch.where(bits_c.bool(), torch.arange(M)[:, None].float() + 1, torch.zeros(1))
want_slot = torch.where(bits_c.bool(), slot_of.float() + 1, torch.zeros(1))
report["row_match"] = float((res["row"] == want_row).float().mean())
report["slot_match"] = float((res["slot"] == want_slot).float().mean())
bad = (res["row"] != want_row) | (res["slot"] != want_slot)
report["n_bad"] = int(bad.sum())
if report["n_bad"]:
    idx = bad.nonzero()[:40].tolist()
    report["examples"] = [(m, k, int(bits_c[m, k]), float(res["row"][m, k]) - 1, float(res["slot"][m, k]) - 1,
                           float(want_slot[m, k]) - 1) for m, k in idx]
    # per (m % 16, k % 32) failure histogram
    hist = torch.zeros(16, 32)
    for m, k in bad.nonzero().tolist():
        hist[m % 16, k % 32] += 1
    report["hist_m16_k32"] = hist.int().tolist()
print(json.dumps(report))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(report, open("gpurun_out/debug_sparse.json", "w"))
