"""One training step of the 2:4 FFN block (K1 refresh, fwd, bwd with the fused decay), one K2
step, and one fused dense step, for compute-sanitizer (memcheck / racecheck / synccheck).
mvue: the same block with the MVUE weight gradient (K8 exact: certified fp32 + float64 fallback,
then the forced float64 path), the token-operand transpose and the two-slab 2:4 dW GEMM (run with
S24_SDW_SLABS=1 so the small shape takes it).
python tools/sanitize_step.py <c2|c5|c3-small|mvue|train>
train: run_training (gated epilogues, K1, MVUE exact, fused Adam + compression) and the autograd
module on fp32 parameters (the fp32 K2 path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench as B  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = dict(B.CONFIGS["c5" if name == "c5" else "c2"])
if name == "c5":
    cfg["layers"] = 1  # one block of the GPT-2 large stack
if name == "c3-small":  # the gated (SwiGLU) epilogues at a sanitizer-friendly size
    cfg = dict(d=1024, d_ff=2816, act="swiglu", tokens=4096, workload="c3-shaped small")
dev = torch.device("cuda", 0)
w_in, bias, w2, x, dy = B.make_problem(cfg, dev, 1)
if name == "train":
    # the training-loop kernels: run_training (GEGLU, K1 refreshes, MVUE exact, the fused fp32
    # Adam + next-step compression) and the autograd module on fp32 parameters (K2 fp32 path)
    import paper_2404_01847_b200 as P
    from paper_2404_01847_b200.module import SparseFFN

    P.run_training(P.TrainConfig(d=256, d_ff=512, depth=1, batch=256, steps=4))
    mod = SparseFFN(256, 512, act="gelu", decay_lambda=1e-4, device=dev)
    xin = torch.randn(512, 256, device=dev).bfloat16()
    for _ in range(2):
        y = mod(xin)
        y.float().square().sum().backward()
        with torch.no_grad():
            for prm in mod.parameters():
                prm -= 1e-3 * prm.grad
                prm.grad = None
elif name == "mvue":
    from paper_2404_01847_b200 import engine as E

    st = B.SparseStep(w_in, bias, w2, cfg["act"], 1, mvue="exact")
    st(x, dy)  # refresh step: K1 + fwd + bwd with K8 exact, transposes, two-slab 2:4 dW GEMMs
    st(x, dy)
    E.mvue_compress(dy, 3, exact=2)  # the float64 path for every group
else:
    st = B.SparseStep(w_in, bias, w2, cfg["act"], 1)
    st(x, dy)  # refresh step: K1 + fwd + bwd
    st(x, dy)  # K2 step
    B.DenseFusedStep(w_in, bias, w2, cfg["act"])(x, dy)
torch.cuda.synchronize()
print("sanitize step ok", name)
