"""Run a few C2 FFN steps (for ncu): python tools/prof_one_step.py [steps]"""
import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = bench.CONFIGS[os.environ.get("S24_CFG", "c2")]
w_in, bias, w2, x, dy = bench.make_problem(cfg, torch.device("cuda"), 1)
st = bench.SparseStep(w_in, bias, w2, cfg["act"], 1)
for _ in range(steps):
    st(x, dy)
torch.cuda.synchronize()
print("done")
