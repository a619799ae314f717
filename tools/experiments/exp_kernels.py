"""Per-kernel times inside full steps (CUDA events on the launching stream).
python tools/experiments/exp_kernels.py <cfg> [steps]  -- env knobs (S24_GROUP_M, ...) are read by the library."""
import json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
import bench
from paper_2404_01847_b200 import engine as E

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w_in, bias, w2, x, dy = bench.make_problem(cfg, torch.device("cuda"), 1)
st = bench.SparseStep(w_in, bias, w2, cfg["act"], 1)
for _ in range(5):
    st(x, dy)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    st(x, dy)
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1) / steps
timer = bench.EventTimer()
E.TIMER = timer
for _ in range(steps):
    st(x, dy)
tot = timer.totals()
E.TIMER = E._NoTimer()
out = {k: round(v[0] / v[1], 4) for k, v in sorted(tot.items())}
out["step_ms"] = round(step_ms, 4)
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("S24_")}
print(json.dumps(out))
