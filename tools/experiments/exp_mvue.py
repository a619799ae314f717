"""Per-kernel times of the MVUE-dW step (fast / exact) at a config."""
import json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
import bench
from paper_2404_01847_b200 import engine as E

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
w_in, bias, w2, x, dy = bench.make_problem(cfg, torch.device("cuda"), 1)
st = bench.SparseStep(w_in, bias, w2, cfg["act"], 1, mvue=mode)
for _ in range(4):
    st(x, dy)
timer = bench.EventTimer()
E.TIMER = timer
for _ in range(10):
    st(x, dy)
tot = timer.totals()
print(json.dumps({k: round(v[0] / v[1], 4) for k, v in sorted(tot.items())}))
