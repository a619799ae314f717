import sys, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch, bench
from paper_2404_01847_b200 import engine as E
cfg = bench.CONFIGS[os.environ.get("S24_CFG", "c2")]
w_in, bias, w2, x, dy = bench.make_problem(cfg, torch.device("cuda"), 1)
for mode in ("fast", "exact", None):
    st = bench.SparseStep(w_in, bias, w2, cfg["act"], 1, mvue=mode)
    for _ in range(3): st(x, dy)
    t = bench.EventTimer(); E.TIMER = t
    for _ in range(5): st(x, dy)
    tot = t.totals(); E.TIMER = E._NoTimer()
    print(mode, {k: round(v[0] / v[1] * 1000, 1) for k, v in tot.items()})
