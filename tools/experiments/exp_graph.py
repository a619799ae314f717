"""Eager vs CUDA-graph step time and host enqueue time of the bench's sparse step.
python tools/experiments/exp_graph.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch

import bench

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfg_name]
w_in, bias, w2, x, dy = bench.make_problem(cfg, torch.device("cuda"), 1)
st = bench.SparseStep(w_in, bias, w2, cfg["act"], 1)
st.t = 1  # skip the refresh branch


def step():
    st.t = 1
    st(x, dy)


for _ in range(5):
    step()
torch.cuda.synchronize()
# host enqueue time: GPU blocked behind a long sleep so the queue never back-pressures
K = 20
torch.cuda._sleep(int(2e9))
h0 = time.perf_counter()
for _ in range(K):
    step()
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"{cfg_name}: host enqueue {1e3 * (h1 - h0) / K:.3f} ms/step")

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record()
    for _ in range(K):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(f"eager {e0.elapsed_time(e1) / K:.4f} ms/step")

s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for rep in range(3):
    e0.record()
    for _ in range(K):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph {e0.elapsed_time(e1) / K:.4f} ms/step")
