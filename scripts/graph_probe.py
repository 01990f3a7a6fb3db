"""Can a whole Lloyd iteration sequence be captured in one CUDA graph? (probe, under gpurun)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = CONFIGS[cfgname]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))

def make():
    e = LloydEngine(P, k, max_iters=40)
    e.init_labels_device(0)
    e.init_centroids_from_labels()
    e.state.zero_()
    for t in range(4):
        e.iteration(t)
    torch.cuda.synchronize()
    return e

ref = make()
t0 = time.perf_counter()
for t in range(4, 24):
    ref.iteration(t)
torch.cuda.synchronize()
t_eager = time.perf_counter() - t0

eng = make()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for t in range(4, 24):
            eng.iteration(t)
torch.cuda.synchronize()
t0 = time.perf_counter()
g.replay()
torch.cuda.synchronize()
t_graph = time.perf_counter() - t0
same = torch.equal(ref.labels[0], eng.labels[0]) and torch.equal(ref.labels[1], eng.labels[1])
print(cfgname, "eager ms/iter", t_eager / 20 * 1e3, "graph ms/iter", t_graph / 20 * 1e3, "labels equal", same,
      "C maxdiff", (ref.C - eng.C).abs().max().item(), "iters", int(ref.state[0]), int(eng.state[0]))
