"""bench.py's e2e leg with per-phase wall timers patched onto LloydEngine (diagnostic, under gpurun)."""
import sys, os, time, functools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, make_shard
import paper_2501_05587_b200 as pcb
from paper_2501_05587_b200 import engine as E

T = {}
def timed(name, f):
    @functools.wraps(f)
    def w(*a, **kw):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **kw)
        torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t
        return r
    return w
for nm in ("__init__", "init_labels_device", "init_centroids_from_labels", "run", "collect"):
    setattr(E.LloydEngine, nm, timed(nm, getattr(E.LloydEngine, nm)))

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
dev = torch.device("cuda")
if len(sys.argv) > 2:  # simulate the main bench leg's footprint first
    x = torch.empty(int(float(sys.argv[2]) * 2**30), dtype=torch.uint8, device=dev); del x
P_host = make_shard(n, d, k, 0, 0, dev).cpu().numpy()
torch.cuda.empty_cache()
c = pcb.KKMeansConfig(k=k, max_iters=30, record_label_history=False)
pcb.run_lloyd(P_host[:100_000], pcb.KKMeansConfig(k=k, max_iters=2))
torch.cuda.synchronize()
for rep in range(3):
    T.clear()
    t0 = time.perf_counter()
    res = pcb.run_lloyd(P_host, c)
    wall = time.perf_counter() - t0
    print(f"rep {rep} wall {wall*1e3:.1f} ms", {k_: round(v * 1e3, 1) for k_, v in T.items()}, flush=True)
