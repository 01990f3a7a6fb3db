"""Default-contract (label_history on) fit at c3: wall time of two consecutive calls."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import make_shard, CONFIGS
import paper_2501_05587_b200 as pcb
cfg = CONFIGS["c3"]; n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda", 0)).cpu().numpy()
pcb.run_lloyd(P[:100000], pcb.KKMeansConfig(k=k, max_iters=2))
for hist in (False, True, True):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, max_iters=30, record_label_history=hist))
    print("history", hist, "wall", round(time.perf_counter() - t, 3), "s", len(r.label_history), flush=True)
