import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from bench import make_shard, CONFIGS
from paper_2501_05587_b200.engine import LloydEngine
cfg = CONFIGS["c3"]; n, d, k = cfg["n"], cfg["d"], cfg["k"]
if len(sys.argv) > 1: n = int(sys.argv[1])
P = make_shard(n, d, k, 0, 0, torch.device("cuda", 0))
eng = LloydEngine(P, k, max_iters=20)
eng.init_labels_device(0)
eng.init_centroids_from_labels()
for t in range(14):
    r = eng.traced_iteration(t) if t >= 11 else None
    if r is None:
        eng.iteration(t)
    else:
        print(t, r["screen"], "flagged", int(eng.flag_count.item()), "ovf", int(eng.ovf_count.item()), "mode", r["update_mode"])
