"""Cold-start iteration (all rows through the 3xTF32 resolver + exact pass):
flagged / thin-margin row counts and per-iteration times of the first fit
iterations (c3)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import torch

from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
dev = torch.device("cuda", 0)
P = make_shard(n, d, k, 0, 0, dev)
for rep in range(2):
    eng = LloydEngine(P, k, max_iters=8)
    eng.init_labels_device(0)
    eng.init_centroids_from_labels()
    eng.state.zero_()
    for t in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.iteration(t)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        fc = eng.flag_count.cpu().tolist()
        print(f"rep {rep} it {t}: {dt:8.2f} ms  flagged {fc[0]} ovf {int(eng.ovf_count.item())} "
              f"amb {int(eng.amb_count.item())} two {int(eng.two_count.item())} repairs {int(eng.rep_hist[t].item())}",
              flush=True)
