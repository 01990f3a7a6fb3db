"""Per-iteration update mode (0 full / 1 delta), changed fraction and repairs at a config (probe)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))
eng = LloydEngine(P, k, max_iters=30)
eng.init_labels_device(0); eng.init_centroids_from_labels(); eng.state.zero_()
kd = k * d
for t in range(10):
    eng.iteration(t)
    torch.cuda.synchronize()
    print(t, "mode", int(eng.state[6]), "changed", round(float(eng.acc[kd + k + 1]) / n, 5),
          "repairs", int(eng.rep_hist[t]), flush=True)
