import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import make_shard
from paper_2501_05587_b200.engine import LloydEngine
n, d, k = 10_000_000, 128, 1024
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))
eng = LloydEngine(P, k, variant="bf16s", max_iters=30)
eng.state = torch.zeros(48, dtype=torch.int64, device="cuda")
eng.init_labels_device(0); eng.init_centroids_from_labels()
for t in range(8):
    eng.state[8:].zero_()
    eng.iteration(t); torch.cuda.synchronize()
    c = eng.state[8:41].cpu().numpy()
    warps = n / 32
    print(t, "full-path fraction per chunk position (first 2 tiles):", np.round(c[:8] / warps, 3), "rest avg", round(float(c[8:32].sum() / warps / 24), 3), "total", round(float(c[:33].sum() / warps / 32), 3), flush=True)
