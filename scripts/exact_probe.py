"""How many ambiguous rows of each kind, and how many take the f64 fallback? (probe)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))
eng = LloydEngine(P, k, max_iters=30)
eng.init_labels_device(0); eng.init_centroids_from_labels(); eng.state.zero_()
for t in range(8):
    eng.iteration(t)
torch.cuda.synchronize()
amb = int(eng.amb_count.item()); two = int(eng.two_count.item()); ovf = int(eng.ovf_count.item())
cn = eng.cand_n[:min(amb, eng.cand_n.numel())].cpu().numpy()
print("two-candidate rows", two, "pass-2 rows", amb, "overflow rows", ovf)
print("pass-2 candidate counts:", np.bincount(np.minimum(cn, 70))[:71].nonzero()[0].tolist(), np.bincount(np.minimum(cn, 70)).tolist()[-8:])
