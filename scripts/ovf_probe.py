"""Which rows does the E4M3 screen hand to the 3xTF32 resolver in steady state
(c3)?  Prints candidate counts from pass 2, |p|, the exact top-2 gap."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np
import torch

from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
dev = torch.device("cuda", 0)
P = make_shard(n, d, k, 0, 0, dev)
eng = LloydEngine(P, k, max_iters=8)
eng.init_labels_device(0)
eng.init_centroids_from_labels()
for t in range(6):
    C_in = eng.C.cpu().numpy().astype(np.float64)
    eng.iteration(t)
torch.cuda.synchronize()
amb = int(eng.amb_count.item()); two = int(eng.two_count.item()); ovf = int(eng.ovf_count.item())
print("amb", amb, "two", two, "ovf", ovf, "bypass", eng.bypass, "flagged", int(eng.flag_count.item()))
cn = eng.cand_n[:amb].cpu().numpy()
print("pass-2 candidate count histogram:", np.bincount(np.minimum(cn, 70))[[0, 1, 2, 3, 4, 8, 16, 32, 64, 65, 66, 69]]
      if cn.size else None, "n<1:", int((cn < 1).sum()), "n>64:", int((cn > 64).sum()))
rows = eng.ovf_list[:ovf].cpu().numpy()
print("ovf rows sample:", rows[:10])
Pr = P[torch.from_numpy(rows[:500]).to(dev)].cpu().numpy().astype(np.float64)
D = ((Pr[:, None, :] - C_in[None, :, :]) ** 2).sum(-1)
srt = np.sort(D, axis=1)
print("|p|^2 mean", (Pr ** 2).sum(1).mean(), "all rows", float((P[:100000].double() ** 2).sum(1).mean()))
print("d1 mean", srt[:, 0].mean(), "d2-d1 mean", (srt[:, 1] - srt[:, 0]).mean(), "d65-d1", (srt[:, 64] - srt[:, 0]).mean())
print("centroid norms range", (C_in ** 2).sum(1).min(), (C_in ** 2).sum(1).max())
cnt = eng.acc[k * d:k * d + k].cpu().numpy()
print("counts min/max", cnt.min(), cnt.max(), "zero counts", int((cnt == 0).sum()))
dup = 0
Cs = np.unique(C_in, axis=0)
print("distinct centroids", Cs.shape[0], "of", k)
print("bstat", eng.bstat.cpu().numpy()[:9])
