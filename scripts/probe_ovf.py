"""Which rows overflow the screen's candidate lists at c3 steady state (diagnostic)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from bench import make_shard, CONFIGS
from paper_2501_05587_b200.engine import LloydEngine
cfg = CONFIGS["c3"]; n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda", 0))
eng = LloydEngine(P, k, max_iters=20)
eng.init_labels_device(0)
eng.init_centroids_from_labels()
for t in range(12):
    r = eng.traced_iteration(t) if t == 11 else None
    if r is None:
        eng.iteration(t)
nov = int(eng.ovf_count.item())
rows = eng.ovf_list[:nov].long()
lab = eng.labels[0].long()[rows] if hasattr(eng, "labels") else None
C = eng.C.double()
Pr = P[rows].double()
D = torch.cdist(Pr, C) ** 2
best = D.min(1).values
srt = D.sort(1).values
print("ovf rows", nov, "distinct labels", int(torch.unique(D.argmin(1)).numel()))
print("row norms: ovf mean", float(Pr.norm(dim=1).mean()), "all mean", float(P[:100000].double().norm(dim=1).mean()))
print("best dist mean", float(best.mean()), "2nd-best gap mean", float((srt[:, 1] - srt[:, 0]).mean()),
      "64th gap mean", float((srt[:, 63] - srt[:, 0]).mean()))
cn = C.norm(dim=1)
print("centroid norm min/mean/max", float(cn.min()), float(cn.mean()), float(cn.max()))
cc = torch.cdist(C, C); cc.fill_diagonal_(1e30)
print("min centroid-centroid distance", float(cc.min()), "pairs < 1.0:", int((cc < 1.0).sum()) // 2)
am = D.argmin(1)
u, cnts = torch.unique(am, return_counts=True)
print("top labels of ovf rows", list(zip(u[cnts.argsort(descending=True)][:8].tolist(), cnts.sort(descending=True).values[:8].tolist())))
print("bstat", eng.bstat[:8].tolist())
