"""Debug helper: which rows of the candidate-overflow case disagree with the exact argmin."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from conftest import make_rng
from paper_2501_05587_b200.engine import LloydEngine

rng = make_rng(23)
n, d, k = 4000, 96, 64
C = rng.uniform(-10, 10, size=(k, d)).astype(np.float32)
C[50:62] = C[50] + rng.normal(0, 1e-3, size=(12, d)).astype(np.float32)
true = rng.integers(0, k, size=n)
P = (C[true] + rng.normal(0, 1, size=(n, d))).astype(np.float32)
for variant in ("bf16s", "tc1xtf32s", "tc3xtf32"):
    eng = LloydEngine(P, k, variant=variant, max_iters=1)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = ((P64[:, None, :] - C64[None, :, :]) ** 2).sum(-1)
    exact = D.argmin(1)
    srt = np.sort(D, 1)
    gap = (srt[:, 1] - srt[:, 0]) / srt[:, 0]
    raw = out["raw_labels"]
    bad = np.flatnonzero((raw != exact) & (gap >= 1e-5))
    print(variant, "bad", len(bad), "amb", int(eng.amb_count.item()) if hasattr(eng, "amb_count") else None,
          "ovf", int(eng.ovf_count.item()) if hasattr(eng, "ovf_count") else None)
    if variant == "bf16s":
        amb = eng.amb_list[:int(eng.amb_count.item())].cpu().numpy()
        ovf = set(eng.ovf_list[:int(eng.ovf_count.item())].cpu().numpy().tolist())
        cn = eng.cand_n[:len(amb)].cpu().numpy()
        cand = eng.cand[:len(amb)].cpu().numpy()
        thr = eng.amb_thr[:len(amb)].cpu().numpy()
        pos = {int(r): i for i, r in enumerate(amb)}
    for r in bad[:10]:
        info = ""
        if variant == "bf16s":
            i = pos.get(int(r))
            info = f"amb_pos={i} ovf={int(r) in ovf} " + (f"nc={cn[i]} cand={cand[i][:min(cn[i],8)]} thr={thr[i]}" if i is not None else "")
        print(f"  row {r} gpu {raw[r]} exact {exact[r]} gap {gap[r]:.3g} D[gpu]={D[r, raw[r]]:.6f} D[ex]={D[r, exact[r]]:.6f} {info}")
