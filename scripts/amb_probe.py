import sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import make_shard
from paper_2501_05587_b200.engine import LloydEngine
from paper_2501_05587_b200.clustering import init_assignments
n, d, k = 2_000_000, 128, 1024
P = make_shard(n, d, k, 0, 0, torch.device('cuda'))
eng = LloydEngine(P, k, variant='tc1xtf32s', max_iters=20)
eng.init_centroids_from_labels(init_assignments(n, k, 0))
for t in range(8):
    eng.iteration(t)
    torch.cuda.synchronize()
    print(t, 'amb', eng.amb_count.item(), 'bstat', eng.bstat.cpu().numpy(), 'dan med', eng.danorm.median().item(), 'an med', eng.anorm.median().item())
