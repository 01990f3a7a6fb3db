"""Worker for the gloo multi-process tests (spawned; CPU only)."""
import os
import pickle
import sys

import numpy as np


def run(rank, world, port, case, out_dir):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist

    import oracle
    from cpu_shard import NumpyShard
    from paper_2501_05587_b200.distributed import Comm, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P, k, iters, seed, cc, tol = case
    n = P.shape[0]
    lo, hi = shard_range(n, rank, world)
    labels0 = oracle.init_assignments(n, k, seed)
    C0 = oracle.mean_centroids_f64(P, labels0, k)
    comm = Comm()
    shard = NumpyShard(P[lo:hi], k, n, lo, comm, labels0[lo:hi], C0, iters)
    res = shard.fit(iters, cc, tol)
    res["lo"], res["hi"] = lo, hi
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()
