"""Kernel K-means (f4) throughput on one B200: K build + per-iteration time.

    python scripts/bench_kernel.py [--n 60000 --d 784 --k 10 --family polynomial --iters 10]

Synthetic blobs on the device; K (n x n f32) resident in HBM.  Per iteration
the dominant kernel streams K once (segmented row sums), so the roofline is
HBM: algorithmic bytes/iter = 4 n^2 (K) + 8 k n (S write + read).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_05587_b200.kernels import KernelSpec  # noqa: E402
from paper_2501_05587_b200.kkmeans import KernelEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=60000)
    ap.add_argument("--d", type=int, default=784)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--family", default="polynomial")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.rand((a.k, a.d), device="cuda", generator=g)
    idx = torch.randint(0, a.k, (a.n,), device="cuda", generator=g)
    P = (centers[idx] + 0.1 * torch.randn((a.n, a.d), device="cuda", generator=g)).contiguous()
    spec = KernelSpec(family=a.family, gamma=1.0 / a.d, coef=1.0, degree=2)
    KernelEngine(P[:1024].contiguous(), a.k, spec, max_iters=1)  # module load / first-launch costs
    torch.cuda.synchronize()
    eng = KernelEngine(P, a.k, spec, max_iters=a.warmup + a.iters)
    kms = eng.kernel_matrix_seconds() * 1e3
    eng.init_labels_device(0)
    eng.state.zero_()
    for t in range(a.warmup):
        eng.iteration(t)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.iters)]
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(a.iters):
        eng.iteration(a.warmup + i, events=evs[i])
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    dist_ms = float(np.mean([x[0].elapsed_time(x[1]) for x in evs]))
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    bytes_iter = 4.0 * a.n * a.n + 16.0 * a.k * a.n
    gram_flops = 3 * 2.0 * a.n * a.n * a.d / 2  # upper triangle, 3 TF32 products
    print(json.dumps({
        "workload": f"kernel k-means n={a.n} d={a.d} k={a.k} {a.family}",
        "kernel_matrix_ms": kms, "iter_ms": ms, "iters_per_s": 1e3 / ms, "distance_phase_ms": dist_ms,
        "hbm_roofline": {"bytes_per_iter": bytes_iter, "achieved_GBs": bytes_iter / (ms * 1e-3) / 1e9,
                         "peak_GBs": peaks["hbm_gbs"], "frac": bytes_iter / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
        "gram": {"tf32_mma_tflops": gram_flops / (kms * 1e-3) / 1e12,
                 "write_GBs": 4.0 * a.n * a.n / (kms * 1e-3) / 1e9},
        "objective_last": float(eng.obj_hist[a.warmup + a.iters - 1].item()),
    }))


if __name__ == "__main__":
    main()
