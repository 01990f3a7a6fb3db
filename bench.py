#!/usr/bin/env python
"""Lloyd-iteration throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A step is one full Lloyd iteration over the whole dataset (distance+argmin,
centroid update, all-reduce when N>1, repair check, finalize).  Inputs are
synthetic blobs generated on the device and resident in HBM before timing
(P is larger than L2 for c2-c5).  Multi-GPU: launched by torchrun, one rank
per GPU, rows sharded (strong scaling: total n fixed), NCCL all-reduce of the
fused k*(d+1)+2 accumulator each iteration; time = max over ranks.

Rank 0 prints ONE JSON line.  --impl reference times the reference's CPU
algorithm (the oracle port of popcorn.run_lloyd) on a bounded row sample,
extrapolated linearly in n (per-iteration cost is O(n*k)).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(n=100_000, d=2, k=10),
    "c2": dict(n=1_000_000, d=16, k=64),
    "c3": dict(n=10_000_000, d=128, k=1024),
    "c4": dict(n=4_000_000, d=784, k=256),
    "c5": dict(n=100_000_000, d=64, k=4096),
}
METRIC = "Lloyd iters/sec & point-centroid dists/sec (n=10M,d=128,k=1024) at 1/2/4/8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=1)
        if not self.rows:
            return None
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_shard(n_local: int, d: int, k: int, rank: int, seed: int, device):
    """Synthetic blobs on the device: centers ~ U(-10,10)^{k x d} (PCG64, shared by
    all ranks), true labels uniform, N(0,1) noise (per-rank CUDA generator)."""
    import torch
    centers = np.random.Generator(np.random.PCG64(seed)).uniform(-10, 10, size=(k, d)).astype(np.float32)
    cdev = torch.from_numpy(centers).to(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 1_000_003 + rank)
    P = torch.empty((n_local, d), dtype=torch.float32, device=device)
    chunk = 1 << 22
    for s in range(0, n_local, chunk):
        e = min(n_local, s + chunk)
        true = torch.randint(0, k, (e - s,), generator=gen, device=device)
        P[s:e] = cdev[true] + torch.randn((e - s, d), generator=gen, device=device)
    return P


def cpu_reference_time(P_sample: np.ndarray, k: int, iters: int, threads: int):
    """Oracle port of popcorn.run_lloyd on a row sample; seconds per iteration."""
    import oracle
    t0 = time.perf_counter()
    res = oracle.run_lloyd(P_sample, k, max_iters=iters, seed=0, dtype=np.float32)
    wall = time.perf_counter() - t0
    t = res.timings
    per_iter = (t.pairwise_distances_seconds + t.argmin_update_seconds) / max(1, res.iterations_run)
    return per_iter, wall


def _sample_rows(n: int, d: int, k: int, budget_s: float, rate: float = 6e7) -> int:
    """Rows so that one reference iteration takes ~budget_s at `rate` dists/s."""
    return int(max(min(n, 2000), min(n, budget_s * rate / k)))


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("internal_api") in ("openblas", "mkl", "blis")]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, k = cfg["n"], cfg["d"], cfg["k"]
    ns = _sample_rows(n, d, k, budget_s=args.ref_budget)
    import torch
    # same synthetic recipe as the GPU arm, generated on the CPU for the sample
    centers = np.random.Generator(np.random.PCG64(args.seed)).uniform(-10, 10, size=(k, d))
    g = np.random.Generator(np.random.PCG64(args.seed + 17))
    P = (centers[g.integers(0, k, size=ns)] + g.normal(0, 1, size=(ns, d))).astype(np.float32)
    threads = blas_threads()
    import oracle
    pn = oracle.point_norms(P)
    lab = oracle.init_assignments(ns, k, 0)
    C = oracle.mean_centroids(P, lab, k)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        st = oracle.lloyd_step(P, pn, C, lab, k)
        dt = time.perf_counter() - t0
        C, lab = st.centroids, st.labels
        if s >= args.warmup:
            times.append(dt)
    t_sample = float(np.mean(times))
    t_full = t_sample * n / ns
    value = 1.0 / t_full
    sample = f"{ns} of {n} rows, one Lloyd iteration per step, extrapolated x{n / ns:.1f} in n"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic blobs (host, PCG64)",
        "config": {"workload": args.config, **cfg},
        "dists_per_sec": n * k / t_full,
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ref-budget", type=float, default=4.0, help="seconds per reference iteration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of one CUDA graph")
    ap.add_argument("--n-override", type=int, default=0, help="diagnostics only: rows of the config")
    ap.add_argument("--e2e-iters", type=int, default=30)
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.n_override > 0:
        cfg["n"] = args.n_override
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_2501_05587_b200 import _lib
    from paper_2501_05587_b200.distributed import Comm, init_from_env, shard_range
    from paper_2501_05587_b200.engine import LloydEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        init_from_env("nccl")
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = Comm() if world > 1 else None

    n, d, k = cfg["n"], cfg["d"], cfg["k"]
    lo, hi = shard_range(n, rank, world)
    P = make_shard(hi - lo, d, k, rank, args.seed, dev)
    W, K = args.warmup, args.steps
    eng = LloydEngine(P, k, variant=args.variant, comm=comm, n_total=n, max_iters=W + K + 1)
    if comm is not None:
        comm.offset = lo
    eng.init_labels_device(0, lo)  # init_assignments(n, k, 0), drawn on the device
    eng.init_centroids_from_labels()
    for t in range(W):
        eng.iteration(t)
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    # single rank: the K timed iterations are one captured CUDA graph (every
    # decision is on the device; external event nodes time each iteration and
    # the dominant kernel inside it); multi-rank: eager (host repair check)
    use_graph = world == 1 and not args.no_graph
    evs = None
    if use_graph:
        try:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(5)] for _ in range(K)]
            with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
                for s in range(K):
                    eng.iteration(W + s, events=evs[s])
            torch.cuda.current_stream().wait_stream(cs)
        except Exception as exc:  # eager fallback, same kernels
            print(f"bench: graph capture failed ({exc!r}); timing eagerly", file=sys.stderr)
            use_graph = False
    if not use_graph:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    torch.cuda.synchronize()
    start.record()
    if use_graph:
        g.replay()
    else:
        for s in range(K):
            eng.iteration(W + s, events=evs[s])
    end.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if comm is not None:
        comm.barrier()
    ms = start.elapsed_time(end)
    assign_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    upd_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    kern_ms = float(np.mean([e[3].elapsed_time(e[4]) for e in evs]))
    t = torch.tensor([ms, assign_ms, upd_ms, kern_ms], dtype=torch.float64, device=dev)
    if comm is not None:
        comm.all_reduce_max(t)
    ms, assign_ms, upd_ms, kern_ms = (float(x) for x in t.cpu())
    st = eng.state.cpu().numpy()
    if st[5] != 0:
        raise SystemExit("non-finite distances during the bench")
    amb = int(eng.amb_count.item()) if getattr(eng, "amb_count", None) is not None else None
    if amb is not None and getattr(eng, "two_count", None) is not None:
        amb += int(eng.two_count.item())  # two-candidate rows resolved without the second pass

    ms_per_step = ms / K
    value = 1e3 / ms_per_step  # whole-job iterations/s (all ranks, n total)
    peaks, peak_src = _peaks()
    n_local = hi - lo
    flops = 2.0 * n_local * k * d  # algorithmic: one dot product per point-centroid pair
    if d <= 32 and eng.variant not in ("tc3xtf32", "tc1xtf32s", "bf16s", "fp8s"):
        # small-d FFMA path: report against HBM (bytes of P read + labels)
        traffic_alg = n_local * (4 * d + 8 + 4) + k * d * 4
        roof = {"bound": "hbm", "achieved": traffic_alg / (kern_ms * 1e-3) / 1e9,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "traffic": None,
                "peak_source": f"{peak_src} copy bandwidth"}
    else:
        # kind::tf32 issues at half the bf16 rate; the burst bf16 figure is used
        # (the kernel runs near max clocks, see "clocks"), i.e. the larger peak.
        tf32 = peaks["bf16_tflops"] / 2.0
        if eng.variant == "tc3xtf32":  # three TF32 products per dot product
            peak, src = tf32 / 3.0, "3xTF32 effective = bf16 burst / 6"
        elif eng.variant == "bf16s":  # one BF16 (kind::f16) pass
            peak, src = peaks["bf16_tflops"], "bf16 burst (dense)"
        elif eng.variant == "fp8s":  # one E4M3 (kind::f8f6f4) pass: twice the BF16 rate
            peak, src = 2.0 * peaks["bf16_tflops"], "fp8 = 2 x bf16 burst (dense, derived)"
        else:
            peak, src = tf32, "TF32 = bf16 burst / 2"
        roof = {"bound": "tensor", "achieved": flops / (kern_ms * 1e-3) / 1e12, "peak": peak,
                "unit": "TFLOP/s", "traffic": None, "peak_source": f"{peak_src} {src}"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    scr = {"res": "assign_screen_res_kernel", "pair": "assign_screen_2sm_kernel",
           "stream": "assign_screen_kernel"}.get(os.environ.get("PCB_SCREEN_IMPL", "res"), "assign_screen_res_kernel")
    roof["kernel"] = {"tc1xtf32s": scr, "tc3xtf32": "assign_tc3xtf32_kernel",
                      "bf16s": "assign_screen_bf16_kernel", "fp8s": "assign_screen_bf16_kernel<F8>"}.get(
        eng.variant, f"assign[{eng.variant}]")
    roof["kernel_ms"] = kern_ms
    roof["algorithmic_per_launch"] = f"2*n*k*d = {flops:.4g} flop" if roof["unit"] == "TFLOP/s" else \
        f"{traffic_alg:.4g} bytes"
    roof["assign_ms"] = assign_ms
    roof["update_ms"] = upd_ms
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{eng.variant}.json")
    if os.path.exists(prof):
        try:
            roof["traffic"] = json.load(open(prof)).get("bytes_per_launch")
        except Exception:
            pass

    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",  # inputs/results f32; the screen's operands are bf16/e4m3, certified exact
        "data": "synthetic blobs generated on device (centers U(-10,10), N(0,1) noise)",
        "config": {"workload": f"{args.config}: n={n} d={d} k={k}", "n": n, "d": d, "k": k,
                   "variant": eng.variant, "parallelism": f"dp{world} row-sharded",
                   "launch": "cuda graph (K iterations)" if use_graph else "eager",
                   "l2": "inputs larger than L2" if n * d * 4 > 126e6 else "inputs fit in L2 (no flush)"},
        "dists_per_sec": n * k / (ms_per_step * 1e-3),
        "roofline": roof,
        # library kernels per steady-state iteration (counted from the ncu launch
        # lists in profiles/), plus the relayouts that fall inside the window
        "gpu_launches": {"fp8s": 21, "bf16s": 19, "tc1xtf32s": 15}.get(eng.variant, 9) * K
                        + sum(1 for t in getattr(eng, "RELAYOUT_AT", ()) if W <= t < W + K
                              and eng.variant in ("fp8s", "bf16s")),
        "screen_ambiguous_rows_last_iter": amb,
        "clocks": clocks,
    }
    del eng, P
    if n * d * 4 > 20e9:  # very large shards (c5): return the cache before the e2e fit
        torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_e2e:
        line["e2e"] = e2e_run(args, cfg, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns = _sample_rows(n, d, k, budget_s=args.ref_budget)
        Ps = make_shard(ns, d, k, 0, args.seed, dev).cpu().numpy()
        per_iter, _ = cpu_reference_time(Ps, k, 2, blas_threads())
        line["cpu_baseline"] = {"value": 1.0 / (per_iter * n / ns), "unit": "iters/s",
                                "cores": blas_threads(), "kind": "port",
                                "sample": f"{ns} of {n} rows, 2 iterations, extrapolated linearly in n"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_run(args, cfg, dev):
    """Through the public drop-in API with host buffers: run_lloyd(P_host, cfg)."""
    import torch
    import paper_2501_05587_b200 as pcb
    n, d, k = cfg["n"], cfg["d"], cfg["k"]
    P_host = make_shard(n, d, k, 0, args.seed, dev).cpu().numpy()
    if n * d * 4 > 20e9:
        torch.cuda.empty_cache()
    # otherwise the allocator keeps the blocks of the timed leg's fit (same
    # sizes), as in a process that has fitted before
    it = args.e2e_iters
    c = pcb.KKMeansConfig(k=k, max_iters=it, record_label_history=False)
    pcb.run_lloyd(P_host[: min(n, 100_000)], pcb.KKMeansConfig(k=k, max_iters=2))  # warm libs + staging buffers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pcb.run_lloyd(P_host, c)
    wall = time.perf_counter() - t0
    h2d = n * d * 4 + n * 4
    d2h = n * 4 + it * 16 + k * d * 4
    return {"value": res.iterations_run / wall, "unit": "iters/s",
            "h2d_bytes_per_step": h2d // it, "d2h_bytes_per_step": d2h // it,
            "step": f"one run_lloyd(host numpy, max_iters={it}) call = {it} steps", "wall_s": wall}


if __name__ == "__main__":
    sys.exit(main())
