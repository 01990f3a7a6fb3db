"""Per-iteration time of one rank's shard at N GPUs (n/N rows, single process,
no collective): the compute part of the strong-scaling run.  Under gpurun."""
import sys, os, time, json, subprocess
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for N in (1, 2, 4, 8):
    n = 10_000_000 // N
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "c3", "--no-e2e",
                          "--no-cpu-baseline", "--n-override", str(n)], capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        r = d["roofline"]
        print(f"N={N} shard n={n}: {d['ms_per_step']:.3f} ms/iter, kernel {r['kernel_ms']:.3f}, assign {r['assign_ms']:.3f}, update {r['update_ms']:.3f}", flush=True)
    except Exception:
        print(out.stderr[-500:])
