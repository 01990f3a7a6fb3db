"""Generate golden fixtures for the Lloyd hot path FROM THE REFERENCE ITSELF.

Run in the authoring container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs on small seeded instances into ``lloyd_golden.npz``.  The
fixtures pin (a) the oracle restatement in ``oracle/`` and (b) the GPU path in
the parity tests.  Nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lloyd_golden.npz")


def _instances():
    """(name, points, k, seed, dtype, check_convergence, tol, max_iters)."""
    out = []
    # acceptance grid of the reference (test_acceptance.py:37-50): uniform [0,1)
    grid = [(n, d, k) for n in (64, 256, 512) for d in (2, 16) for k in (2, 10, 50)]
    grid += [(512, 2, 10), (256, 16, 50)]
    for i, (n, d, k) in enumerate(grid):
        P = np.random.Generator(np.random.PCG64(4000 + i)).random((n, d))
        for dt in ("f64", "f32"):
            out.append((f"grid{i}_{dt}", P, k, i, dt, False, 0.0, 30))
    # blobs (test_clustering.py:153-160 style) and estimator-style blobs
    rng = np.random.Generator(np.random.PCG64(6))
    blobs = np.vstack([rng.normal(loc=c, scale=0.3, size=(25, 3)) for c in (0.0, 4.0, 8.0)])
    out.append(("blobs75_f64", blobs, 3, 2, "f64", False, 0.0, 30))
    out.append(("blobs75_f32", blobs, 3, 2, "f32", False, 0.0, 30))
    # k == n fixpoint (test_clustering.py:140-145)
    P = np.random.Generator(np.random.PCG64(5)).random((4, 2))
    out.append(("fixpoint4", P, 4, 0, "f32", True, 0.0, 30))
    # 1-D pairs (test_clustering.py:147-151)
    out.append(("pairs1d", np.array([[0.0], [0.1], [10.0], [10.1]]), 2, 1, "f64", True, 0.0, 30))
    # convergence with tolerance
    P = np.random.Generator(np.random.PCG64(16)).random((60, 4))
    out.append(("tol1", P, 4, 0, "f32", True, 1.0, 30))
    out.append(("conv_blobs", blobs, 3, 5, "f32", True, 0.0, 100))
    # repair-heavy instances: many duplicate points so clusters empty out
    for s in range(6):
        g = np.random.Generator(np.random.PCG64(100 + s))
        base = np.zeros((40, 3))
        spread = g.normal(0.0, 5.0, size=(24, 3))
        P = np.vstack([base, spread])
        g.shuffle(P)
        for dt in ("f32", "f64"):
            out.append((f"repair{s}_{dt}", P, 12, s, dt, False, 0.0, 10))
    # larger blob instances at the shapes of the benchmark configs (scaled down)
    for name, (n, d, k) in {"c1": (2000, 2, 10), "c2": (3000, 16, 64),
                            "c3": (1024, 128, 64), "c4": (384, 784, 12),
                            "c5": (2048, 64, 128)}.items():
        g = np.random.Generator(np.random.PCG64(7))
        centers = g.uniform(-10, 10, size=(k, d))
        true = g.integers(0, k, size=n)
        P = (centers[true] + g.normal(0, 1, size=(n, d))).astype(np.float32)
        out.append((f"blob_{name}", P, k, 0, "f32", False, 0.0, 8))
    return out


def main():
    sys.path.insert(0, REF)
    import popcorn
    from popcorn import (KKMeansConfig, KernelSpec, augmented_distance_oracle,
                         init_assignments, repair_empty_clusters, run_lloyd)
    from popcorn.clustering import _mean_centroids

    g = {}
    # init goldens (clustering.py:91-108)
    inits = [(100, 10, 42), (64, 5, 7), (12, 9, 3), (3, 3, 11), (1000, 37, 0), (4, 1, 99)]
    g["init_cases"] = np.array(inits, dtype=np.int64)
    for i, (n, k, s) in enumerate(inits):
        g[f"init_{i}"] = init_assignments(n, k, s)

    # repair goldens (clustering.py:111-139)
    rep = []
    rep.append((np.array([0, 0, 0, 0]), np.array([[1.0, 9], [2, 9], [3, 9], [4, 9]]), 2))
    rep.append((np.array([0, 0, 0]), np.array([[5.0, 0], [5, 0], [1, 0]]), 2))
    for s in range(8):
        r = np.random.Generator(np.random.PCG64(s))
        n, k = 20 + s, 6 + s % 3
        labels = r.integers(0, 2, size=n)
        rep.append((labels, r.random((n, k)), k))
    g["repair_count"] = np.array(len(rep))
    for i, (lab, D, k) in enumerate(rep):
        g[f"repair_{i}_labels"] = lab.astype(np.int32)
        g[f"repair_{i}_D"] = D
        g[f"repair_{i}_k"] = np.array(k)
        g[f"repair_{i}_out"] = repair_empty_clusters(lab, D, k)

    # augmented-form worked values (analysis.py:83-102; PAPER.md attachment)
    g["aug_cases"] = np.array([augmented_distance_oracle([3.0], [7.0]),
                               augmented_distance_oracle([1.0], [7.0]),
                               augmented_distance_oracle([5.0, 2.0], [1.0, 4.0]),
                               augmented_distance_oracle([4.0, 3.0, 2.0], [5.0, 2.0, 3.0])])

    names = []
    for (name, P, k, seed, dt, cc, tol, mi) in _instances():
        dtype = np.float32 if dt == "f32" else np.float64
        cfg = KKMeansConfig(k=k, max_iters=mi, tol=tol, check_convergence=cc, seed=seed,
                            kernel=KernelSpec("linear"), dtype=dtype)
        res = run_lloyd(P, cfg)
        Pd = np.ascontiguousarray(P, dtype=dtype)
        cents = [_mean_centroids(Pd, lab, k) for lab in res.label_history]
        g[f"run_{name}_P"] = Pd
        g[f"run_{name}_meta"] = np.array([k, seed, int(cc), mi, 1 if dt == "f32" else 2], dtype=np.int64)
        g[f"run_{name}_tol"] = np.array(tol)
        g[f"run_{name}_labels"] = np.stack(res.label_history)
        g[f"run_{name}_objective"] = res.objective_history
        g[f"run_{name}_repairs"] = res.repairs
        g[f"run_{name}_converged"] = np.array(res.converged)
        g[f"run_{name}_centroids"] = np.stack(cents)
        names.append(name)
    g["run_names"] = np.array(names)
    g["numpy_version"] = np.array(np.__version__)
    g["popcorn_version"] = np.array(popcorn.__version__)
    np.savez_compressed(OUT, **g)
    reps = sum(int(g[f"run_{n}_repairs"].sum() > 0) for n in names)
    print(f"wrote {OUT}: {len(names)} runs ({reps} with repairs), "
          f"{os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
