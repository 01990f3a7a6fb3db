"""Golden fixtures for the kernel K-means path (f4), produced by running the
reference itself (pkg/src/popcorn: compute_gram/apply_kernel, run_popcorn,
run_baseline).  Run in the authoring container:
    python tests/golden/make_kernel_golden.py
Writes tests/golden/kernel_golden.npz.  Tests never import the reference.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from popcorn import KKMeansConfig  # noqa: E402
from popcorn.clustering import run_baseline, run_popcorn  # noqa: E402
from popcorn.kernels import GramMethod, KernelSpec, apply_kernel, compute_gram  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def blobs(seed, n, d, c, spread=0.3, scale=1.0):
    g = np.random.default_rng(seed)
    centers = g.uniform(-scale, scale, size=(c, d))
    return centers[g.integers(0, c, size=n)] + g.normal(0, spread, size=(n, d))


def main():
    out = {}
    specs = {
        "linear": KernelSpec("linear"),
        "poly2": KernelSpec("polynomial", gamma=1.0, coef=1.0, degree=2),
        "poly3": KernelSpec("polynomial", gamma=0.5, coef=0.25, degree=3),
        "gauss": KernelSpec("gaussian", gamma=1.0, sigma=1.5),
        "sigmoid": KernelSpec("sigmoid", gamma=0.05, coef=0.1),
    }
    # kernel matrices (both gram routes)
    P = blobs(1, 150, 7, 4)
    out["kmat_P"] = P
    for name, sp in specs.items():
        for dt in ("f32", "f64"):
            Pd = P.astype(np.float32 if dt == "f32" else np.float64)
            for g in ("gemm", "syrk"):
                out[f"kmat_{name}_{dt}_{g}"] = apply_kernel(compute_gram(Pd, GramMethod(g)), sp)
    # full runs
    runs = [
        ("blobs_poly2", blobs(2, 300, 5, 6), 6, specs["poly2"], 12, 3, "f32"),
        ("blobs_poly2_f64", blobs(2, 300, 5, 6), 6, specs["poly2"], 12, 3, "f64"),
        ("blobs_gauss", blobs(3, 400, 3, 5, scale=3.0), 5, specs["gauss"], 15, 1, "f32"),
        ("blobs_linear", blobs(4, 256, 8, 4, scale=2.0), 4, specs["linear"], 10, 0, "f32"),
        ("blobs_sigmoid", blobs(5, 200, 6, 3, scale=2.0), 3, specs["sigmoid"], 10, 2, "f64"),
        ("uniform_poly3", np.random.default_rng(6).random((500, 4)), 8, specs["poly3"], 20, 5, "f32"),
        ("repair_dups", np.vstack([np.zeros((60, 3)), np.random.default_rng(7).normal(0, 3, (20, 3))]), 12,
         specs["gauss"], 6, 4, "f64"),
    ]
    out["run_names"] = np.array([r[0] for r in runs])
    for name, P, k, sp, iters, seed, dt in runs:
        cfg = KKMeansConfig(k=k, max_iters=iters, seed=seed, kernel=sp, dtype=np.float32 if dt == "f32" else np.float64)
        res = run_popcorn(P, cfg)
        out[f"run_{name}_P"] = P
        out[f"run_{name}_meta"] = np.array([k, iters, seed, 0 if dt == "f32" else 1])
        out[f"run_{name}_spec"] = np.array([list(specs).index([s for s in specs if specs[s] == sp][0]),
                                            sp.gamma, sp.coef, sp.degree, sp.sigma])
        out[f"run_{name}_labels"] = np.stack(res.label_history)
        out[f"run_{name}_objective"] = res.objective_history
        out[f"run_{name}_repairs"] = res.repairs
        base = run_baseline(P, cfg)
        out[f"run_{name}_baseline_labels"] = np.stack(base.label_history)
        out[f"run_{name}_baseline_objective"] = base.objective_history
    out["spec_names"] = np.array(list(specs))
    np.savez_compressed(os.path.join(HERE, "kernel_golden.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
