"""Pins the kernel K-means oracle (oracle/kernel_oracle.py) to fixtures produced
by the reference itself (tests/golden/make_kernel_golden.py): kernel matrices
of every family through both Gram routes, and full run_popcorn / run_baseline
label and objective histories.  CPU only."""
import os

import numpy as np
import pytest

import oracle.kernel_oracle as ko
from conftest import ROOT

G = np.load(os.path.join(ROOT, "tests", "golden", "kernel_golden.npz"))
SPECS = {"linear": dict(family="linear"),
         "poly2": dict(family="polynomial", gamma=1.0, coef=1.0, degree=2),
         "poly3": dict(family="polynomial", gamma=0.5, coef=0.25, degree=3),
         "gauss": dict(family="gaussian", gamma=1.0, sigma=1.5),
         "sigmoid": dict(family="sigmoid", gamma=0.05, coef=0.1)}


@pytest.mark.parametrize("name", list(SPECS))
@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("gram", ["gemm", "syrk"])
def test_kernel_matrix_bit_identical(name, dt, gram):
    P = G["kmat_P"].astype(np.float32 if dt == "f32" else np.float64)
    K = ko.apply_kernel(ko.compute_gram(P, gram), **SPECS[name])
    np.testing.assert_array_equal(K, G[f"kmat_{name}_{dt}_{gram}"])


def _spec(run):
    idx, gamma, coef, degree, sigma = G[f"run_{run}_spec"]
    fam = SPECS[str(G["spec_names"][int(idx)])]["family"]
    return dict(family=fam, gamma=float(gamma), coef=float(coef), degree=int(degree), sigma=float(sigma))


@pytest.mark.parametrize("run", [str(r) for r in G["run_names"]])
def test_runs_bit_identical(run):
    k, iters, seed, f64 = (int(x) for x in G[f"run_{run}_meta"])
    P = G[f"run_{run}_P"]
    kw = dict(max_iters=iters, seed=seed, dtype=np.float64 if f64 else np.float32, **_spec(run))
    res = ko.run_popcorn(P, k, **kw)
    np.testing.assert_array_equal(np.stack(res.label_history), G[f"run_{run}_labels"])
    np.testing.assert_array_equal(res.objective_history, G[f"run_{run}_objective"])
    np.testing.assert_array_equal(res.repairs, G[f"run_{run}_repairs"])
    base = ko.run_baseline(P, k, **kw)
    np.testing.assert_array_equal(np.stack(base.label_history), G[f"run_{run}_baseline_labels"])
    np.testing.assert_array_equal(base.objective_history, G[f"run_{run}_baseline_objective"])


def test_repair_case_exercises_repair():
    assert G["run_repair_dups_repairs"].sum() > 0
