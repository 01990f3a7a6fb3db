"""The drop-in through the reference's own plugin registry.

The unmodified reference package (installed offline into baseline/_ref by
scripts/install_reference.sh; it travels to the GPU box with the repo) is
imported, ``paper_2501_05587_b200.popcorn_plugin.register`` adds the B200
driver to ``popcorn.estimator._ALGORITHMS`` (estimator.py:18), and
``popcorn.KernelKMeans(algorithm="lloyd_b200")`` — the reference's estimator,
dispatching at estimator.py:107 — is compared with
``KernelKMeans(algorithm="lloyd")`` (the reference's numpy driver) on the
golden grid of seeded runs: f64 runs must reproduce the reference exactly
(labels, iterations, convergence, objective history, repairs); f32 runs to
the north-star tolerance.
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_runs

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def popcorn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "popcorn")):
        pytest.skip("reference not installed (scripts/install_reference.sh)")
    sys.path.insert(0, REF)
    import popcorn as pc
    from paper_2501_05587_b200 import popcorn_plugin
    popcorn_plugin.register(pc)
    yield pc
    pc.estimator._ALGORITHMS.pop("lloyd_b200", None)


def _meta(golden, name):
    k, seed, cc, mi, dtc = (int(x) for x in golden[f"run_{name}_meta"])
    return k, seed, bool(cc), mi, ("float32" if dtc == 1 else "float64")


def _check_f32_objectives(P, k, seed, got, ref, name):
    """Inertia per iteration, f32 runs.

    The reference's objective (clustering.py:146) sums its f32 expansion
    pn - 2 p.c + cn (clustering.py:311), which carries its own rounding error
    (~2^-22 of pn + cn per row).  Where the label histories agree, the step's
    centroids are known (f32 means of the previous labels, clustering.py:282),
    so the EXACT f64 inertia is computable: ours must be within 1e-6 of it
    (the north-star bar, no allowance), and the reference's within its own
    expansion error of it.
    """
    P32 = np.asarray(P, dtype=np.float32)
    P64 = P32.astype(np.float64)
    pn = (P64 ** 2).sum(1)
    prev = oracle.init_assignments(P32.shape[0], k, seed)
    gh, rh = got.result_.label_history, ref.result_.label_history
    for t in range(min(len(gh), len(rh))):
        C = oracle.mean_centroids(P32, prev, k).astype(np.float64)
        if not np.array_equal(gh[t], rh[t]):
            break
        lab = rh[t]
        exact = float(((P64 - C[lab]) ** 2).sum())
        g, r = got.objective_history_[t], ref.objective_history_[t]
        assert abs(g - exact) <= 1e-6 * abs(exact), (name, t, g, exact)
        ref_err = 2.0 ** -22 * float((pn + (C ** 2).sum(1)[lab]).sum())
        assert abs(r - exact) <= 1e-6 * abs(exact) + ref_err, (name, t, r, exact)
        prev = lab


def test_registry_dispatch_matches_reference_estimator(popcorn, golden):
    checked = 0
    for name in golden_runs(golden):
        k, seed, cc, mi, dt = _meta(golden, name)
        P = golden[f"run_{name}_P"]
        kw = dict(n_clusters=k, max_iter=mi, check_convergence=cc, random_state=seed, dtype=dt)
        ref = popcorn.KernelKMeans(algorithm="lloyd", **kw).fit(P)
        got = popcorn.KernelKMeans(algorithm="lloyd_b200", **kw).fit(P)
        assert got.n_iter_ == ref.n_iter_ and got.converged_ == ref.converged_, name
        if dt == "float64":
            np.testing.assert_array_equal(got.labels_, ref.labels_, err_msg=name)
            np.testing.assert_array_equal(np.stack(got.result_.label_history), np.stack(ref.result_.label_history))
            np.testing.assert_array_equal(got.result_.repairs, ref.result_.repairs)
            # the reference's f64 expansion (clustering.py:311) cancels on exact fits
            np.testing.assert_allclose(got.objective_history_, ref.objective_history_, rtol=1e-12, atol=1e-12)
        else:
            _check_f32_objectives(P, k, seed, got, ref, name)
            assert np.mean(got.labels_ == ref.labels_) >= 0.999, name
        # (the reference's predict branches on algorithm == "lloyd" — a new
        # name takes its kernel branch; test_replace_lloyd_in_registry covers it)
        assert got.score(P) == -got.inertia_
        checked += 1
    assert checked >= 24


def test_replace_lloyd_in_registry(popcorn):
    from paper_2501_05587_b200 import popcorn_plugin
    rng = np.random.Generator(np.random.PCG64(3))
    X = np.vstack([rng.normal(c, 0.3, size=(200, 5)) for c in (0.0, 4.0, 8.0)])
    ref = popcorn.KernelKMeans(n_clusters=3, algorithm="lloyd", dtype="float64", random_state=1).fit(X)
    saved = popcorn.estimator._ALGORITHMS["lloyd"]
    try:
        popcorn_plugin.register(popcorn, replace_lloyd=True)
        got = popcorn.KernelKMeans(n_clusters=3, algorithm="lloyd", dtype="float64", random_state=1).fit(X)
    finally:
        popcorn.estimator._ALGORITHMS["lloyd"] = saved
    np.testing.assert_array_equal(got.labels_, ref.labels_)
    assert got.inertia_ == pytest.approx(ref.inertia_, rel=1e-12)
    np.testing.assert_array_equal(got.predict(X), ref.predict(X))  # the reference's Lloyd predict branch
