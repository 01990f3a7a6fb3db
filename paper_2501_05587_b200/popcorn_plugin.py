"""Registration of the B200 Lloyd driver in the reference's plugin registry.

The reference dispatches drivers through ``popcorn.estimator._ALGORITHMS``
(``pkg/src/popcorn/estimator.py:18``); ``KernelKMeans.fit`` calls
``_ALGORITHMS[self.algorithm](X, cfg)`` (``estimator.py:107``) with the
reference's own ``KKMeansConfig`` and expects the reference's
``ClusteringResult`` back.  ``register(popcorn)`` adds ``"lloyd_b200"`` (and,
with ``replace_lloyd=True``, substitutes ``"lloyd"``) so that

    import popcorn, paper_2501_05587_b200.popcorn_plugin as plug
    plug.register(popcorn)
    popcorn.KernelKMeans(n_clusters=64, algorithm="lloyd_b200").fit(X)

runs the reference's estimator on the B200 path.  INTEGRATION.md §1.
"""
from __future__ import annotations


def make_driver(popcorn):
    """driver(points, cfg) -> popcorn.ClusteringResult over run_lloyd (B200)."""
    from . import clustering as b200

    def run_lloyd_b200(points, cfg):
        res = b200.run_lloyd(points, b200.KKMeansConfig(
            k=cfg.k, max_iters=cfg.max_iters, tol=cfg.tol, check_convergence=cfg.check_convergence,
            seed=cfg.seed, dtype=cfg.dtype))
        t = res.timings
        return popcorn.clustering.ClusteringResult(
            labels=res.labels, iterations_run=res.iterations_run, objective_history=res.objective_history,
            converged=res.converged,
            timings=popcorn.clustering.TimingBreakdown(0.0, t.pairwise_distances_seconds, t.argmin_update_seconds),
            label_history=res.label_history, repairs=res.repairs)

    run_lloyd_b200.__doc__ = "Drop-in for popcorn.run_lloyd on a B200 (clustering.py:291-325)."
    return run_lloyd_b200


def register(popcorn, replace_lloyd: bool = False):
    """Add "lloyd_b200" to popcorn.estimator._ALGORITHMS (and optionally
    substitute "lloyd"); returns the driver."""
    drv = make_driver(popcorn)
    popcorn.estimator._ALGORITHMS["lloyd_b200"] = drv
    if replace_lloyd:
        popcorn.estimator._ALGORITHMS["lloyd"] = drv
    return drv
