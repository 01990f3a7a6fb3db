"""B200-native Lloyd hot path of arXiv 2501.05587's K-means (reference: `popcorn`).

Drop-in for the reference's Lloyd path: the same ``run_lloyd(points, cfg)``
driver contract, ``KKMeansConfig``/``ClusteringResult`` types and the
``KernelKMeans(algorithm="lloyd")`` estimator, computed by hand-written sm_100a
kernels behind the C ABI in ``include/popcorn_b200.h``.
"""
from .clustering import (ClusteringResult, KKMeansConfig, TimingBreakdown, init_assignments,
                         lloyd_step, run_lloyd)
from .estimator import _ALGORITHMS, KernelKMeans
from .io import load_csv, load_libsvm, synthesize_points, write_results
from .validation import as_float_matrix, check_labels, normalize_dtype

__version__ = "0.1.0"

__all__ = [
    "ClusteringResult",
    "KKMeansConfig",
    "KernelKMeans",
    "TimingBreakdown",
    "as_float_matrix",
    "check_labels",
    "init_assignments",
    "load_csv",
    "load_libsvm",
    "lloyd_step",
    "normalize_dtype",
    "run_lloyd",
    "synthesize_points",
    "write_results",
]
