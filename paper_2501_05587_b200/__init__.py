"""B200-native K-means of arXiv 2501.05587 (reference: `popcorn`).

Drop-in for the reference's drivers: the same ``run_lloyd`` / ``run_popcorn``
/ ``run_baseline(points, cfg)`` contract, ``KKMeansConfig``/``ClusteringResult``
types, the ``KernelKMeans`` estimator, the dataset loaders and the CLI,
computed by hand-written sm_100a kernels behind the C ABI in
``include/popcorn_b200.h``.
"""
from .clustering import (ClusteringResult, KKMeansConfig, TimingBreakdown, init_assignments,
                         lloyd_step, run_lloyd)
from .estimator import _ALGORITHMS, KernelKMeans
from .io import load_csv, load_libsvm, synthesize_points, write_results
from .kernels import GRAM_VARIANTS, KERNEL_FAMILIES, GramMethod, KernelSpec, select_gram_algorithm
from .kkmeans import run_baseline, run_popcorn
from .validation import as_float_matrix, check_labels, normalize_dtype

__version__ = "0.1.0"

__all__ = [
    "GRAM_VARIANTS",
    "GramMethod",
    "KERNEL_FAMILIES",
    "KernelSpec",
    "run_baseline",
    "run_popcorn",
    "select_gram_algorithm",
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
