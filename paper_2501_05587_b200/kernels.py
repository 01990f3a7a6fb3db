"""Kernel specification and the device kernel matrix (the reference's kernels.py).

``KernelSpec`` / ``GramMethod`` / ``KERNEL_FAMILIES`` / ``GRAM_VARIANTS`` /
``select_gram_algorithm`` keep the reference's names, defaults and validation
(kernels.py:18-82).  ``kernel_matrix`` builds K = kernel(P P^T) in HBM with one
fused kernel (csrc/kernel_kmeans.cu): a tcgen05 3xTF32 GEMM over the upper
triangle with the elementwise kernel in the epilogue (f32), or a SIMT DFMA
GEMM (f64).  K comes out exactly symmetric, like the reference's syrk route;
the gemm/syrk choice of ``GramMethod`` only changes rounding there, so both
map to the same device kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L

KERNEL_FAMILIES = ("linear", "polynomial", "gaussian", "sigmoid")
GRAM_VARIANTS = ("auto", "gemm", "syrk")
GAUSSIAN_EXP_FLOOR = -88.0
FAMILY_CODE = {"linear": 0, "polynomial": 1, "gaussian": 2, "sigmoid": 3}


@dataclass(frozen=True)
class KernelSpec:
    """Kernel family plus parameters (kernels.py:25-54).

    polynomial: (gamma * <x, y> + coef) ** degree
    gaussian:   exp(-gamma * ||x - y||^2 / sigma^2)
    sigmoid:    tanh(gamma * <x, y> + coef)
    linear:     <x, y>
    """

    family: str = "polynomial"
    gamma: float = 1.0
    coef: float = 1.0
    degree: int = 2
    sigma: float = 1.0

    def __post_init__(self):
        if self.family not in KERNEL_FAMILIES:
            raise ValueError(f"unknown kernel family {self.family!r}; expected one of {KERNEL_FAMILIES}")
        if not float(self.degree).is_integer():
            raise ValueError(f"kernel degree must be an integer, got {self.degree!r}")
        object.__setattr__(self, "degree", int(self.degree))
        if self.degree < 1:
            raise ValueError("kernel degree must be >= 1")
        if self.family == "gaussian" and not self.sigma > 0:
            raise ValueError("sigma must be positive for the gaussian kernel")


@dataclass(frozen=True)
class GramMethod:
    """Gram algorithm choice (kernels.py:57-69)."""

    variant: str = "auto"
    threshold: float = 100.0

    def __post_init__(self):
        if self.variant not in GRAM_VARIANTS:
            raise ValueError(f"unknown gram variant {self.variant!r}; expected one of {GRAM_VARIANTS}")
        if not self.threshold > 0:
            raise ValueError("gram threshold must be positive")


def select_gram_algorithm(n: int, d: int, method: GramMethod = GramMethod()) -> str:
    """'gemm' iff n / d > threshold under 'auto' (kernels.py:72-82)."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be >= 1")
    if method.variant != "auto":
        return method.variant
    return "gemm" if n / d > method.threshold else "syrk"


def padded_ld(n: int) -> int:
    """Leading dimension of the device K (rows 128-byte aligned)."""
    return (n + 31) // 32 * 32


def kernel_matrix(P, spec: KernelSpec, out=None):
    """K = kernel(P P^T) on the device (kernels.py:85-131, fused).

    P: CUDA tensor (n x d, f32 or f64).  Returns the n x ldk tensor (ldk =
    padded_ld(n); columns >= n are padding).  Raises FloatingPointError like
    require_finite if any entry is not finite.
    """
    import torch

    from .engine import _p, _stream
    n, d = int(P.shape[0]), int(P.shape[1])
    f64 = P.dtype == torch.float64
    ldk = padded_ld(n)
    dev = P.device
    K = out if out is not None else torch.empty((n, ldk), dtype=P.dtype, device=dev)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
    fam = FAMILY_CODE[spec.family]
    args = (fam, float(spec.gamma), float(spec.coef), int(spec.degree), float(spec.sigma), _p(nonfinite),
            _stream())
    dvec = torch.empty(n, dtype=P.dtype, device=dev)
    L.call(f"pcb_point_norms_{'f64' if f64 else 'f32'}", _p(P), n, d, _p(dvec), _stream())
    if f64:
        L.call("pcb_kernel_gram_f64", _p(P), n, d, _p(dvec), _p(K), ldk, *args)
    else:
        ld = (d + 31) // 32 * 32
        hi = torch.empty((n, ld), dtype=torch.float32, device=dev)
        lo = torch.empty_like(hi)
        L.call("pcb_split_tf32", _p(P), n, d, ld, _p(hi), _p(lo), _stream())
        L.call("pcb_kernel_gram_f32", _p(hi), _p(lo), ld, n, _p(dvec), _p(K), ldk, *args)
        del hi, lo
    if int(nonfinite.item()) != 0:
        raise FloatingPointError(f"apply_kernel[{spec.family}] produced non-finite values")
    return K


__all__ = ["KERNEL_FAMILIES", "GRAM_VARIANTS", "GAUSSIAN_EXP_FLOOR", "KernelSpec", "GramMethod",
           "select_gram_algorithm", "kernel_matrix"]
