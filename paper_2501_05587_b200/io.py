"""Dataset loading and result writing (the reference's io.py:16-117).

Same functions, arguments, outputs and error messages as the reference:
``load_libsvm`` / ``load_csv`` parse text into a dense n x d matrix and raise
``ValueError`` with the reference's message (path:line: ...) on the first
problem the reference would hit; ``write_results`` writes one label per line
plus the ``.timings.csv`` sibling.  The parsing runs in the native library
(csrc/io_text.cpp, multi-threaded C++), not in Python.

``synthesize_points`` (cli.py:102-105) draws the reference's uniform dataset
on the device (bit-identical PCG64 stream, init.cu).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib as L
from .clustering import ClusteringResult
from .validation import normalize_dtype

_TEXT_LEN = 1 << 16


def _load(fn: str, path, n: int, d: int, dtype, zero: bool) -> np.ndarray:
    dt = normalize_dtype(dtype)
    n, d = int(n), int(d)
    spath = os.fspath(path)
    # the reference allocates np.zeros((n, d)) first: negative sizes raise there
    out = np.zeros((n, d), dtype=dt) if zero else np.empty((n, d), dtype=dt)
    info = (ctypes.c_int64 * 4)()
    text = ctypes.create_string_buffer(_TEXT_LEN)
    rc = getattr(L.load(), fn)(os.fsencode(spath), n, d, int(dt == np.float64), out.ctypes.data, info, text,
                              _TEXT_LEN, 0)
    if rc > 0:
        raise OSError(rc, os.strerror(rc), spath)
    if rc == -4:
        raise ValueError(_message(spath, n, d, info, text))
    L.check(rc, fn)
    return out


def _message(path: str, n: int, d: int, info, text) -> str:
    kind, lineno, count = int(info[0]), int(info[1]), int(info[2])
    tok = text.value.decode("utf-8", errors="surrogateescape")
    if kind == 1:
        return f"{path}:{lineno}: malformed label {tok!r}"
    if kind == 2:
        return f"{path}:{lineno}: malformed feature token {tok!r}"
    if kind == 3:
        return f"{path}:{lineno}: feature index {int(tok)} out of range [1, {d}]"
    if kind == 4:
        return f"{path}: expected {n} data lines, found {count}"
    if kind == 5:
        return f"{path}: file is empty"
    if kind == 6:
        return f"{path}:{lineno}: non-numeric cell in row {tok!r}"
    if kind == 7:
        return f"{path}:{lineno}: expected {d} columns, found {count}"
    if kind == 8:
        return f"{path}: expected {n} data rows, found {count}"
    return f"{path}: parse error {kind}"


def load_libsvm(path, n: int, d: int, dtype=np.float32) -> np.ndarray:
    """Read the first ``n`` points of a libsvm file into a dense n x d matrix (io.py:16-46)."""
    return _load("pcb_load_libsvm", path, n, d, dtype, zero=True)


def load_csv(path, n: int, d: int, dtype=np.float32) -> np.ndarray:
    """Read an n x d CSV file; a single leading non-numeric header row is skipped (io.py:49-77)."""
    return _load("pcb_load_csv", path, n, d, dtype, zero=False)


def write_results(result: ClusteringResult, path) -> None:
    """One cluster index per line, plus a ``<path>.timings.csv`` sibling (io.py:88-117)."""
    path = str(path)
    try:
        labels = np.asarray(result.labels).astype(np.int64, copy=False)
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(map(str, labels.tolist())) + ("\n" if labels.size else ""))
        t = result.timings
        with open(path + ".timings.csv", "w", encoding="utf-8") as fh:
            fh.write("phase,seconds\n")
            fh.write(f"kernel_matrix,{t.kernel_matrix_seconds:.9f}\n")
            fh.write(f"pairwise_distances,{t.pairwise_distances_seconds:.9f}\n")
            fh.write(f"argmin_update,{t.argmin_update_seconds:.9f}\n")
    except OSError as exc:
        raise OSError(f"failed to write results to {path!r}: {exc}") from exc


def synthesize_points(n: int, d: int, seed: int, dtype=np.float32, device=None, as_tensor: bool = False):
    """Uniform [0, 1) dataset from the seeded PCG64 stream (cli.py:102-105),
    drawn on the device.  Returns numpy like the reference, or the CUDA tensor
    itself with ``as_tensor=True`` (no round trip through the host)."""
    import torch

    from .engine import _p, _stream, require_cuda
    dt = normalize_dtype(dtype)
    n, d, seed = int(n), int(d), int(seed)
    if n < 0 or d < 0:
        raise ValueError("negative dimensions are not allowed")
    if seed < 0 or seed >= 1 << 64:
        raise ValueError(f"seed must be a non-negative integer below 2**64, got {seed}")
    dev = require_cuda(device)
    with torch.cuda.device(dev):
        out = torch.empty((n, d), dtype=torch.float64 if dt == np.float64 else torch.float32, device=dev)
        if n * d > 0:
            L.call("pcb_synthesize_uniform", n * d, seed, int(dt == np.float64), _p(out), _stream())
    return out if as_tensor else out.cpu().numpy()


__all__ = ["load_libsvm", "load_csv", "write_results", "synthesize_points"]
