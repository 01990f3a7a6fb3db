"""Dataset loaders (f3) against fixtures produced by the reference's own
io.load_libsvm / io.load_csv (tests/golden/make_io_golden.py), plus the
reference's test_io.py cases.  CPU only: the parser is host C++ in the library.
"""
import json
import os

import numpy as np
import pytest

import paper_2501_05587_b200 as pcb
from paper_2501_05587_b200.io import load_csv, load_libsvm, write_results
from conftest import ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden")
META = json.load(open(os.path.join(GOLDEN, "io_golden.json")))
ARR = np.load(os.path.join(GOLDEN, "io_golden.npz"))


@pytest.mark.parametrize("case", META, ids=[m["name"] for m in META])
def test_matches_reference_loader(case, tmp_path):
    name = case["name"]
    path = tmp_path / (name + (".libsvm" if case["format"] == "libsvm" else ".csv"))
    path.write_bytes(ARR["content_" + name].tobytes())
    fn = load_libsvm if case["format"] == "libsvm" else load_csv
    dt = np.float32 if case["dtype"] == "f32" else np.float64
    if case["error"] is not None:
        with pytest.raises(ValueError) as ei:
            fn(path, case["n"], case["d"], dtype=dt)
        assert str(ei.value) == case["error"].replace("{PATH}", str(path))
    else:
        got = fn(path, case["n"], case["d"], dtype=dt)
        want = ARR["expect_" + name]
        assert got.dtype == want.dtype and got.shape == want.shape
        np.testing.assert_array_equal(got, want)  # bit-exact (NaN == NaN)
        assert np.array_equal(np.signbit(got), np.signbit(want))


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(FileNotFoundError):
        load_csv(tmp_path / "nope.csv", 1, 1)
    with pytest.raises(IsADirectoryError):
        load_libsvm(tmp_path, 1, 1)


def test_negative_sizes_raise_like_numpy(tmp_path):
    f = tmp_path / "a.csv"
    f.write_text("1,2\n")
    with pytest.raises(ValueError):
        load_csv(f, -1, 2)


def test_thread_count_does_not_change_results(tmp_path):
    from paper_2501_05587_b200 import _lib
    import ctypes
    g = np.random.default_rng(3)
    X = g.standard_normal((4096, 7)).astype(np.float32)
    f = tmp_path / "t.csv"
    f.write_text("".join(",".join(repr(float(v)) for v in r) + "\n" for r in X))
    outs = []
    for th in (1, 3, 16):
        out = np.empty_like(X)
        info = (ctypes.c_int64 * 4)()
        assert _lib.load().pcb_load_csv(str(f).encode(), 4096, 7, 0, out.ctypes.data, info, None, 0, th) == 0
        outs.append(out)
    for o in outs:
        np.testing.assert_array_equal(o, X)


# ---- the reference's own test_io.py cases -------------------------------------
def test_reference_basic_libsvm(tmp_path):
    f = tmp_path / "a.libsvm"
    f.write_text("1 1:0.5 3:2.0\n")
    np.testing.assert_allclose(load_libsvm(f, 1, 3), [[0.5, 0.0, 2.0]])


def test_reference_malformed_line_number(tmp_path):
    f = tmp_path / "bad.libsvm"
    f.write_text("1 1:0.5\n1 oops\n")
    with pytest.raises(ValueError, match=":2:"):
        load_libsvm(f, 2, 2)


def test_reference_csv_round_trip(tmp_path):
    data = np.random.default_rng(5).random((1000, 6)).astype(np.float32)
    f = tmp_path / "big.csv"
    f.write_text("".join(",".join(repr(float(v)) for v in row) + "\n" for row in data))
    np.testing.assert_array_equal(load_csv(f, 1000, 6), data)


def test_write_results_format(tmp_path):
    labels = np.array([0, 1, 0], dtype=np.int32)
    res = pcb.ClusteringResult(labels=labels, iterations_run=1, objective_history=np.array([0.0]),
                               converged=True, timings=pcb.TimingBreakdown(1.0, 2.0, 0.5),
                               label_history=[labels], repairs=np.array([0]))
    path = tmp_path / "out.labels"
    write_results(res, path)
    assert path.read_text() == "0\n1\n0\n"
    lines = (tmp_path / "out.labels.timings.csv").read_text().splitlines()
    assert lines == ["phase,seconds", "kernel_matrix,1.000000000", "pairwise_distances,2.000000000",
                     "argmin_update,0.500000000"]
    with pytest.raises(OSError, match="out.labels"):
        write_results(res, tmp_path / "missing_dir" / "out.labels")
