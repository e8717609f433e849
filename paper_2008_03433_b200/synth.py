"""Deterministic synthetic inputs (native, in libtron_b200.so).

* ``testgen_*``: the reference's own fixture generators
  (proj/tests/support/testgen.cpp:24-90), bit-compatible.
* ``synth_sparse`` / ``synth_dense`` and the ``SHAPES`` table: SYNTH-v1, the
  frozen benchmark inputs of SURVEY.md §8(d) / BASELINE.json configs.
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import lib
from .tron import FeatureMatrix, Problem, _raise

PD = ctypes.POINTER(ctypes.c_double)
PI64 = ctypes.POINTER(ctypes.c_int64)
PI32 = ctypes.POINTER(ctypes.c_int32)


def _p(a, t):
    return a.ctypes.data_as(t)


def testgen_dense_problem(seed, l, n, C, flip=0.1) -> Problem:
    vals = np.empty(l * n)
    y = np.empty(l)
    lib.tron_testgen_dense_problem(seed, l, n, flip, _p(vals, PD), _p(y, PD))
    return Problem(FeatureMatrix.dense(l, n, vals), y, C)


def testgen_dense_problem_scaled(seed, l, n, C, scale, flip=0.02) -> Problem:
    vals = np.empty(l * n)
    y = np.empty(l)
    lib.tron_testgen_dense_problem_scaled(seed, l, n, scale, flip, _p(vals, PD), _p(y, PD))
    return Problem(FeatureMatrix.dense(l, n, vals), y, C)


def testgen_sparse_problem(seed, l, n, C, density=0.1, flip=0.1) -> Problem:
    nnz = lib.tron_testgen_sparse_problem(seed, l, n, density, flip, None, None, None, None)
    ro = np.empty(l + 1, dtype=np.int64)
    ci = np.empty(max(nnz, 1), dtype=np.int32)
    vals = np.empty(max(nnz, 1))
    y = np.empty(l)
    lib.tron_testgen_sparse_problem(seed, l, n, density, flip, _p(ro, PI64), _p(ci, PI32),
                                    _p(vals, PD), _p(y, PD))
    return Problem(FeatureMatrix.csr(l, n, ro, ci[:nnz], vals[:nnz]), y, C)


def testgen_random_vector(seed, n, span=1.0) -> np.ndarray:
    out = np.empty(n)
    lib.tron_testgen_random_vector(seed, n, span, _p(out, PD))
    return out


def testgen_random_index_set(seed, l, fraction) -> np.ndarray:
    cnt = lib.tron_testgen_random_index_set(seed, l, fraction, None)
    out = np.empty(max(cnt, 1), dtype=np.int64)
    lib.tron_testgen_random_index_set(seed, l, fraction, _p(out, PI64))
    return out[:cnt]


def synth_sparse(seed, l, n, k, s=1.0, flip=0.1, C=1.0) -> Problem:
    ro = np.empty(l + 1, dtype=np.int64)
    ci = np.empty(l * k, dtype=np.int32)
    vals = np.empty(l * k)
    y = np.empty(l)
    _raise(lib.tron_synth_sparse(seed, l, n, k, s, flip, _p(ro, PI64), _p(ci, PI32), _p(vals, PD),
                                 _p(y, PD)))
    return Problem(FeatureMatrix("csr", l, n, vals, ro, ci), y, C)


def synth_dense(seed, l, n=40, decades=2.0, rho=0.0, flip=0.1, C=1.0) -> Problem:
    vals = np.empty(l * n)
    y = np.empty(l)
    _raise(lib.tron_synth_dense(seed, l, n, decades, rho, flip, _p(vals, PD), _p(y, PD)))
    return Problem(FeatureMatrix("dense", l, n, vals), y, C)


# SYNTH-v1 shapes (BASELINE.json "configs")
SHAPES = {
    "R1": dict(kind="sparse", l=20242, n=47236, k=74, loss="logistic",
               desc="rcv1-shaped sparse LR 20,242x47,236, 74 nnz/row"),
    "N1": dict(kind="sparse", l=19996, n=1355191, k=455, loss="logistic",
               desc="news20-shaped sparse LR 19,996x1,355,191, 455 nnz/row"),
    "P1": dict(kind="dense", l=23_000_000, n=40, loss="l2svm",
               desc="proteomics-shaped dense L2-SVM 2.3e7x40"),
    "K1": dict(kind="sparse", l=8_400_000, n=20_000_000, k=36, loss="logistic",
               desc="kdd2010-shaped sparse LR 8.4e6x2.0e7, 36 nnz/row"),
    "Q1": dict(kind="dense", l=215_000_000, n=40, loss="l2svm",
               desc="quarter-billion dense L2-SVM 2.15e8x40"),
}


def make_shape(name, seed=1, rows=None) -> Problem:
    """SYNTH-v1 problem for a named shape (optionally with fewer rows)."""
    s = SHAPES[name]
    l = rows if rows is not None else s["l"]
    if s["kind"] == "sparse":
        return synth_sparse(seed, l, s["n"], s["k"])
    return synth_dense(seed, l, s["n"])
