"""CPU: pin the oracle before trusting it.

* the plain-C restatement (oracle/liboracle.so) is bit-identical to the
  reference compiled from its own sources (oracle/_ref) on every backend;
* both reproduce the reference's frozen golden objectives
  (proj/tests/support/golden.hpp:10-17) and the committed golden fixtures
  (tests/golden/*.json, made by tests/golden/make_golden.py);
* the product's synthetic-input generators reproduce the reference's
  fixture generators (testgen.cpp) bit for bit, and SYNTH-v1 reproduces the
  reference objectives recorded in BASELINE.md §3.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT, rel_err
from paper_2008_03433_b200 import TrustRegionConfig, synth
from pyoracle import L2SVM, LOGISTIC

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def test_golden_objectives(port):
    p = synth.testgen_dense_problem(1001, 50, 5, 1.0)
    _, t = port.solve(p, LOGISTIC, TrustRegionConfig(eps=1e-8))
    assert t["converged"] and rel_err(t["objective"], 23.2600071465565482846) <= 1e-6
    for loss, seed, g in ((LOGISTIC, 2001, 84.0054573043513978445),
                          (L2SVM, 3001, 88.1453447856914700312)):
        p = synth.testgen_dense_problem(seed, 200, 20, 1.0)
        _, t = port.solve(p, loss, TrustRegionConfig(eps=1e-8, max_outer_iters=100))
        assert t["converged"] and rel_err(t["objective"], g) <= 1e-6


@pytest.mark.parametrize("loss", [LOGISTIC, L2SVM])
@pytest.mark.parametrize("precond", [False, True])
def test_port_bit_identical_to_reference(port, ref, loss, precond):
    p = synth.testgen_sparse_problem(3400, 400, 60, 2.0, 0.15)
    cfg = TrustRegionConfig(eps=1e-7, use_preconditioner=precond)
    w, t = port.solve(p, loss, cfg)
    for backend, workers in ((ref.SEQ, 1), (ref.PAR, 4), (ref.STAGED, 1), (ref.MIX, 4)):
        w2, t2 = ref.solve(p, loss, cfg, backend=backend, workers=workers)
        assert np.array_equal(w, w2) and t == t2


def test_port_kernels_bit_identical(port, ref):
    for seed in range(3):
        p = synth.testgen_dense_problem(300 + seed, 57, 13, 0.5 + seed)
        q = synth.testgen_sparse_problem(400 + seed, 61, 17, 1.5, 0.2)
        for prob in (p, q):
            w = synth.testgen_random_vector(10 + seed, prob.X.cols, 0.3)
            v = synth.testgen_random_vector(20 + seed, prob.X.cols)
            a, b = port.logistic(prob, w, v), ref.logistic(prob, w, v)
            for k in ("f", "z", "zhat", "dvec", "alpha", "g", "hv", "M"):
                assert np.array_equal(a[k], b[k]), k
            a, b = port.svm(prob, w, v), ref.svm(prob, w, v)
            for k in ("f", "z", "active", "g", "hv", "M"):
                assert np.array_equal(a[k], b[k]), k


def test_generators_match_reference_testgen(ref):
    vals, y = ref.dense_problem(1001, 50, 5)
    p = synth.testgen_dense_problem(1001, 50, 5, 1.0)
    assert np.array_equal(vals, p.X.values) and np.array_equal(y, p.y)
    vals, y = ref.dense_problem_scaled(117, 80, 8, 20.0)
    p = synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0)
    assert np.array_equal(vals, p.X.values) and np.array_equal(y, p.y)
    ro, ci, v, y = ref.sparse_problem(6000, 300, 500, 0.02)
    q = synth.testgen_sparse_problem(6000, 300, 500, 1.0, 0.02)
    assert np.array_equal(ro, q.X.row_offsets) and np.array_equal(ci, q.X.col_indices)
    assert np.array_equal(v, q.X.values) and np.array_equal(y, q.y)
    assert np.array_equal(ref.random_vector(5, 10, 0.7), synth.testgen_random_vector(5, 10, 0.7))
    assert np.array_equal(ref.random_index_set(3, 40, 0.2), synth.testgen_random_index_set(3, 40, 0.2))


def test_synth_r1_reference_objective(port):
    """SYNTH-v1 rcv1 shape: f and counts recorded from the reference."""
    p = synth.make_shape("R1")
    assert p.X.rows == 20242 and p.X.cols == 47236 and p.X.stored() == 20242 * 74
    w, t = port.solve(p, LOGISTIC, eps=0.01)
    assert t["objective"] == 1.097269983508039e04 or rel_err(t["objective"], 1.097269983508039e04) <= 1e-15
    its = t["iterations"]
    assert (len(its), t["accepted_steps"], sum(r["cg_iters"] for r in its)) == (3, 3, 16)


def _golden_files():
    return sorted(f for f in os.listdir(GOLDEN_DIR) if f.endswith(".json"))


@pytest.mark.parametrize("fname", _golden_files())
def test_port_matches_committed_golden(port, fname):
    g = json.load(open(os.path.join(GOLDEN_DIR, fname)))
    from golden.make_golden import build_problem  # noqa: E402
    p = build_problem(g["problem"])
    cfg = TrustRegionConfig(**g["config"])
    loss = LOGISTIC if g["loss"] == "logistic" else L2SVM
    w, t = port.solve(p, loss, cfg)
    assert t["objective"] == g["objective"]
    assert w.tolist() == g["w"]
    assert [(r["accepted"], r["cg_iters"], r["cg_exit"]) for r in t["iterations"]] == \
        [tuple(r) for r in g["iterations"]]
