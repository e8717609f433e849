"""GPU parity of the hot-path kernels (fun / grad / Hv / preconditioner / CG)
against the oracle, through the C ABI.  GPU twins of the reference KATs in
proj/tests/test_loss.cpp and test_linalg.cpp, plus random-fixture parity.

Tolerances: bit-exact where the reference's arithmetic order is reproduced
(dense margins z, hence the L2-SVM active set); otherwise FP64 rounding
level (<= 1e-12 relative, oracles::rel_err), since device reductions sum in
a different (fixed) order than the reference's 64-block tree.
"""
import math

import numpy as np
import pytest

from conftest import rel_err
from paper_2008_03433_b200 import (BoundsError, BudgetExceededError, DimensionError, ExecutionPlan,
                                   FeatureMatrix, LogicError, LossKind, Problem,
                                   StrategyPreconditionError, SvmStrategy, TrustRegionConfig,
                                   make_evaluator, solve, synth)
from paper_2008_03433_b200.tron import CgExit

pytestmark = pytest.mark.gpu

LR, SVM = LossKind.Logistic, LossKind.L2Svm


def gpu(problem, loss, **kw):
    return make_evaluator(problem, loss, ExecutionPlan.gpu(**kw))


def dense(rows, cols, vals, y, C=1.0):
    return Problem(FeatureMatrix.dense(rows, cols, vals), np.array(y, dtype=float), C)


# ---------------------------------------------------------------- KATs (test_loss.cpp)

def test_logistic_fused_pass_at_zero():  # test_loss.cpp:45-55
    p = synth.testgen_dense_problem(5, 4, 3, 1.0)
    with gpu(p, LR) as ev:
        f = ev.eval_candidate(np.zeros(3))
        assert rel_err(f, 4 * math.log(2.0)) <= 1e-14
        s = ev.candidate_state()
        assert np.all(s.z == 0.0)
        assert np.all(s.dvec == 0.25)
        assert np.array_equal(s.zhat, -p.y / 2.0)


def test_logistic_saturates_cleanly():  # test_loss.cpp:57-78
    p = dense(2, 1, [1000.0, 1000.0], [1.0, -1.0])
    with gpu(p, LR) as ev:
        f = ev.eval_candidate([2.0])
        s = ev.candidate_state()
        assert s.zhat[0] == 0.0 and s.dvec[0] == 0.0
        assert s.zhat[1] == 1.0 and s.dvec[1] == 0.0
        assert math.isfinite(f)
    q = dense(2, 1, [1000.0, 500.0], [1.0, 1.0])
    with gpu(q, LR) as ev:
        assert ev.eval_candidate([2.0]) == 0.5 * 4.0


def test_logistic_one_by_one():  # test_loss.cpp:80-91
    p = dense(1, 1, [1.0], [1.0], C=2.0)
    with gpu(p, LR) as ev:
        f = ev.eval_candidate([1.0])
        assert rel_err(f, 0.5 + 2.0 * math.log1p(math.exp(-1.0))) <= 1e-12
        ev.commit()
        g = ev.gradient()
        assert rel_err(g[0], 1.0 - 2.0 / (1.0 + math.exp(1.0))) <= 1e-12


def test_logistic_hessian_basics():  # test_loss.cpp:139-165
    p = synth.testgen_dense_problem(41, 6, 4, 2.0)
    w = synth.testgen_random_vector(42, 4)
    with gpu(p, LR) as ev:
        ev.eval_candidate(w)
        ev.commit()
        assert np.array_equal(ev.hessian_vec(np.zeros(4)), np.zeros(4))
    zero = dense(3, 2, [0.0] * 6, [1.0, -1.0, 1.0], C=5.0)
    with gpu(zero, LR) as ev:
        ev.eval_candidate([1.0, 2.0])
        ev.commit()
        assert np.array_equal(ev.hessian_vec([0.5, -0.25]), [0.5, -0.25])
    eye = dense(2, 2, [1.0, 0.0, 0.0, 1.0], [1.0, -1.0])
    with gpu(eye, LR) as ev:
        ev.eval_candidate([0.0, 0.0])
        ev.commit()
        out = ev.hessian_vec([1.0, 1.0])
        assert rel_err(out[0], 1.25) <= 1e-15 and rel_err(out[1], 1.25) <= 1e-15


def test_svm_active_set_kats():  # test_loss.cpp:167-209
    p = synth.testgen_dense_problem(51, 5, 3, 1.0)
    with gpu(p, SVM) as ev:
        assert ev.eval_candidate(np.zeros(3)) == 5.0
        assert ev.candidate_state().active.size == 5
    q = dense(3, 1, [1.0, 2.0, 1.0], [1.0, 1.0, -1.0], C=7.0)
    with gpu(q, SVM) as ev:
        ev.eval_candidate([1.0])
        assert list(ev.candidate_state().active) == [2]
    r = dense(3, 1, [1.0, 2.0, 1.0], [1.0, 1.0, 1.0], C=7.0)
    with gpu(r, SVM) as ev:
        assert ev.eval_candidate([1.0]) == 0.5
        assert ev.candidate_state().active.size == 0
    one = dense(1, 1, [1.0], [1.0])
    with gpu(one, SVM) as ev:
        ev.eval_candidate([1.0 - 1e-9])
        assert ev.candidate_state().active.size == 1
        ev.eval_candidate([1.0])
        assert ev.candidate_state().active.size == 0
        ev.eval_candidate([1.0 + 1e-9])
        assert ev.candidate_state().active.size == 0


def test_svm_gradient_and_hessian_kats():  # test_loss.cpp:211-259
    q = dense(1, 1, [1.0], [1.0], C=3.0)
    with gpu(q, SVM) as ev:
        ev.eval_candidate([2.0])
        ev.commit()
        assert np.array_equal(ev.gradient(), [2.0])  # empty active set
    r = dense(1, 1, [1.0], [1.0])
    with gpu(r, SVM) as ev:
        ev.eval_candidate([0.5])
        ev.commit()
        assert np.array_equal(ev.gradient(), [-0.5])
    # active = {0, 2} of a 3x2 problem, v = (1, 0) -> (5, 2)
    p = dense(3, 2, [1.0, 0.0, 0.0, 1.0, 1.0, 1.0], [1.0, 1.0, -1.0])
    with gpu(p, SVM) as ev:
        ev.eval_candidate([0.0, 0.0])  # all margins 1 -> I = {0,1,2}
        ev.commit()
        out = ev.hessian_vec([1.0, 0.0])
        assert np.array_equal(out, [1.0 + 2.0 * 2.0, 2.0 * 1.0])


def test_preconditioner_kats():  # test_loss.cpp:278-298
    zero = dense(2, 3, [0.0] * 6, [1.0, -1.0], C=4.0)
    with gpu(zero, LR) as ev:
        ev.eval_candidate(np.zeros(3))
        ev.commit()
        assert np.array_equal(ev.precond_diagonal(), np.ones(3))
    p = dense(1, 1, [2.0], [1.0])
    with gpu(p, LR) as ev:
        ev.eval_candidate([0.0])
        ev.commit()
        assert np.array_equal(ev.precond_diagonal(), [2.0])
    with gpu(p, SVM) as ev:
        ev.eval_candidate([0.0])
        ev.commit()
        assert np.array_equal(ev.precond_diagonal(), [1.0 + 2.0 * 4.0])


# ---------------------------------------------------------------- random-fixture parity

def _fixtures():
    out = []
    for seed in range(3):
        out.append(("dense", synth.testgen_dense_problem(300 + seed, 257, 13, 0.5 + seed)))
        out.append(("sparse", synth.testgen_sparse_problem(400 + seed, 611, 97, 1.5, 0.08)))
    out.append(("dense40", synth.synth_dense(7, 3001, 40)))
    out.append(("synth", synth.synth_sparse(9, 2000, 5000, 37)))
    out.append(("wide", synth.testgen_dense_problem(77, 50, 70, 1.0)))  # n > 64: CSR path
    return out


@pytest.mark.parametrize("case", range(9))
@pytest.mark.parametrize("loss", [LR, SVM])
def test_fun_grad_hv_precond_parity(port, case, loss):
    name, p = _fixtures()[case]
    n = p.X.cols
    w = synth.testgen_random_vector(1000 + case, n, 0.3)
    v = synth.testgen_random_vector(2000 + case, n, 1.0)
    want = port.logistic(p, w, v) if loss == LR else port.svm(p, w, v)
    with gpu(p, loss) as ev:
        f = ev.eval_candidate(w)
        assert rel_err(f, want["f"]) <= 1e-13, name
        s = ev.candidate_state()
        if p.X.layout == "dense" and n <= 64:
            assert np.array_equal(s.z, want["z"]), "dense margins must be bit-exact"
        else:
            assert rel_err(s.z, want["z"]) <= 1e-14
        if loss == SVM:
            assert np.array_equal(s.active, want["active"]), "active set must be identical"
        else:
            assert rel_err(s.zhat, want["zhat"]) <= 1e-13
            assert rel_err(s.dvec, want["dvec"]) <= 1e-13
        gn = ev.commit()
        g = ev.gradient()
        assert rel_err(g, want["g"]) <= 1e-12, name
        assert rel_err(gn, np.linalg.norm(want["g"])) <= 1e-12
        assert rel_err(ev.hessian_vec(v), want["hv"]) <= 1e-12, name
        assert rel_err(ev.precond_diagonal(), want["M"]) <= 1e-12, name
        # committed state is the candidate we evaluated
        cs = ev.committed_state()
        assert rel_err(cs.z, want["z"]) <= 1e-14


def test_csc_transposed_product_zipf_columns(port):
    # Zipf-hot columns span many merge-path tiles; empty columns must emit w_j.
    p = synth.synth_sparse(3, 6000, 20000, 12)
    w = np.zeros(p.X.cols)
    want = port.logistic(p, w)
    with gpu(p, LR) as ev:
        ev.eval_candidate(w)
        ev.commit()
        g = ev.gradient()
    assert rel_err(g, want["g"]) <= 1e-12
    cols_used = np.zeros(p.X.cols, bool)
    cols_used[p.X.col_indices] = True
    assert np.all(g[~cols_used] == 0.0)


def test_gradient_deterministic_across_runs():
    p = synth.synth_sparse(5, 3000, 8000, 20)
    w = synth.testgen_random_vector(6, p.X.cols, 0.1)
    outs = []
    for _ in range(2):
        with gpu(p, LR) as ev:
            ev.eval_candidate(w)
            ev.commit()
            outs.append((ev.gradient(), ev.hessian_vec(w), ev.precond_diagonal()))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- device CG

@pytest.mark.parametrize("case", [0, 1, 6, 7])
@pytest.mark.parametrize("precond", [False, True])
def test_device_cg_matches_host_cg(port, case, precond):
    name, p = _fixtures()[case]
    n = p.X.cols
    w = synth.testgen_random_vector(3000 + case, n, 0.3)
    with gpu(p, LR) as ev:
        ev.eval_candidate(w)
        ev.commit()
        g = ev.gradient()
        M = ev.precond_diagonal() if precond else None
        # SYNTH dense (2-decade column scales) is ill-conditioned: beyond ~12 CG
        # iterations rounding differences grow ~10x per iteration in any two
        # FP64 implementations, so that case runs at TRON's own cg_tol (0.1).
        cg_tol = 0.1 if name == "dense40" else 1e-6
        # d: the two CGs share Hv but not the order of their dot products; at
        # cg_tol 1e-6 (~25 iterations) that difference grows to ~1e-10
        for delta, tol in ((1e6, 1e-9), (0.5 * np.linalg.norm(g), 1e-9), (1e-3, 1e-9)):
            cfg = TrustRegionConfig(cg_tol=cg_tol, use_preconditioner=precond)
            dev = ev.truncated_cg(delta, cfg)
            host = port.truncated_cg(g, ev.hessian_vec, delta, M, cg_tol=cg_tol)
            assert dev.iters == host["iters"], name
            assert int(dev.exit) == host["exit"], name
            assert rel_err(dev.d, host["d"]) <= tol, name
            assert rel_err(dev.model_value, host["model_value"]) <= 1e-9, name
            assert np.linalg.norm(dev.d) <= delta * (1 + 1e-12)


# the CG engines on the same mid-size problem: single cluster kernel per step
# (default for 4096 < n <= 32768), the cooperative large-n step (default above),
# and the host-driven loop (no graph), each against the host restatement
@pytest.mark.parametrize("engine", ["cluster", "coop", "nograph"])
@pytest.mark.parametrize("precond", [False, True])
def test_cg_engines_match_host_cg(port, monkeypatch, engine, precond):
    if engine == "coop":
        monkeypatch.setenv("TRON_B200_CLUSTER_CG", "0")
    if engine == "nograph":
        monkeypatch.setenv("TRON_B200_NO_GRAPH", "1")
    p = synth.synth_sparse(9, 2000, 5000, 37)  # n = 5000 > kSmallCgMaxN
    w = synth.testgen_random_vector(3007, p.X.cols, 0.3)  # the state of fixture case 7 above
    with gpu(p, LR) as ev:
        ev.eval_candidate(w)
        ev.commit()
        g = ev.gradient()
        M = ev.precond_diagonal() if precond else None
        for delta in (1e6, 0.5 * np.linalg.norm(g), 1e-3):
            cfg = TrustRegionConfig(cg_tol=1e-6, use_preconditioner=precond)
            dev = ev.truncated_cg(delta, cfg)
            host = port.truncated_cg(g, ev.hessian_vec, delta, M, cg_tol=1e-6)
            assert dev.iters == host["iters"]
            assert int(dev.exit) == host["exit"]
            # shared Hv, different dot-product order: ~2e-10 after ~20 iterations
            assert rel_err(dev.d, host["d"]) <= 1e-9
            assert rel_err(dev.model_value, host["model_value"]) <= 1e-9
        # the iteration cap ends the loop on the device (exit MaxIters)
        cfg = TrustRegionConfig(cg_tol=1e-9, max_cg_iters=2, use_preconditioner=precond)
        dev = ev.truncated_cg(1e6, cfg)
        host = port.truncated_cg(g, ev.hessian_vec, 1e6, M, cg_tol=1e-9, max_cg_iters=2)
        assert dev.iters == host["iters"] == 2 and int(dev.exit) == host["exit"]
        assert rel_err(dev.d, host["d"]) <= 1e-10


def test_device_cg_iteration_cap():  # test_tron.cpp:75-90
    p = synth.testgen_dense_problem(1100, 30, 6, 1.0)
    w = synth.testgen_random_vector(1101, 6)
    with gpu(p, LR) as ev:
        ev.eval_candidate(w)
        ev.commit()
        res = ev.truncated_cg(1e6, TrustRegionConfig(max_cg_iters=1, cg_tol=1e-10))
        assert res.iters == 1 and res.exit == CgExit.MaxIters and res.model_value < 0.0


# ---------------------------------------------------------------- errors (error.hpp)

def test_validation_errors():
    with pytest.raises(DimensionError):
        gpu(dense(2, 1, [1.0, 2.0], [1.0, 3.0]), LR)
    with pytest.raises(DimensionError):
        gpu(dense(2, 1, [1.0, 2.0], [1.0, -1.0], C=0.0), LR)
    bad_col = Problem(FeatureMatrix("csr", 1, 2, np.array([1.0]), np.array([0, 1], np.int64),
                                    np.array([5], np.int32)), np.array([1.0]))
    with pytest.raises(BoundsError):
        gpu(bad_col, LR)
    unsorted = Problem(FeatureMatrix("csr", 1, 2, np.array([1.0, 2.0]), np.array([0, 2], np.int64),
                                     np.array([1, 0], np.int32)), np.array([1.0]))
    with pytest.raises(DimensionError):
        gpu(unsorted, LR)


def test_evaluator_misuse():  # test_backend.cpp:95-102
    p = synth.testgen_dense_problem(2030, 10, 3, 1.0)
    with gpu(p, LR) as ev:
        with pytest.raises(LogicError):
            ev.commit()
        with pytest.raises(LogicError):
            ev.hessian_vec([1.0, 2.0, 3.0])


def test_gathered_budget_names_mix():  # test_backend.cpp:104-139
    n = 18
    p = synth.testgen_dense_problem(3100, 10000, n, 1.0)
    with gpu(p, SVM, svm_strategy=SvmStrategy.Gathered, gathered_budget_bytes=1 << 20) as ev:
        ev.eval_candidate(np.zeros(n))
        with pytest.raises(BudgetExceededError) as e:
            ev.commit()
        assert "MixedActiveSet" in str(e.value)
    for l in (100, 1000, 10000):
        p = synth.testgen_dense_problem(3000 + l, l, n, 1.0)
        plan = ExecutionPlan.gpu(svm_strategy=SvmStrategy.Gathered)
        with make_evaluator(p, SVM, plan) as ev:
            ev.eval_candidate(np.zeros(n))
            ev.commit()
            lg = ev.ledger()
            assert lg.gathered_submatrix_bytes == l * n * 8
            assert lg.index_set_bytes == l * 8


def test_gathered_equals_indirect(port):
    p = synth.testgen_dense_problem(71, 4000, 6, 1.5)
    w = synth.testgen_random_vector(72, 6, 0.5)
    outs = []
    for strat in (SvmStrategy.Gathered, SvmStrategy.Indirect):
        with gpu(p, SVM, svm_strategy=strat) as ev:
            ev.eval_candidate(w)
            ev.commit()
            outs.append([ev.hessian_vec(synth.testgen_random_vector(90 + k, 6)) for k in range(5)])
    for a, b in zip(*outs):
        assert rel_err(a, b) <= 1e-12


# Gathered L2-SVM on CSR features (gather_rows' CSR branch, linalg.cpp:212-228):
# X_I and its CSC copy are rebuilt at every commit; Hv over them equals the
# masked traversal and the reference evaluator, and the budget check uses the
# reference's projected_gather_bytes (backend.cpp:47-54).
@pytest.mark.parametrize("strategy", [SvmStrategy.Gathered, SvmStrategy.Auto])
def test_gathered_csr_equals_indirect_and_reference(port, strategy):
    p = synth.synth_sparse(5, 3000, 8000, 40)
    n = p.X.cols
    w = synth.testgen_random_vector(61, n, 2.0)
    want = port.svm(p, w, None)
    outs = {}
    for strat in (strategy, SvmStrategy.Indirect):
        with gpu(p, SVM, svm_strategy=strat) as ev:
            ev.eval_candidate(w)
            ev.commit()
            assert rel_err(ev.gradient(), want["g"]) <= 1e-12
            vs = [synth.testgen_random_vector(300 + k, n) for k in range(4)]
            outs[strat] = [ev.hessian_vec(v) for v in vs]
            if strat == SvmStrategy.Gathered:
                nnz_I = int(sum(p.X.row_offsets[i + 1] - p.X.row_offsets[i] for i in want["active"]))
                assert ev.ledger().gathered_submatrix_bytes == nnz_I * 12 + (want["active"].size + 1) * 8
    for k, (a, b) in enumerate(zip(outs[strategy], outs[SvmStrategy.Indirect])):
        ref_hv = port.svm(p, w, synth.testgen_random_vector(300 + k, n))["hv"]
        assert rel_err(a, b) <= 1e-13 and rel_err(a, ref_hv) <= 1e-12


def test_gathered_csr_budget_names_mix():
    p = synth.synth_sparse(5, 3000, 8000, 40)
    with gpu(p, SVM, svm_strategy=SvmStrategy.Gathered, gathered_budget_bytes=1 << 16) as ev:
        ev.eval_candidate(np.zeros(p.X.cols))
        with pytest.raises(BudgetExceededError) as e:
            ev.commit()
        assert "MixedActiveSet" in str(e.value)
    # Auto never raises: over budget it stays on the masked traversal
    with gpu(p, SVM, svm_strategy=SvmStrategy.Auto, gathered_budget_bytes=1 << 16) as ev:
        ev.eval_candidate(np.zeros(p.X.cols))
        ev.commit()
        assert ev.ledger().gathered_submatrix_bytes == 0


@pytest.mark.parametrize("case", range(3))
def test_device_quadratic_model(port, case):
    """tron_gpu_quadratic_model (tron.cpp:31-35) at the committed iterate against
    the oracle's g.d + 0.5 d.Hd; and the CG's residual identity (tron.cpp:106):
    the CG result's model value is q(d) of its own step."""
    from paper_2008_03433_b200 import quadratic_model
    probs = [(synth.synth_sparse(3, 800, 20000, 30), LossKind.Logistic, 0),
             (synth.synth_dense(2, 3000, 40), LossKind.L2Svm, 1),
             (synth.synth_sparse(6, 700, 5000, 25), LossKind.L2Svm, 1)]
    p, loss, ol = probs[case]
    n = p.X.cols
    w = synth.testgen_random_vector(11, n, 0.05)
    d = synth.testgen_random_vector(12, n, 1.0)
    with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
        ev.eval_candidate(w)
        ev.commit()
        q = ev.quadratic_model(d)
        q_host = quadratic_model(ev.gradient(), ev.hessian_vec, d)
        cg = ev.truncated_cg(np.linalg.norm(ev.gradient()), TrustRegionConfig(eps=0.01))
        q_step = ev.quadratic_model(cg.d)
    want = port.logistic(p, w, d) if ol == 0 else port.svm(p, w, d)
    q_ref = float(want["g"] @ d + 0.5 * d @ want["hv"])
    assert abs(q - q_ref) <= 1e-11 * abs(q_ref)
    assert abs(q - q_host) <= 1e-12 * abs(q_ref)
    assert abs(q_step - cg.model_value) <= 1e-9 * abs(cg.model_value)


@pytest.mark.parametrize("hot_rows", [140_000, 400_000])
def test_csc_long_fixup_spans(port, hot_rows):
    """Columns spanning more than kFixCta = 512 chunks (131k+ entries, like K1's
    Zipf-hot columns) are finished by a CTA of their own: gradient, Hv (with
    the fused p.Hp of the solve) and the preconditioner against the oracle,
    bit-reproducible run to run."""
    rng = np.random.default_rng(7)
    l, n = hot_rows, 3000
    hot = [0, 1, 17]  # three columns present in (almost) every row
    rows_cols = []
    for i in range(l):
        cols = set(hot[:2] if i % 3 else hot)
        cols.update(rng.integers(18, n, size=3).tolist())
        rows_cols.append(sorted(cols))
    ro = np.zeros(l + 1, np.int64)
    ro[1:] = np.cumsum([len(c) for c in rows_cols])
    ci = np.concatenate([np.array(c, np.int32) for c in rows_cols])
    vals = rng.uniform(0.01, 1.0, ci.size)
    y = np.where(rng.random(l) < 0.5, -1.0, 1.0)
    p = Problem(FeatureMatrix("csr", l, n, vals, ro, ci), y, 1.0)
    w = rng.uniform(-0.01, 0.01, n)
    v = rng.uniform(-1, 1, n)
    want = port.logistic(p, w, v)
    outs = []
    for _ in range(2):
        with gpu(p, LR) as ev:
            ev.eval_candidate(w)
            ev.commit()
            outs.append((ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()))
    g, hv, m = outs[0]
    assert rel_err(g, want["g"]) <= 1e-12
    assert rel_err(hv, want["hv"]) <= 1e-12
    assert rel_err(m, want["M"]) <= 1e-12
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    r = solve(p, LR, TrustRegionConfig(eps=1e-3), ExecutionPlan.gpu())
    w_ref, t_ref = port.solve(p, 0, TrustRegionConfig(eps=1e-3))
    assert rel_err(r.objective, t_ref["objective"]) <= 1e-10 and rel_err(r.w, w_ref) <= 1e-7


@pytest.mark.parametrize("width", [1000, 4096, 30000])
def test_column_panels_row_products(port, monkeypatch, width):
    """Column panels of the row products (opt-in TRON_B200_PANEL_COLS): fun /
    grad / Hv of LR and of the sparse L2-SVM against the oracle, and whole
    solves against the unpaneled ones."""
    monkeypatch.setenv("TRON_B200_PANEL_COLS", str(width))
    p = synth.synth_sparse(13, 3000, 40000, 30)
    n = p.X.cols
    w = synth.testgen_random_vector(21, n, 0.05)
    v = synth.testgen_random_vector(22, n, 1.0)
    for loss, ol in ((LR, 0), (SVM, 1)):
        want = port.logistic(p, w, v) if ol == 0 else port.svm(p, w, v)
        with gpu(p, loss) as ev:
            f = ev.eval_candidate(w)
            st = ev.candidate_state()
            ev.commit()
            g, hv = ev.gradient(), ev.hessian_vec(v)
            r = ev.solve(TrustRegionConfig(eps=1e-6))
        assert rel_err(f, want["f"]) <= 1e-13
        assert rel_err(st.z, want["z"]) <= 1e-13
        assert rel_err(g, want["g"]) <= 1e-12 and rel_err(hv, want["hv"]) <= 1e-12
        monkeypatch.setenv("TRON_B200_PANEL_COLS", "0")
        r0 = solve(p, loss, TrustRegionConfig(eps=1e-6), ExecutionPlan.gpu())
        monkeypatch.setenv("TRON_B200_PANEL_COLS", str(width))
        # whole solves near the optimum (at loose eps the two summation splits
        # may stop at different iterations of the same path)
        assert rel_err(r.objective, r0.objective) <= 1e-10 and rel_err(r.w, r0.w) <= 1e-5
