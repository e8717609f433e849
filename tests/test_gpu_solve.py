"""End-to-end TRON solves on the GPU vs the reference CPU solver on the same
inputs (BASELINE.json parity gate): objective and w within 1e-6 relative,
outer/accepted/CG iteration counts identical or within +-1, L2-SVM active
set and test predictions identical.  Also the reference's solver-level
properties (proj/tests/test_tron.cpp, test_backend.cpp) on the GPU backend.
"""
import math

import numpy as np
import pytest

from conftest import rel_err
from paper_2008_03433_b200 import (ExecutionPlan, FeatureMatrix, LossKind, NumericalFailureError,
                                   Problem, SvmStrategy, TrustRegionConfig, make_evaluator, solve,
                                   synth)

pytestmark = pytest.mark.gpu

LR, SVM = LossKind.Logistic, LossKind.L2Svm
GOLDEN = {  # proj/tests/support/golden.hpp:10-17
    "lr50x5": 23.2600071465565482846,
    "lr200x20": 84.0054573043513978445,
    "svm200x20": 88.1453447856914700312,
}


def plan(**kw):
    return ExecutionPlan.gpu(**kw)


def counts(trace):
    its = trace.iterations if hasattr(trace, "iterations") else trace["iterations"]
    if its and isinstance(its[0], dict):
        return len(its), sum(r["accepted"] for r in its), sum(r["cg_iters"] for r in its)
    return len(its), sum(r.accepted for r in its), sum(r.cg_iters for r in its)


def predict(X, w):  # model.cpp:88-117: sign(x.w), ties -> +1
    scores = X.to_dense() @ w if X.layout == "csr" else X.values.reshape(X.rows, X.cols) @ w
    return np.where(scores < 0.0, -1.0, 1.0)


def assert_parity(res, w_ref, t_ref, X=None, tol=1e-6):
    assert rel_err(res.objective, t_ref["objective"]) <= tol
    assert rel_err(res.w, w_ref) <= tol
    o, a, c = counts(res.trace)
    o2, a2, c2 = counts(t_ref)
    assert abs(o - o2) <= 1 and abs(a - a2) <= 1 and abs(c - c2) <= 1, ((o, a, c), (o2, a2, c2))
    assert res.converged == t_ref["converged"]
    if X is not None:
        assert np.array_equal(predict(X, res.w), predict(X, w_ref))


@pytest.mark.parametrize("mode", ["device", "host_cg"])
def test_golden_objectives(mode):  # test_tron.cpp:199-207, acceptance criterion 3
    p = synth.testgen_dense_problem(1001, 50, 5, 1.0)
    r = solve(p, LR, TrustRegionConfig(eps=1e-8), plan(solve_mode=mode))
    assert r.converged and rel_err(r.objective, GOLDEN["lr50x5"]) <= 1e-6
    for loss, seed, key in ((LR, 2001, "lr200x20"), (SVM, 3001, "svm200x20")):
        p = synth.testgen_dense_problem(seed, 200, 20, 1.0)
        r = solve(p, loss, TrustRegionConfig(eps=1e-8, max_outer_iters=100), plan(solve_mode=mode))
        assert r.converged and rel_err(r.objective, GOLDEN[key]) <= 1e-6


CASES = [
    ("dense-lr", lambda: synth.testgen_dense_problem(1300, 60, 8, 4.0), LR, 1e-6),
    ("dense-svm", lambda: synth.testgen_dense_problem(1300, 60, 8, 4.0), SVM, 1e-6),
    ("sparse-lr", lambda: synth.testgen_sparse_problem(3400, 400, 60, 2.0, 0.15), LR, 1e-7),
    ("sparse-svm", lambda: synth.testgen_sparse_problem(3400, 400, 60, 2.0, 0.15), SVM, 1e-7),
    ("crit4-lr", lambda: synth.testgen_sparse_problem(6000, 10000, 500, 1.0, 0.02), LR, 1e-4),
    ("crit4-svm", lambda: synth.testgen_dense_problem(6001, 10000, 18, 1.0), SVM, 1e-4),
    ("scaled-lr", lambda: synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0), LR, 1e-6),
    ("scaled-svm", lambda: synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0), SVM, 1e-6),
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("mode", ["device", "host_cg"])
def test_solve_parity_vs_reference(ref, case, precond, mode):
    name, mk, loss, eps = CASES[case]
    p = mk()
    cfg = TrustRegionConfig(eps=eps, use_preconditioner=precond)
    w_ref, t_ref = ref.solve(p, 0 if loss == LR else 1, cfg)
    r = solve(p, loss, cfg, plan(solve_mode=mode))
    assert_parity(r, w_ref, t_ref, X=p.X)
    # lazy-gradient contract (acceptance criterion 6)
    assert r.trace.gradient_materializations == r.trace.accepted_steps + 1
    assert r.trace.objective_evaluations == len(r.trace.iterations) + 1
    if loss == SVM:
        with make_evaluator(p, SVM, plan()) as ev:
            ev.eval_candidate(r.w)
            got = ev.candidate_state().active
        want = ref.svm(p, w_ref, np.zeros(p.X.cols))["active"]
        assert np.array_equal(got, want)


def test_synth_r1_full_size(ref):
    """rcv1-shaped SYNTH-v1 (BASELINE.json configs[0]) at full size."""
    p = synth.make_shape("R1")
    cfg = TrustRegionConfig(eps=0.01)
    w_ref, t_ref = ref.solve(p, 0, cfg, backend=1, workers=8)
    assert rel_err(t_ref["objective"], 1.097269983508039e04) <= 1e-15
    r = solve(p, LR, cfg, plan())
    assert_parity(r, w_ref, t_ref)
    assert counts(r.trace) == counts(t_ref)


def test_synth_n1_full_size_evaluator(ref):
    """news20-shaped SYNTH-v1 (configs[1], the bench's default) at full size:
    f, gradient, Hv and the preconditioner diagonal against the reference
    evaluator on the same inputs -- the staged segmented CSC product, its
    empty-column list and the fix-ups of Zipf-hot columns spanning hundreds of
    chunks, the vectorised row products."""
    p = synth.make_shape("N1")
    n = p.X.cols
    w = synth.testgen_random_vector(41, n, 0.01)
    v = synth.testgen_random_vector(42, n, 1.0)
    want = ref.logistic(p, w, v)
    with make_evaluator(p, LR, plan()) as ev:
        f = ev.eval_candidate(w)
        ev.commit()
        g, hv, M = ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()
    assert rel_err(f, want["f"]) <= 1e-13
    assert rel_err(g, want["g"]) <= 1e-12
    assert rel_err(hv, want["hv"]) <= 1e-12
    assert rel_err(M, want["M"]) <= 1e-12
    cols_used = np.zeros(n, bool)
    cols_used[p.X.col_indices] = True
    assert np.array_equal(hv[~cols_used], v[~cols_used])  # empty columns: v + C*0


@pytest.mark.parametrize("loss,precond", [(0, False), (1, False), (1, True)])
def test_large_n_sparse_solve_cooperative_engine(ref, loss, precond):
    """n > 32768 runs the cooperative CG step (one grid kernel per
    iteration, p.Hp from the Hv emission) and the emission-fused gradient
    norm: sparse LR and sparse L2-SVM (indirect strategy), with and without
    the preconditioner, against the reference solver."""
    # At eps = 0.01 this problem's sparse SVM trajectory is sensitive: CG counts
    # of 12/13/14 in the first outer iteration, from different FP64 summation
    # orders alone, give w 3e-4 .. 1e-2 apart with objectives 2e-7 apart.  So
    # both solvers run to eps = 1e-6 here and must meet at the same optimum.
    p = synth.synth_sparse(11, 6000, 300_000, 30)
    cfg = TrustRegionConfig(eps=1e-6, use_preconditioner=precond)
    w_ref, t_ref = ref.solve(p, loss, cfg, backend=1, workers=8)
    kind = LR if loss == 0 else SVM
    r = solve(p, kind, cfg, plan(svm_strategy=SvmStrategy.Indirect) if loss else plan())
    assert r.converged and t_ref["converged"]
    assert rel_err(r.objective, t_ref["objective"]) <= 1e-10
    assert rel_err(r.w, w_ref) <= 1e-5


@pytest.mark.parametrize("nccl_graph", ["0", "1"])
def test_large_n_sharded_path_single_rank_nccl(ref, monkeypatch, nccl_graph):
    """The row-sharded path (one NCCL rank) on the cooperative CG engine:
    allreduced raw products, then the epilogue, with the CG loop host-driven
    or captured in the graph together with the allreduces."""
    monkeypatch.setenv("TRON_B200_FORCE_NCCL", "1")
    monkeypatch.setenv("TRON_B200_NCCL_GRAPH", nccl_graph)
    p = synth.synth_sparse(12, 6000, 300_000, 30)
    cfg = TrustRegionConfig(eps=1e-6)
    w_ref, t_ref = ref.solve(p, 0, cfg, backend=1, workers=8)
    r = solve(p, LR, cfg, plan())
    assert r.converged and t_ref["converged"]
    assert rel_err(r.objective, t_ref["objective"]) <= 1e-10
    assert rel_err(r.w, w_ref) <= 1e-5


def test_synth_p1_reduced_rows_active_set(ref):
    """proteomics-shaped dense L2-SVM (configs[2]) at 2e5 rows: active set + predictions."""
    p = synth.synth_dense(1, 200_000, 40)
    cfg = TrustRegionConfig(eps=0.01)
    w_ref, t_ref = ref.solve(p, 1, cfg, backend=1, workers=8)
    r = solve(p, SVM, cfg, plan())
    assert_parity(r, w_ref, t_ref, X=p.X)
    with make_evaluator(p, SVM, plan()) as ev:
        ev.eval_candidate(w_ref)  # same w: the active set must be bit-identical
        got = ev.candidate_state().active
    want = ref.svm(p, w_ref, np.zeros(40))["active"]
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- solver properties

def test_stationary_start_and_quadratic():  # test_tron.cpp:159-197
    l, n = 4, 3
    y = np.ones(l)
    y[0::2] = -1.0
    p = Problem(FeatureMatrix.dense(l, n, np.zeros(l * n)), y, 1.0)
    r = solve(p, LR, TrustRegionConfig(), plan())
    assert r.converged and not r.trace.iterations
    assert rel_err(r.objective, 4 * math.log(2.0)) <= 1e-14
    q = Problem(FeatureMatrix.dense(3, 4, np.zeros(12)), np.array([-1.0, 1.0, -1.0]), 2.0)
    r = solve(q, LR, TrustRegionConfig(eps=1e-12), plan(), warm_start=[1.0, -2.0, 0.5, 3.0])
    assert r.converged and len(r.trace.iterations) == 1
    assert r.trace.iterations[0].accepted
    assert abs(r.trace.iterations[0].sigma - 1.0) <= 1e-12
    assert np.linalg.norm(r.w) <= 1e-12


def test_symmetric_two_point():  # test_tron.cpp:171-182
    p = Problem(FeatureMatrix.dense(2, 1, [1.0, 1.0]), np.array([1.0, -1.0]), 1.0)
    r = solve(p, LR, TrustRegionConfig(eps=1e-10), plan())
    assert r.converged and abs(r.w[0]) <= 1e-10


def test_descent_and_stopping_rule():  # test_tron.cpp:209-236
    for loss in (LR, SVM):
        p = synth.testgen_dense_problem(1300, 60, 8, 4.0)
        cfg = TrustRegionConfig(eps=1e-6)
        pl = plan()
        r = solve(p, loss, cfg, pl)
        assert r.converged
        last = r.trace.f_initial
        for rec in r.trace.iterations:
            if rec.accepted:
                assert rec.f_candidate < last
                last = rec.f_candidate
        assert pl.ledger.gradient_materializations == r.trace.accepted_steps + 1
        with make_evaluator(p, loss, plan()) as ev:
            ev.eval_candidate(r.w)
            ev.commit()
            assert np.linalg.norm(ev.gradient()) <= cfg.eps * r.trace.gradient_norm_initial * (1 + 1e-12)


def test_determinism():  # test_tron.cpp:264-274
    p = synth.testgen_sparse_problem(1500, 120, 30, 2.0, 0.2)
    cfg = TrustRegionConfig(eps=1e-7)
    a = solve(p, SVM, cfg, plan())
    b = solve(p, SVM, cfg, plan())
    assert a.trace == b.trace and np.array_equal(a.w, b.w)


def test_preconditioning_neutrality():  # test_tron.cpp:276-290
    for loss in (LR, SVM):
        p = synth.testgen_dense_problem(1600, 80, 10, 2.0)
        off = solve(p, loss, TrustRegionConfig(eps=1e-8), plan())
        on = solve(p, loss, TrustRegionConfig(eps=1e-8, use_preconditioner=True), plan())
        assert off.converged and on.converged
        assert rel_err(on.objective, off.objective) <= 1e-8


@pytest.mark.parametrize("mode", ["device", "host_cg"])
def test_nonfinite_objective_aborts(mode):  # test_tron.cpp:292-304
    p = synth.testgen_dense_problem(1700, 10, 3, 1.0)
    with pytest.raises(NumericalFailureError) as e:
        solve(p, LR, TrustRegionConfig(), plan(solve_mode=mode), warm_start=[1e200] * 3)
    assert e.value.trace.objective_evaluations == 1


def test_outer_cap():  # test_tron.cpp:306-315
    p = synth.testgen_dense_problem(1800, 60, 8, 50.0)
    r = solve(p, LR, TrustRegionConfig(eps=1e-14, max_outer_iters=2), plan())
    assert not r.converged and len(r.trace.iterations) == 2


def test_gathered_vs_indirect_solve():  # test_backend.cpp:245-257
    p = synth.testgen_dense_problem(3500, 200, 18, 1.0)
    cfg = TrustRegionConfig(eps=1e-8)
    pg = plan(svm_strategy=SvmStrategy.Gathered)
    a = solve(p, SVM, cfg, pg)
    b = solve(p, SVM, cfg, plan(svm_strategy=SvmStrategy.Indirect))
    assert rel_err(a.w, b.w) <= 1e-10 and rel_err(a.objective, b.objective) <= 1e-10
    assert pg.ledger.gathered_submatrix_bytes > 0


@pytest.mark.parametrize("strategy", [SvmStrategy.Gathered, SvmStrategy.Auto])
@pytest.mark.parametrize("mode", ["device", "host_cg"])
def test_gathered_csr_solve_matches_reference(ref, strategy, mode):
    # sparse L2-SVM, Gathered on CSR: the device CG runs over X_I (graph rebuilt
    # per commit); same optimum and counts as Indirect and the reference
    p = synth.synth_sparse(3, 20000, 30000, 30)
    cfg = TrustRegionConfig(eps=1e-3)
    pg = plan(svm_strategy=strategy, solve_mode=mode)
    a = solve(p, SVM, cfg, pg)
    b = solve(p, SVM, cfg, plan(svm_strategy=SvmStrategy.Indirect, solve_mode=mode))
    w_ref, t_ref = ref.solve(p, 1, cfg)
    assert_parity(a, w_ref, t_ref, X=p.X)
    assert rel_err(a.w, b.w) <= 1e-8  # X_I vs masked X: different FP64 summation orders
    if strategy == SvmStrategy.Gathered:
        assert pg.ledger.gathered_submatrix_bytes > 0


def test_host_cg_ledger_schedule():  # test_backend.cpp:152-184 (staged semantics)
    p = synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0)
    pl = plan(solve_mode="host_cg")
    r = solve(p, LR, TrustRegionConfig(eps=1e-6), pl)
    assert pl.ledger.scalar_returns == r.trace.objective_evaluations
    assert pl.ledger.margin_passes == r.trace.objective_evaluations
    assert pl.ledger.bulk_handoffs == r.trace.accepted_steps + 1
    assert any(not it.accepted for it in r.trace.iterations)


# The sharded (multi-GPU) code path on one GPU: a real one-rank NCCL
# communicator (TRON_B200_FORCE_NCCL=1) routes every partial through
# ncclAllReduce on the solver stream, the epilogues through the raw + vector
# epilogue kernels and CG through the host-driven loop.  Against the
# host-driven single-GPU path (same kernels, same order) it must be
# bit-identical; against the reference, within tolerance.  (The graph path
# finishes the dense Hv partials in another order; on SYNTH dense SVM the
# third CG run is chaotic in the last bit -- the reference itself goes
# [4, 9, 23] -> [4, 9, 19] -> [4, 9, 18] CG steps for C -> C(1+ulp) -> C(1+2ulp).)
@pytest.mark.parametrize("case", ["sparse_lr", "dense_svm", "dense_lr"])
def test_sharded_path_single_rank_nccl(ref, monkeypatch, case):
    p, loss = {
        "sparse_lr": (synth.synth_sparse(9, 2000, 5000, 37), LossKind.Logistic),
        "dense_svm": (synth.testgen_dense_problem(3001, 200, 20, 1.0), LossKind.L2Svm),
        "dense_lr": (synth.testgen_dense_problem(2001, 200, 20, 1.0), LossKind.Logistic),
    }[case]
    cfg = TrustRegionConfig(eps=0.01)
    monkeypatch.setenv("TRON_B200_NO_GRAPH", "1")
    base = solve(p, loss, cfg, ExecutionPlan.gpu())
    monkeypatch.delenv("TRON_B200_NO_GRAPH")
    monkeypatch.setenv("TRON_B200_FORCE_NCCL", "1")
    monkeypatch.setenv("TRON_B200_NCCL_GRAPH", "0")  # host-driven CG loop
    got = solve(p, loss, cfg, ExecutionPlan.gpu())
    monkeypatch.setenv("TRON_B200_NCCL_GRAPH", "1")  # allreduces inside the CG graph
    in_graph = solve(p, loss, cfg, ExecutionPlan.gpu())
    assert [it.cg_iters for it in in_graph.trace.iterations] == [it.cg_iters for it in base.trace.iterations]
    assert rel_err(in_graph.w, base.w) <= 1e-12
    assert got.objective == base.objective
    assert np.array_equal(got.w, base.w)
    assert [it.cg_iters for it in got.trace.iterations] == [it.cg_iters for it in base.trace.iterations]
    w_ref, t_ref = ref.solve(p, 0 if loss == LossKind.Logistic else 1, cfg)
    assert rel_err(got.objective, t_ref["objective"]) <= 1e-6
    assert rel_err(got.w, w_ref) <= 1e-6


# The drop-in boundary, literally: the reference's own tron::solve
# (tron.cpp:127-217, compiled from /root/reference into oracle/_ref) driving a
# tron::LossEvaluator whose every method forwards to the C ABI of
# libtron_b200.so -- the binding INTEGRATION.md §1 proposes for backend.cpp.
@pytest.mark.parametrize("case", ["sparse_lr", "dense_svm", "sparse_svm_precond"])
def test_reference_solver_drives_the_gpu_evaluator(ref, case):
    from paper_2008_03433_b200 import LIB_PATH
    p, loss, over = {
        "sparse_lr": (synth.synth_sparse(1, 20242, 47236, 74), 0, {}),
        "dense_svm": (synth.testgen_dense_problem(3001, 200, 20, 1.0), 1, dict(eps=1e-8)),
        "sparse_svm_precond": (synth.testgen_sparse_problem(3400, 400, 60, 2.0, 0.15), 1,
                               dict(eps=1e-7, use_preconditioner=True)),
    }[case]
    cfg = TrustRegionConfig(eps=over.pop("eps", 0.01), **over)
    w_gpu, t_gpu = ref.solve_with_gpu_evaluator(LIB_PATH, p, loss, cfg)
    w_ref, t_ref = ref.solve(p, loss, cfg)
    assert rel_err(t_gpu["objective"], t_ref["objective"]) <= 1e-9
    assert rel_err(w_gpu, w_ref) <= 1e-6
    assert [it["cg_iters"] for it in t_gpu["iterations"]] == [it["cg_iters"] for it in t_ref["iterations"]]


# predict (model.cpp:88-117) on the device against the reference's own predict:
# at the same w the labels are bit-identical (sequential row sums, no FMA), and
# each solver's own model labels a held-out set identically.
@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_predict_matches_reference(ref, kind):
    if kind == "dense":
        p, pt, loss, oloss = synth.synth_dense(1, 200_000, 40), synth.synth_dense(2, 100_000, 40), SVM, 1
    else:
        p, pt = synth.synth_sparse(1, 20242, 47236, 74), synth.synth_sparse(2, 10000, 47236, 74)
        loss, oloss = LR, 0
    cfg = TrustRegionConfig(eps=0.01)
    res = solve(p, loss, cfg, plan())
    w_ref, _ = ref.solve(p, oloss, cfg)
    Xt = pt.X
    Xt.y = pt.y
    with make_evaluator(pt, loss, plan()) as ev:
        lab_ref_w, c_ref_w = ev.predict(w_ref)
        lab_gpu, _ = ev.predict(res.w)
    lab_ref, c_ref = ref.predict(Xt, w_ref)
    assert np.array_equal(lab_ref_w, lab_ref) and c_ref_w == c_ref
    assert np.array_equal(lab_gpu, lab_ref)
    assert set(np.unique(lab_gpu)) <= {-1.0, 1.0}
