"""Device-resident outer trust-region loop (trloop.cu):
the whole solve after the initial commit is one graph launch.  It runs the
same kernels in the same order as the host-driven loop (TRON_B200_DEVICE_LOOP=0),
so both give the same bits -- w, objective, every iteration record -- and both
meet the reference (tron.cpp:127-217) within the north-star tolerance."""
import numpy as np
import pytest

from conftest import rel_err
from paper_2008_03433_b200 import (ExecutionPlan, LossKind, NumericalFailureError, TrustRegionConfig,
                                   make_evaluator, synth)

pytestmark = pytest.mark.gpu
LR, SVM = LossKind.Logistic, LossKind.L2Svm

CASES = [
    ("sparse-lr-small", lambda: synth.synth_sparse(9, 600, 3000, 20), LR),
    ("sparse-lr-cluster", lambda: synth.synth_sparse(3, 800, 20000, 30), LR),
    ("sparse-lr-coop", lambda: synth.synth_sparse(4, 1500, 300000, 40), LR),
    ("sparse-svm", lambda: synth.synth_sparse(6, 700, 5000, 25), SVM),
    ("dense-svm", lambda: synth.synth_dense(1, 20000, 40), SVM),
    ("dense-lr", lambda: synth.testgen_dense_problem(2001, 200, 20, 1.0), LR),
]


def run(p, loss, cfg, monkeypatch, device_loop, plan=None):
    monkeypatch.setenv("TRON_B200_DEVICE_LOOP", "1" if device_loop else "0")
    with make_evaluator(p, loss, plan or ExecutionPlan.gpu()) as ev:
        r = ev.solve(cfg)
        g = ev.gradient()
        led = ev.ledger()
    return r, g, led


def records(r):
    return [(it.f_candidate, it.gradient_norm, it.delta, it.sigma, it.accepted, int(it.cg_exit), it.cg_iters)
            for it in r.trace.iterations]


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_device_loop_equals_host_loop(case, precond, monkeypatch):
    name, make, loss = CASES[case]
    p = make()
    cfg = TrustRegionConfig(eps=1e-4, use_preconditioner=precond)
    a, ga, la = run(p, loss, cfg, monkeypatch, True)
    b, gb, lb = run(p, loss, cfg, monkeypatch, False)
    assert np.array_equal(a.w.view(np.uint64), b.w.view(np.uint64)), name
    assert a.objective == b.objective
    assert records(a) == records(b)
    assert a.converged == b.converged and a.hessian_products == b.hessian_products
    assert np.array_equal(ga.view(np.uint64), gb.view(np.uint64))  # gradient() of the committed iterate
    assert (a.trace.accepted_steps, a.trace.gradient_materializations, a.trace.objective_evaluations) == \
        (b.trace.accepted_steps, b.trace.gradient_materializations, b.trace.objective_evaluations)
    assert (la.margin_passes, la.gradient_materializations) == (lb.margin_passes, lb.gradient_materializations)


def test_device_loop_matches_reference(ref):
    p = synth.synth_sparse(3, 800, 20000, 30)
    cfg = TrustRegionConfig(eps=1e-3)
    with make_evaluator(p, LR, ExecutionPlan.gpu()) as ev:
        r = ev.solve(cfg)
    w_ref, t_ref = ref.solve(p, 0, cfg)
    assert rel_err(r.objective, t_ref["objective"]) <= 1e-10
    assert rel_err(r.w, w_ref) <= 1e-8
    assert [it.cg_iters for it in r.trace.iterations] == [it["cg_iters"] for it in t_ref["iterations"]]


@pytest.mark.parametrize("max_outer", [1, 2, 3])
def test_device_loop_outer_limit(max_outer, monkeypatch):
    p = synth.synth_dense(2, 30000, 40)
    cfg = TrustRegionConfig(eps=1e-12, max_outer_iters=max_outer)
    a, _, _ = run(p, SVM, cfg, monkeypatch, True)
    b, _, _ = run(p, SVM, cfg, monkeypatch, False)
    assert len(a.trace.iterations) == max_outer and not a.converged
    assert records(a) == records(b)
    assert np.array_equal(a.w, b.w)


def test_device_loop_rejections_and_small_radius(monkeypatch):
    # a tiny sigma0 / aggressive shrink mix exercises rejected candidates:
    # the committed slot must not move on a rejection
    p = synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0)
    cfg = TrustRegionConfig(eps=1e-8, sigma0=0.5, eta1=0.6, eta2=0.9, max_outer_iters=200)
    a, ga, _ = run(p, LR, cfg, monkeypatch, True)
    b, gb, _ = run(p, LR, cfg, monkeypatch, False)
    assert any(not it.accepted for it in a.trace.iterations)
    assert records(a) == records(b)
    assert np.array_equal(a.w, b.w) and np.array_equal(ga, gb)


def test_device_loop_warm_start_and_reuse(monkeypatch):
    p = synth.synth_sparse(5, 900, 8000, 25)
    cfg = TrustRegionConfig(eps=1e-3)
    monkeypatch.setenv("TRON_B200_DEVICE_LOOP", "1")
    with make_evaluator(p, LR, ExecutionPlan.gpu()) as ev:
        r1 = ev.solve(cfg)
        r2 = ev.solve(cfg)  # same context: graph reused, slots in any parity
        r3 = ev.solve(TrustRegionConfig(eps=1e-6), warm_start=r1.w)
        f_after = ev.eval_candidate(r3.w)
    assert np.array_equal(r1.w, r2.w) and records(r1) == records(r2)
    assert r3.converged and rel_err(f_after, r3.objective) <= 1e-14


def test_device_loop_short_trace_cap(monkeypatch):
    # more outer iterations than the inline read-back of iteration records
    p = synth.testgen_dense_problem_scaled(117, 80, 8, 1000.0, 20.0)
    cfg = TrustRegionConfig(eps=1e-14, sigma0=0.5, eta1=0.6, eta2=0.9, max_outer_iters=90, gamma1=0.01,
                            gamma2=0.02, gamma3=1.01)
    a, _, _ = run(p, LR, cfg, monkeypatch, True)
    b, _, _ = run(p, LR, cfg, monkeypatch, False)
    assert records(a) == records(b)


def test_device_loop_nonfinite_objective(monkeypatch):
    # a huge C overflows the objective at the first candidate step
    p = synth.testgen_dense_problem(1001, 50, 5, 1e308)
    for loop in (True, False):
        monkeypatch.setenv("TRON_B200_DEVICE_LOOP", "1" if loop else "0")
        with make_evaluator(p, LR, ExecutionPlan.gpu()) as ev:
            with pytest.raises(NumericalFailureError):
                ev.solve(TrustRegionConfig(eps=1e-8))
