"""Reference-order reductions (ExecutionPlan.reference_order, refexact.cu):
the dense L2-SVM evaluator and solve are BIT-FOR-BIT the reference's --
fun/grad/Hv/preconditioner against the reference's own loss kernels, and
whole solves (objective, w, every iteration record, active set) against
tron::solve (backend.cpp:314-318)."""
import numpy as np
import pytest

from paper_2008_03433_b200 import (ExecutionPlan, LossKind, SvmStrategy, TrustRegionConfig,
                                   make_evaluator, solve, synth)

pytestmark = pytest.mark.gpu
SVM = LossKind.L2Svm


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def ro_plan(**kw):
    return ExecutionPlan.gpu(reference_order=True, **kw)


CASES = [
    ("testgen200x20", lambda: synth.testgen_dense_problem(3001, 200, 20, 1.0)),
    ("synth1e5x40", lambda: synth.synth_dense(1, 100_000, 40)),
    ("synth777x7", lambda: synth.synth_dense(3, 777, 7)),
    ("synth3e6x40", lambda: synth.synth_dense(5, 3_000_000, 40)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_evaluator_bitwise(ref, case):
    name, make = CASES[case]
    p = make()
    n = p.X.cols
    w = synth.testgen_random_vector(41 + case, n, 0.2)
    v = synth.testgen_random_vector(51 + case, n, 1.0)
    want = ref.svm(p, w, v)
    with make_evaluator(p, SVM, ro_plan()) as ev:
        f = ev.eval_candidate(w)
        assert bits(f) == bits(want["f"]), name
        ev.commit()
        assert np.array_equal(bits(ev.gradient()), bits(want["g"])), name
        assert np.array_equal(bits(ev.hessian_vec(v)), bits(want["hv"])), name
        assert np.array_equal(bits(ev.precond_diagonal()), bits(want["M"])), name
        assert np.array_equal(ev.committed_state().active, want["active"]), name


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("mode", ["device", "host_cg"])
def test_solve_bitwise(ref, case, precond, mode):
    name, make = CASES[case]
    p = make()
    cfg = TrustRegionConfig(eps=0.01 if p.X.rows > 10_000 else 1e-8, use_preconditioner=precond)
    got = solve(p, SVM, cfg, ro_plan(solve_mode=mode))
    w_ref, t_ref = ref.solve(p, 1, cfg)
    assert bits(got.objective) == bits(t_ref["objective"]), name
    assert np.array_equal(bits(got.w), bits(w_ref)), name
    its = [(r.accepted, r.cg_iters, int(r.cg_exit), r.f_candidate, r.delta, r.sigma)
           for r in got.trace.iterations]
    want = [(r["accepted"], r["cg_iters"], r["cg_exit"], r["f_candidate"], r["delta"], r["sigma"])
            for r in t_ref["iterations"]]
    assert its == want, name


def test_reference_order_rejects_what_it_cannot_reproduce():
    from paper_2008_03433_b200 import DeviceError, StrategyPreconditionError
    p = synth.synth_dense(1, 1000, 40)
    with pytest.raises(DeviceError):
        make_evaluator(p, LossKind.Logistic, ro_plan())
    with pytest.raises(StrategyPreconditionError):
        make_evaluator(p, SVM, ro_plan(svm_strategy=SvmStrategy.Gathered))
    with pytest.raises(DeviceError):
        make_evaluator(synth.synth_dense(1, 1000, 60), SVM, ro_plan())
