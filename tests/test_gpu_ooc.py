"""Out-of-core dense problems (the reference's mix
remedy for a budget overflow, backend.cpp:256-261): X stays in host memory and
every pass streams it through two device windows.  Forced on here with small
blocks (several blocks, a ragged last one): the streamed evaluator and solve
agree with the in-memory ones (different partial-sum split: <= 1e-13) and
with the reference; margins, active sets and predictions are bit-identical."""
import numpy as np
import pytest

from conftest import rel_err
from paper_2008_03433_b200 import (ExecutionPlan, LossKind, StrategyPreconditionError, SvmStrategy,
                                   TrustRegionConfig, make_evaluator, synth)
from paper_2008_03433_b200.tron import Error

pytestmark = pytest.mark.gpu
LR, SVM = LossKind.Logistic, LossKind.L2Svm

# (equal column scales: well-conditioned, so whole solves can be compared at
# 1e-6 in w; the 2-decade SYNTH scales leave w flat to ~1e-5 at eps = 1e-6)
CASES = [
    ("svm", lambda: synth.synth_dense(1, 300_000, 40, decades=0.0), SVM, 40_000),
    ("svm-small-blocks", lambda: synth.synth_dense(7, 50_001, 40, decades=0.0), SVM, 256),
    ("lr", lambda: synth.testgen_dense_problem(2001, 60_003, 30, 1.0), LR, 7_000),
]


def evaluate(p, loss, plan, w, v):
    with make_evaluator(p, loss, plan) as ev:
        f = ev.eval_candidate(w)
        st = ev.candidate_state()
        ev.commit()
        g, hv, m = ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()
        lab, correct = ev.predict(w)
        res = ev.solve(TrustRegionConfig(eps=1e-6))
        act = ev.committed_state().active if loss == SVM else None
    return dict(f=f, z=st.z, act_w=getattr(st, "active", None), g=g, hv=hv, m=m, lab=lab,
                correct=correct, res=res, act=act)


@pytest.mark.parametrize("pin", ["1", "0"])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_streamed_equals_in_memory(ref, monkeypatch, case, pin):
    monkeypatch.setenv("TRON_B200_OOC_PIN", pin)
    name, make, loss, blk = CASES[case]
    p = make()
    n = p.X.cols
    w = synth.testgen_random_vector(3, n, 0.1)
    v = synth.testgen_random_vector(4, n, 1.0)
    a = evaluate(p, loss, ExecutionPlan.gpu(out_of_core=1, stream_block_rows=blk), w, v)
    b = evaluate(p, loss, ExecutionPlan.gpu(out_of_core=-1), w, v)
    assert rel_err(a["f"], b["f"]) <= 1e-13
    assert np.array_equal(a["z"].view(np.uint64), b["z"].view(np.uint64))  # sequential row dots
    if loss == SVM:
        assert np.array_equal(a["act_w"], b["act_w"])
    for k in ("g", "hv", "m"):
        assert rel_err(a[k], b[k]) <= 1e-13, k
    assert np.array_equal(a["lab"], b["lab"]) and a["correct"] == b["correct"]
    # whole solves: the same trust-region path up to the summation split of the
    # block partials (the north-star gate: 1e-6, counts +-1)
    ra, rb = a["res"], b["res"]
    assert rel_err(ra.objective, rb.objective) <= 1e-10 and rel_err(ra.w, rb.w) <= 1e-6
    ca, cb = [it.cg_iters for it in ra.trace.iterations], [it.cg_iters for it in rb.trace.iterations]
    assert len(ca) == len(cb) and all(abs(x - y) <= 1 for x, y in zip(ca, cb))
    w_ref, t_ref = ref.solve(p, 0 if loss == LR else 1, TrustRegionConfig(eps=1e-6))
    assert rel_err(ra.objective, t_ref["objective"]) <= 1e-6 and rel_err(ra.w, w_ref) <= 1e-6


def test_streamed_strategy_and_mode_errors():
    p = synth.synth_dense(1, 5000, 40)
    with pytest.raises(StrategyPreconditionError):
        make_evaluator(p, SVM, ExecutionPlan.gpu(out_of_core=1, svm_strategy=SvmStrategy.Gathered))
    with pytest.raises(Error):
        make_evaluator(p, SVM, ExecutionPlan.gpu(out_of_core=1, reference_order=True))
    # Auto falls back to the index-indirect traversal
    with make_evaluator(p, SVM, ExecutionPlan.gpu(out_of_core=1, svm_strategy=SvmStrategy.Auto,
                                                  stream_block_rows=1024)) as ev:
        r = ev.solve(TrustRegionConfig(eps=1e-3))
        assert r.converged


def test_streamed_memory_is_windows_only():
    p = synth.synth_dense(2, 400_000, 40)  # 128 MB of X
    with make_evaluator(p, SVM, ExecutionPlan.gpu(out_of_core=1, stream_block_rows=16384)) as ev:
        held = ev.memory_bytes()
    with make_evaluator(p, SVM, ExecutionPlan.gpu(out_of_core=-1)) as ev:
        full = ev.memory_bytes()
    assert full - held >= 0.9 * p.X.values.nbytes
