"""Small-fixture workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family and every CG engine once.

  compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

Engines covered: single-block CG (n <= 4096, dense and sparse), the 8-CTA
cluster CG step (4096 < n <= 262144), the cooperative grid CG step
(n > 262144, with the p.Hp / ||g|| fused into the segmented emission), the
reference-order dense L2-SVM, the Gathered L2-SVM (dense panel and CSR X_I
with its CSC copy), the preconditioner, predict, the staged-u segmented
product (>= 128 nonzeros per column entry), the dense Gram pass (DMMA; the
default for dense), the tall-skinny traversal, out-of-core streaming and
column panels.  Each solve is checked against
the C oracle so a sanitizer-clean run is also a correct one.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import (ExecutionPlan, LossKind, SvmStrategy, TrustRegionConfig,  # noqa: E402
                                   make_evaluator, synth)
from pyoracle import L2SVM, LOGISTIC, Port  # noqa: E402  (checker)

port = Port()


def check(name, p, loss, plan, eps=0.01, precond=False, tol=1e-6):
    cfg = TrustRegionConfig(eps=eps, use_preconditioner=precond)
    with make_evaluator(p, loss, plan) as ev:
        got = ev.solve(cfg)
        if loss == LossKind.L2Svm:
            ev.committed_state()
        ev.predict(got.w)
        ev.hessian_vec(np.ones(p.X.cols))
        ev.precond_diagonal()
    w_ref, t_ref = port.solve(p, LOGISTIC if loss == LossKind.Logistic else L2SVM, cfg)
    rf = abs(got.objective - t_ref["objective"]) / abs(t_ref["objective"])
    rw = np.linalg.norm(got.w - w_ref) / max(np.linalg.norm(w_ref), 1e-300)
    ok = rf <= tol and rw <= max(tol, 1e-4)
    print(f"{name:40s} rel_f={rf:.1e} rel_w={rw:.1e} {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


LR, SVM = LossKind.Logistic, LossKind.L2Svm
gpu = ExecutionPlan.gpu
cases = [
    ("sparse LR small-n engine", synth.synth_sparse(9, 600, 3000, 20), LR, gpu(), {}),
    ("sparse LR small-n precond", synth.synth_sparse(9, 600, 3000, 20), LR, gpu(), dict(precond=True)),
    ("sparse LR cluster engine", synth.synth_sparse(3, 800, 20000, 30), LR, gpu(), {}),
    ("sparse LR cooperative engine", synth.synth_sparse(4, 1500, 300000, 40), LR, gpu(), {}),
    ("sparse LR staged u (nnz >= 128 n)", synth.synth_sparse(5, 4000, 3000, 200), LR, gpu(), {}),
    ("sparse SVM indirect", synth.synth_sparse(6, 700, 5000, 25), SVM, gpu(), {}),
    ("sparse SVM gathered CSR", synth.synth_sparse(6, 700, 5000, 25), SVM,
     gpu(svm_strategy=SvmStrategy.Gathered), {}),
    ("dense SVM indirect", synth.synth_dense(1, 5000, 40), SVM, gpu(), dict(eps=1e-8)),
    ("dense SVM gathered panel", synth.synth_dense(1, 5000, 40), SVM, gpu(svm_strategy=SvmStrategy.Gathered),
     dict(eps=1e-8)),
    ("dense SVM precond", synth.synth_dense(2, 3000, 40), SVM, gpu(), dict(precond=True)),
    ("dense SVM reference order", synth.synth_dense(1, 5000, 40), SVM, gpu(reference_order=True), {}),
    ("dense LR", synth.testgen_dense_problem(1001, 50, 5, 1.0), LR, gpu(), dict(eps=1e-8)),
    ("dense SVM out-of-core streaming", synth.synth_dense(1, 5000, 40, decades=0.0), SVM,
     gpu(out_of_core=1, stream_block_rows=1024), dict(eps=1e-8)),
    ("dense SVM tall-skinny (no Gram)", synth.synth_dense(1, 5000, 40), SVM, gpu(), dict(eps=1e-8)),
    ("sparse LR column panels", synth.synth_sparse(13, 600, 9000, 20), LR, gpu(), {}),
    ("dense SVM Gram: separate first pass", synth.synth_dense(1, 5000, 40), SVM, gpu(), dict(eps=1e-8)),
    ("dense SVM Gram: no incremental update", synth.synth_dense(1, 5000, 40), SVM, gpu(), dict(eps=1e-8)),
]
# per-case environment (applied before the case's context is created)
ENV = {"dense SVM tall-skinny (no Gram)": {"TRON_B200_DENSE_GRAM": "0"},
       "sparse LR column panels": {"TRON_B200_PANEL_COLS": "2000"},
       "dense SVM Gram: separate first pass": {"TRON_B200_GRAM_FIRST": "separate"},
       "dense SVM Gram: no incremental update": {"TRON_B200_GRAM_DELTA": "0"}}
if sys.argv[1:] == ["--count"]:
    print(len(cases))
    sys.exit(0)
# argv: case indices to run (default: all)
only = {int(a) for a in sys.argv[1:]}
bad = 0
for i, (name, p, loss, plan, kw) in enumerate(cases):
    if only and i not in only:
        continue
    for k, v in ENV.get(name, {}).items():
        os.environ[k] = v
    bad += not check(name, p, loss, plan, **kw)
    for k in ENV.get(name, {}):
        os.environ.pop(k)
print("sanitize cases:", "all ok" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
