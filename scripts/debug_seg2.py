"""Gradient at w=0 (= -C/2 X^T y for LR) against numpy on full-size shapes."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, make_evaluator, synth
for name in sys.argv[1:] or ["R1"]:
    p = synth.make_shape(name)
    X = p.X
    ref = np.zeros(X.cols)
    rows = np.repeat(np.arange(X.rows), np.diff(X.row_offsets))
    np.add.at(ref, X.col_indices, X.values * (-0.5 * p.C * p.y[rows]))
    with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
        ev.eval_candidate(np.zeros(X.cols)); ev.commit()
        g = ev.gradient()
    err = np.abs(g - ref) / (np.abs(ref) + 1e-12)
    bad = np.nonzero(err > 1e-9)[0]
    print(name, "max rel", err.max(), "bad", bad.size, bad[:10], "nan", np.isnan(g).sum())
