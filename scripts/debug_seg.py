import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, make_evaluator, synth
from pyoracle import Port
p = synth.synth_sparse(9, 2000, 5000, 37)
X = p.X
w = synth.testgen_random_vector(1007, X.cols, 0.3)
want = Port().logistic(p, w)
cnt = np.bincount(X.col_indices, minlength=X.cols)
for trial in range(3):
    with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
        ev.eval_candidate(w); ev.commit(); g = ev.gradient()
    bad = np.where(~np.isclose(g, want["g"], rtol=1e-10, atol=1e-12))[0]
    print("trial", trial, "bad", len(bad), "first", bad[:20].tolist())
    print(" lens", cnt[bad[:20]].tolist())
    print(" got", g[bad[:5]].tolist(), "want", want["g"][bad[:5]].tolist(), "w", w[bad[:5]].tolist())
