"""Active-set churn per outer iteration of a dense L2-SVM solve (sizes the
incremental Gram update): solve with max_outer_iters = k for k = 1.. and diff
the committed active sets."""
import sys, json, numpy as np
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth

W = sys.argv[1] if len(sys.argv) > 1 else "P1"
p = synth.make_shape(W, seed=1)
prev = np.arange(len(p.y))  # w0 = 0: every row is active
out = []
with make_evaluator(p, LossKind.L2Svm, ExecutionPlan.gpu()) as ev:
    for k in range(1, 6):
        r = ev.solve(TrustRegionConfig(eps=0.01, max_outer_iters=k))
        a = np.asarray(ev.committed_state().active)
        ent = np.setdiff1d(a, prev, assume_unique=True).size
        left = np.setdiff1d(prev, a, assume_unique=True).size
        out.append(dict(iters=k, active=int(a.size), entered=int(ent), left=int(left), status=str(getattr(r, "status", ""))))
        print(json.dumps(out[-1]), flush=True)
        prev = a
        if getattr(r, "converged", False):
            break
