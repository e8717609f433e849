"""One truncated CG on a workload (host-launched loop when TRON_B200_NO_GRAPH=1), for ncu."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
name = sys.argv[1] if len(sys.argv) > 1 else "N1"
p = synth.make_shape(name)
with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
    ev.eval_candidate(np.zeros(p.X.cols)); ev.commit()
    ev.truncated_cg(1e30, TrustRegionConfig(cg_tol=1e-12, max_cg_iters=6))
