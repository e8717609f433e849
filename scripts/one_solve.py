"""One solve of a workload (for ncu launch lists): create, solve once, exit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
W = sys.argv[1] if len(sys.argv) > 1 else "P1"
p = synth.make_shape(W)
loss = LossKind.Logistic if synth.SHAPES[W]["loss"] == "logistic" else LossKind.L2Svm
with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
    r = ev.solve(TrustRegionConfig(eps=0.01))
    print("device_ms", r.device_ms, [it.cg_iters for it in r.trace.iterations])
