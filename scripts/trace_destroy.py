"""Destroy-phase times (TRON_B200_TRACE=1) of an N1 context after a solve."""
import os, sys, time
os.environ["TRON_B200_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
p = synth.make_shape(sys.argv[1] if len(sys.argv) > 1 else "N1")
for rep in range(3):
    ev = make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu())
    ev.solve(TrustRegionConfig(eps=0.01))
    t0 = time.perf_counter(); ev.close(); t1 = time.perf_counter()
    print(f"destroy {1e3*(t1-t0):.3f} ms", file=sys.stderr, flush=True)
