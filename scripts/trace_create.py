"""Phase times of context creation + one solve through the public API (TRON_B200_TRACE=1),
from pageable and from pinned host arrays."""
import os, sys, time
os.environ["TRON_B200_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from bench import pin_problem
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
for name in sys.argv[1:] or ["N1"]:
    p0 = synth.make_shape(name)
    loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
    for kind, p in (("pageable", p0), ("pinned", pin_problem(p0, torch))):
        for rep in range(3):
            t0 = time.perf_counter()
            with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
                t1 = time.perf_counter()
                r = ev.solve(TrustRegionConfig(eps=0.01))
                t2 = time.perf_counter()
            t3 = time.perf_counter()
            print(f"{name} {kind} rep{rep}: create {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms "
                  f"(device {r.device_ms:.2f}), destroy {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f}",
                  file=sys.stderr, flush=True)
