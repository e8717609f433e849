"""Probe: can the NCCL allreduces of the sharded path live inside the CG while-graph?
Runs one-rank forced-NCCL solves with and without the graph and compares."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["TRON_B200_FORCE_NCCL"] = "1"
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
cfg = TrustRegionConfig(eps=0.01)
for name in ["R1", "N1"]:
    p = synth.make_shape(name)
    for g in ("0", "1"):
        os.environ["TRON_B200_NCCL_GRAPH"] = g
        try:
            with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
                r = ev.solve(cfg)
                ts = []
                for _ in range(5):
                    r = ev.solve(cfg); ts.append(r.device_ms)
            print(name, "nccl-graph" if g == "1" else "nccl-hostloop", "obj", r.objective, "hv", r.hessian_products, "ms", min(ts), flush=True)
        except Exception as e:
            print(name, g, "FAILED", type(e).__name__, str(e)[:200], flush=True)
