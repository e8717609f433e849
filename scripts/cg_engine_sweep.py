"""Device time of sparse LR solves, 8-CTA cluster CG vs cooperative-grid CG, over n
(sizes kClusterCgMaxN): python scripts/cg_engine_sweep.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
cfg = TrustRegionConfig(eps=0.01)
for n in (6000, 12000, 24000, 47236, 100000, 200000):
    p = synth.synth_sparse(1, 20242, n, 74)
    row = {"n": n}
    for eng in ("1", "0"):
        os.environ["TRON_B200_CLUSTER_CG"] = eng
        with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
            for _ in range(3):
                ev.solve(cfg)
            ts = [ev.solve(cfg).device_ms for _ in range(7)]
            r = ev.solve(cfg)
        row["cluster" if eng == "1" else "coop"] = round(float(np.median(ts)), 4)
        row["cg_" + ("cluster" if eng == "1" else "coop")] = [it.cg_iters for it in r.trace.iterations]
    print(json.dumps(row), flush=True)
