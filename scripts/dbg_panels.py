"""Panel solve debugging: LR sparse, panels on/off, device/host loop, traces."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
p = synth.synth_sparse(13, 3000, 40000, 30)
for pw in ("1000", "0"):
    for loop in ("1", "0"):
        os.environ["TRON_B200_PANEL_COLS"] = pw
        os.environ["TRON_B200_DEVICE_LOOP"] = loop
        with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
            try:
                r = ev.solve(TrustRegionConfig(eps=1e-9))
                print(pw, loop, "ok", r.objective, [(it.cg_iters, round(it.sigma, 4), it.accepted) for it in r.trace.iterations])
            except Exception as e:
                print(pw, loop, "FAIL", e, [(it.cg_iters, it.f_candidate, it.sigma) for it in e.trace.iterations] if hasattr(e, "trace") else "")
