"""Per-CG-iteration cost inside the device CG graph (wall-clock difference of
truncated_cg with 21 vs 1 iterations), plus fun / commit wall times."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
for name in sys.argv[1:] or ["R1", "N1"]:
    p = synth.make_shape(name)
    loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
    with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
        w = np.zeros(p.X.cols)
        ev.eval_candidate(w); ev.commit()
        def t_cg(k, reps=20):
            cfg = TrustRegionConfig(cg_tol=1e-12, max_cg_iters=k)
            ev.truncated_cg(1e30, cfg)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter(); ev.truncated_cg(1e30, cfg); ts.append(time.perf_counter() - t0)
            return min(ts)
        a, b = t_cg(1), t_cg(21)
        tf = []
        for _ in range(20):
            t0 = time.perf_counter(); ev.eval_candidate(w); tf.append(time.perf_counter() - t0)
        tc = []
        for _ in range(10):
            ev.eval_candidate(w)
            t0 = time.perf_counter(); ev.commit(); tc.append(time.perf_counter() - t0)
        print(f"{name}: per CG iteration {1e6*(b-a)/20:.1f} us; 1-iteration CG call {1e6*a:.0f} us; "
              f"eval_candidate {1e6*min(tf):.0f} us; commit {1e6*min(tc):.0f} us", flush=True)
