"""Diagnose dense small-n CG/solve parity on the GPU."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, solve, synth
from pyoracle import Port, Reference
port, ref = Port(), Reference()
def rel(a, b): return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))
for l in (3001, 20000, 200000):
    p = synth.synth_dense(1, l, 40)
    for loss, ol in ((LossKind.L2Svm, 1), (LossKind.Logistic, 0)):
        cfg = TrustRegionConfig(eps=0.01)
        w_ref, t_ref = ref.solve(p, ol, cfg)
        for mode in ("device", "host_cg"):
            r = solve(p, loss, cfg, ExecutionPlan.gpu(solve_mode=mode))
            print(f"l={l} {loss.name} {mode}: rel_f={rel(r.objective, t_ref['objective']):.2e} rel_w={rel(r.w, w_ref):.2e}",
                  "gpu", [(it.accepted, it.cg_iters, int(it.cg_exit), f"{it.f_candidate:.10g}") for it in r.trace.iterations],
                  "ref", [(it['accepted'], it['cg_iters'], it['cg_exit'], f"{it['f_candidate']:.10g}") for it in t_ref['iterations']], flush=True)
        # CG at w=0 with increasing caps
        with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
            ev.eval_candidate(np.zeros(40)); ev.commit(); g = ev.gradient()
            want = (port.svm if ol else port.logistic)(p, np.zeros(40), g)
            print("  g rel", rel(g, want["g"]), "hv rel", rel(ev.hessian_vec(g), want["hv"]))
            for cap in (1, 2, 3, 5, 8, 12, 20, 40):
                dev = ev.truncated_cg(1e9, TrustRegionConfig(cg_tol=1e-9, max_cg_iters=cap))
                host = port.truncated_cg(g, ev.hessian_vec, 1e9, None, cg_tol=1e-9, max_cg_iters=cap)
                print(f"  cap={cap}: dev it={dev.iters} ex={int(dev.exit)} host it={host['iters']} ex={host['exit']} rel_d={rel(dev.d, host['d']):.2e} q {dev.model_value:.12g} {host['model_value']:.12g}", flush=True)
