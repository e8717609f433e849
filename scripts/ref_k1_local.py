"""K1 reference solves for the tight-eps parity study (CPU only; run where the
reference is compiled).  The reference is deterministic and thread-count
independent, so these w's are the ones a run on the GPU box
would produce.  Writes scratch/k1_ref_<eps>.npy + scratch/k1_ref.json; the
GPU side (scripts/parity_k1_tight.py) compares against them.
  python scripts/ref_k1_local.py [eps ...]"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import synth  # SYNTH-v1 generator (bit-identical to testgen)
from pyoracle import Reference

eps_list = [float(e) for e in sys.argv[1:]] or [0.01, 1e-6]
out_dir = os.path.join(ROOT, "scratch")
os.makedirs(out_dir, exist_ok=True)
t0 = time.time()
p = synth.make_shape("K1")
rec = {"generate_s": time.time() - t0, "threads": len(os.sched_getaffinity(0)), "solves": {}}
ref = Reference()
path = os.path.join(out_dir, "k1_ref.json")
if os.path.exists(path):
    rec = json.load(open(path))
for e in eps_list:
    t0 = time.time()
    w, t = ref.solve(p, 0, None, backend=Reference.PAR, workers=len(os.sched_getaffinity(0)), eps=e)
    secs = time.time() - t0
    np.save(os.path.join(out_dir, f"k1_ref_{e!r}.npy"), w)
    g = ref.logistic(p, w, np.zeros(p.X.cols))
    rec["solves"][repr(e)] = {
        "seconds": secs, "objective": t["objective"], "converged": t["converged"],
        "outer": len(t["iterations"]), "accepted": sum(r["accepted"] for r in t["iterations"]),
        "cg_iters": [r["cg_iters"] for r in t["iterations"]],
        "gradient_norms": [r["gradient_norm"] for r in t["iterations"]],
        "gradient_norm_initial": t["gradient_norm_initial"],
        "reference_gradient_norm_at_w": float(np.linalg.norm(g["g"])), "w_norm": float(np.linalg.norm(w))}
    json.dump(rec, open(path, "w"), indent=1)
    print(e, rec["solves"][repr(e)], flush=True)
