"""Generates tests/golden/*.json from the reference CPU solver compiled from
/root/reference sources (oracle/_ref/libtronref.so, built by oracle/Makefile).

Run from the repo root:  python tests/golden/make_golden.py
Each fixture records the reference's objective, w, and per-iteration
(accepted, cg_iters, cg_exit) for a deterministic problem, so the oracle and
the GPU path stay pinned even where the reference build is unavailable.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

CASES = [
    dict(name="lr_dense_50x5", problem=dict(gen="dense", seed=1001, l=50, n=5, C=1.0),
         loss="logistic", config=dict(eps=1e-8)),
    dict(name="lr_dense_200x20", problem=dict(gen="dense", seed=2001, l=200, n=20, C=1.0),
         loss="logistic", config=dict(eps=1e-8, max_outer_iters=100)),
    dict(name="svm_dense_200x20", problem=dict(gen="dense", seed=3001, l=200, n=20, C=1.0),
         loss="l2svm", config=dict(eps=1e-8, max_outer_iters=100)),
    dict(name="lr_sparse_400x60", problem=dict(gen="sparse", seed=3400, l=400, n=60, C=2.0, density=0.15),
         loss="logistic", config=dict(eps=1e-7)),
    dict(name="svm_sparse_400x60_precond",
         problem=dict(gen="sparse", seed=3400, l=400, n=60, C=2.0, density=0.15),
         loss="l2svm", config=dict(eps=1e-7, use_preconditioner=True)),
    dict(name="lr_scaled_rejections", problem=dict(gen="scaled", seed=117, l=80, n=8, C=1000.0, scale=20.0),
         loss="logistic", config=dict(eps=1e-6)),
    dict(name="svm_synth_dense_20000x40", problem=dict(gen="synth_dense", seed=1, l=20000, n=40, C=1.0),
         loss="l2svm", config=dict(eps=0.01)),
    dict(name="lr_synth_sparse_2000x5000", problem=dict(gen="synth_sparse", seed=9, l=2000, n=5000, k=37, C=1.0),
         loss="logistic", config=dict(eps=0.01)),
]


def build_problem(spec):
    from paper_2008_03433_b200 import synth
    g = spec["gen"]
    if g == "dense":
        return synth.testgen_dense_problem(spec["seed"], spec["l"], spec["n"], spec["C"])
    if g == "scaled":
        return synth.testgen_dense_problem_scaled(spec["seed"], spec["l"], spec["n"], spec["C"], spec["scale"])
    if g == "sparse":
        return synth.testgen_sparse_problem(spec["seed"], spec["l"], spec["n"], spec["C"], spec["density"])
    if g == "synth_dense":
        return synth.synth_dense(spec["seed"], spec["l"], spec["n"], C=spec["C"])
    if g == "synth_sparse":
        return synth.synth_sparse(spec["seed"], spec["l"], spec["n"], spec["k"], C=spec["C"])
    raise ValueError(g)


def main():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from paper_2008_03433_b200 import TrustRegionConfig
    from pyoracle import L2SVM, LOGISTIC, Reference
    ref = Reference()
    for case in CASES:
        p = build_problem(case["problem"])
        loss = LOGISTIC if case["loss"] == "logistic" else L2SVM
        w, t = ref.solve(p, loss, TrustRegionConfig(**case["config"]))
        out = dict(case, objective=t["objective"], w=w.tolist(), converged=t["converged"],
                   accepted_steps=t["accepted_steps"],
                   iterations=[(r["accepted"], r["cg_iters"], r["cg_exit"]) for r in t["iterations"]],
                   source="oracle/_ref/libtronref.so (reference sources, proj/src/*.cpp)")
        with open(os.path.join(HERE, case["name"] + ".json"), "w") as f:
            json.dump(out, f, indent=1)
        print(case["name"], t["objective"], len(t["iterations"]))


if __name__ == "__main__":
    main()
