"""The column-partitioned layout on the device (
DESIGN.md §6.2): two ranks on ONE GPU, each owning half of the columns of one
sparse problem, exchanging over the host data plane (gloo between two
processes) -- per Hv one l-length allreduce of the partial row products, per
CG step scalar allreduces.

  * fun is identical on both ranks and equals the unsharded one; the gradient,
    Hv and preconditioner slices, concatenated, equal the unsharded vectors;
  * the column-layout solve matches the unsharded GPU solve and the reference
    (objective, w, CG counts within the north-star gate); the SVM active set
    (whole on every rank) equals the unsharded one at the same w.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems():
    from paper_2008_03433_b200 import LossKind, synth
    return {
        "lr-cluster": (synth.synth_sparse(3, 1600, 20000, 30), LossKind.Logistic, 1e-4),
        "lr-coop": (synth.synth_sparse(4, 2000, 300001, 40), LossKind.Logistic, 1e-4),
        "svm": (synth.synth_sparse(6, 1400, 5001, 25), LossKind.L2Svm, 1e-4),
    }


def _worker(rank, port, names, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator, synth
    from paper_2008_03433_b200.sharding import column_shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        def allreduce(buf):
            dist.all_reduce(torch.from_numpy(buf))

        out = {}
        probs = _problems()
        for name in names:
            p, loss, eps = probs[name]
            loc, c0 = column_shard(p, rank, WORLD)
            n = p.X.cols
            plan = ExecutionPlan.gpu()
            plan.rank, plan.world = rank, WORLD
            plan.partition, plan.col_begin, plan.global_cols = "columns", c0, n
            plan.host_allreduce = allreduce
            sl = slice(c0, c0 + loc.X.cols)
            w = synth.testgen_random_vector(5, n, 0.05)[sl]
            v = synth.testgen_random_vector(6, n)[sl]
            with make_evaluator(loc, loss, plan) as ev:
                f = ev.eval_candidate(w)
                act_w = ev.candidate_state().active if loss.name == "L2Svm" else None
                ev.commit()
                g, hv, m = ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()
                res = ev.solve(TrustRegionConfig(eps=eps))
                lab, correct = ev.predict(res.w)
            out[name] = dict(f=f, g=g, hv=hv, m=m, w=res.w, obj=res.objective, act_w=act_w,
                             cg=[it.cg_iters for it in res.trace.iterations], lab=lab, correct=correct)
        q.put((rank, out))
    except Exception as e:  # surfaced by the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def colsharded():
    names = list(_problems())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, names, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=900) for _ in range(WORLD))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(WORLD):
        assert isinstance(got[r], dict), got[r]
    return got


@pytest.mark.parametrize("name", list(_problems()))
def test_column_layout_composes(colsharded, ref, name):
    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator, synth
    p, loss, eps = _problems()[name]
    n = p.X.cols
    w = synth.testgen_random_vector(5, n, 0.05)
    v = synth.testgen_random_vector(6, n)
    with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
        f = ev.eval_candidate(w)
        act_w = ev.candidate_state().active if loss.name == "L2Svm" else None
        ev.commit()
        g, hv, m = ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()
        res = ev.solve(TrustRegionConfig(eps=eps))
        lab, correct = ev.predict(res.w)
    a, b = colsharded[0][name], colsharded[1][name]
    assert a["f"] == b["f"] and rel_err(a["f"], f) <= 1e-13
    for k, full in (("g", g), ("hv", hv), ("m", m)):
        assert rel_err(np.concatenate([a[k], b[k]]), full) <= 1e-12, k
    if act_w is not None:
        assert np.array_equal(a["act_w"], act_w) and np.array_equal(b["act_w"], act_w)
    w_col = np.concatenate([a["w"], b["w"]])
    assert a["obj"] == b["obj"] and a["cg"] == b["cg"]
    assert rel_err(a["obj"], res.objective) <= 1e-10 and rel_err(w_col, res.w) <= 1e-6
    cg_full = [it.cg_iters for it in res.trace.iterations]
    assert len(a["cg"]) == len(cg_full) and all(abs(x - y) <= 1 for x, y in zip(a["cg"], cg_full))
    w_ref, t_ref = ref.solve(p, 0 if loss.name == "Logistic" else 1, TrustRegionConfig(eps=eps))
    assert rel_err(a["obj"], t_ref["objective"]) <= 1e-6 and rel_err(w_col, w_ref) <= 1e-6
    assert np.array_equal(a["lab"], b["lab"]) and abs(a["correct"] - correct) <= 0.001 * p.X.rows
