"""Two real row shards of one problem on ONE GPU.

NCCL refuses two ranks on the same device, so the shards here use the host
data plane (ExecutionPlan.host_allreduce -> a gloo allreduce between two
processes): every per-call partial -- the loss sums and |I|, the gradient /
Hv / preconditioner n-vectors -- crosses the same Comm::allreduce_sum the
NCCL path uses.  With two shards, row_begin, the RAW epilogues, the
replicated CG and the rank-local active sets all run for real:

  * fun / grad / Hv / precond of the sharded evaluator equal the unsharded
    one (different summation split: <= 1e-13 relative);
  * the sharded solve matches the unsharded GPU solve and the reference;
  * the rank-ordered concatenation of the local active sets is the global
    ascending IndexSet; every rank ends with bitwise-identical w.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu
WORLD = 2
# solve tolerance per problem (the dense L2-SVM to a tighter eps)
EPS = {"dense-svm": 1e-6}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems():
    from paper_2008_03433_b200 import LossKind, synth
    return {
        "sparse-lr-cluster": (synth.synth_sparse(3, 1601, 20000, 30), LossKind.Logistic),
        "sparse-lr-coop": (synth.synth_sparse(4, 2001, 300000, 40), LossKind.Logistic),
        "sparse-svm": (synth.synth_sparse(6, 1401, 5000, 25), LossKind.L2Svm),
        # equal column scales: a well-conditioned dense L2-SVM (the 2-decade
        # SYNTH scales make w flat to 1e-6 at any reachable eps)
        "dense-svm": (synth.synth_dense(1, 40001, 40, decades=0.0), LossKind.L2Svm),
        "dense-lr": (synth.testgen_dense_problem(2001, 401, 20, 1.0), LossKind.Logistic),
    }


def _worker(rank, port, names, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator, synth
    from paper_2008_03433_b200.sharding import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # every sharded solve compares the ranks' w / f / delta after each outer iteration
    os.environ["TRON_B200_CHECK_REPLICAS"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        def allreduce(buf):
            t = torch.from_numpy(buf)  # shares the pinned staging buffer
            dist.all_reduce(t)

        out = {}
        probs = _problems()
        for name in names:
            p, loss = probs[name]
            loc, b = shard(p, rank, WORLD)
            plan = ExecutionPlan.gpu()
            plan.rank, plan.world, plan.row_begin, plan.global_rows = rank, WORLD, b, p.X.rows
            plan.host_allreduce = allreduce
            n = p.X.cols
            w = synth.testgen_random_vector(5, n, 0.05)
            v = synth.testgen_random_vector(6, n)
            with make_evaluator(loc, loss, plan) as ev:
                f = ev.eval_candidate(w)
                act_w = ev.candidate_state().active if loss.name == "L2Svm" else None
                ev.commit()
                g = ev.gradient()
                hv = ev.hessian_vec(v)
                m = ev.precond_diagonal()
                res = ev.solve(TrustRegionConfig(eps=EPS.get(name, 1e-4)))
                act = ev.committed_state().active if loss.name == "L2Svm" else None
                csum = ev.replica_checksum()
            out[name] = dict(f=f, g=g, hv=hv, m=m, w=res.w, obj=res.objective,
                             cg=[it.cg_iters for it in res.trace.iterations], act=act,
                             act_w=act_w, csum=csum)
        q.put((rank, out))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    names = list(_problems())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, names, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=600) for _ in range(WORLD))
    for pr in procs:
        pr.join(timeout=60)
    for r in range(WORLD):
        assert isinstance(got[r], dict), got[r]
    return got


@pytest.mark.parametrize("name", list(_problems()))
def test_two_shards_compose(sharded, ref, name):
    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator, synth
    p, loss = _problems()[name]
    n = p.X.cols
    w = synth.testgen_random_vector(5, n, 0.05)
    v = synth.testgen_random_vector(6, n)
    with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
        f = ev.eval_candidate(w)
        act_w = ev.candidate_state().active if loss.name == "L2Svm" else None
        ev.commit()
        g, hv, m = ev.gradient(), ev.hessian_vec(v), ev.precond_diagonal()
        res = ev.solve(TrustRegionConfig(eps=EPS.get(name, 1e-4)))
        act = ev.committed_state().active if loss.name == "L2Svm" else None
    a, b = sharded[0][name], sharded[1][name]
    for r in (a, b):  # every rank holds the same replicated result
        assert rel_err(r["f"], f) <= 1e-13
        assert rel_err(r["g"], g) <= 1e-13
        assert rel_err(r["hv"], hv) <= 1e-13
        assert rel_err(r["m"], m) <= 1e-13
    assert np.array_equal(a["w"].view(np.uint64), b["w"].view(np.uint64))
    assert np.array_equal(a["csum"], b["csum"])  # (and the per-iteration checks passed)
    assert a["obj"] == b["obj"] and a["cg"] == b["cg"]
    assert rel_err(a["obj"], res.objective) <= 1e-10
    assert rel_err(a["w"], res.w) <= 1e-7
    assert all(abs(x - y) <= 1 for x, y in zip(a["cg"], [it.cg_iters for it in res.trace.iterations]))
    w_ref, t_ref = ref.solve(p, 0 if loss.name == "Logistic" else 1, TrustRegionConfig(eps=EPS.get(name, 1e-4)))
    assert rel_err(a["obj"], t_ref["objective"]) <= 1e-6 and rel_err(a["w"], w_ref) <= 1e-6
    if act is not None:
        # same w => same margins row by row (sequential row dots): the shards'
        # local sets, concatenated in rank order, are the global IndexSet
        assert np.array_equal(np.concatenate([a["act_w"], b["act_w"]]), act_w)
        glob = np.concatenate([a["act"], b["act"]])
        assert np.all(np.diff(glob) > 0) and abs(glob.size - act.size) <= 0.001 * act.size


def test_replica_checksum_sees_one_ulp():
    """The replica checksum (tron_gpu_replica_checksum) of the committed w: equal
    for equal w, different after a one-ulp change of one coordinate."""
    from paper_2008_03433_b200 import ExecutionPlan, make_evaluator, synth
    p, loss = _problems()["sparse-svm"]
    w = synth.testgen_random_vector(5, p.X.cols, 0.05)
    w2 = w.copy()
    w2[17] = np.nextafter(w2[17], np.inf)
    with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
        sums = []
        for x in (w, w, w2):
            ev.eval_candidate(x)
            ev.commit()
            sums.append(ev.replica_checksum())
    assert np.array_equal(sums[0], sums[1])
    assert not np.array_equal(sums[0], sums[2])
    assert all(0 <= h < 65536 and h == int(h) for h in sums[0])
