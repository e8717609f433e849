"""CPU: bench.py's contract pieces that need no GPU -- the reference arm runs
the reference through oracle/_ref only (never mapping the product library),
both arms print the same config dict, and the SYNTH-v1 shape table matches
the product's."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_shape_table_matches_product():
    from paper_2008_03433_b200 import synth
    assert bench.SHAPES == synth.SHAPES


def test_config_identical_for_both_arms():
    a = bench.workload_config("P1", 0.01)
    assert a == bench.workload_config("P1", 0.01)
    assert a["workload"] == "P1" and a["l"] == 23_000_000 and a["n"] == 40
    assert a["nnz"] == 23_000_000 * 40


def test_reference_arm_never_maps_product_library(ref, tmp_path):
    code = (
        "import runpy, sys, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'R1', '--rows', '3000', "
        "'--steps', '2', '--warmup', '1']\n"
        "try:\n"
        f"    runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('MAPS', json.dumps(sorted({l.split()[-1] for l in maps.splitlines() if l.endswith('.so')})))\n"
    )
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=str(tmp_path),
                         timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    line = json.loads(lines[-1])
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["config"] == bench.workload_config("R1", 0.01, 3000)
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    maps = json.loads([l for l in out.stdout.splitlines() if l.startswith("MAPS")][0][5:])
    assert not [m for m in maps if "libtron_b200" in m], maps
    assert [m for m in maps if m.endswith("oracle/_ref/libtronref.so")]


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_no_collective_after_the_ranks_part():
    """N > 1: every collective of the own arm happens before rank 0 parts from
    the others (they wait at the closing barrier).  A max_over_ranks inside
    rank 0's JSON line once deadlocked every multi-rank run; this reads main()'s
    source after the split and finds no collective there."""
    import ast
    import inspect
    import bench
    src = inspect.getsource(bench.main)
    tree = ast.parse(src)
    fn = tree.body[0]
    # the statement `if rank != 0: ... return 0` in main's body
    split = next(i for i, st in enumerate(fn.body)
                 if isinstance(st, ast.If) and ast.unparse(st.test).replace(" ", "") == "rank!=0")
    def collectives(stmts):
        mod = ast.Module(body=stmts, type_ignores=[])
        names = [ast.unparse(n.func) for n in ast.walk(mod) if isinstance(n, ast.Call)]
        return sorted(c for c in names if c in ("max_over_ranks", "barrier") or c.startswith("dist."))
    # rank 0 after the split: only its side of the closing barrier, the same
    # calls the other ranks make in the split's branch
    assert collectives(fn.body[split + 1:]) == collectives(fn.body[split].body)
    assert collectives(fn.body[split].body) == ["barrier", "dist.destroy_process_group"]
