"""SYNTH-v1 generators against a sequential pure-Python
restatement of the pseudo-code: the library generates dense rows and labels
in parallel ranges (splitmix64 is seekable) and samples Zipf columns through
a guide table -- both must reproduce the sequential stream bit for bit."""
import bisect
import math

import numpy as np
import pytest

from conftest import ROOT  # noqa: F401  (puts the repo on sys.path)

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


class Rng:  # proj/tests/support/testgen.hpp:14-36
    def __init__(self, seed):
        self.state = seed & M64

    def next_u64(self):
        self.state = (self.state + GOLDEN) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def unit(self):
        return float(self.next_u64() >> 11) * 2.0 ** -53


def labels(rng, rows, n, flip):
    w = [-1.0 + 2.0 * rng.unit() for _ in range(n)]
    y = []
    for row in rows:  # row = [(col, val)]
        s = 0.0
        for c, v in row:
            s += v * w[c]
        lab = 1.0 if s >= 0.0 else -1.0
        if rng.unit() < flip:
            lab = -lab
        y.append(lab)
    return y


def py_sparse(seed, l, n, k, s=1.0, flip=0.1):
    rng = Rng(seed)
    acc, cdf = 0.0, []
    for j in range(n):
        acc += math.pow(j + 1, -s)
        cdf.append(acc)
    cdf = [c / cdf[-1] for c in cdf]
    rows = []
    for _ in range(l):
        row = []
        while len(row) < k:
            c = min(bisect.bisect_left(cdf, rng.unit()), n - 1)  # std::lower_bound
            if c not in row:
                row.append(c)
        row.sort()
        vals, ss = [], 0.0
        for _c in row:
            v = 1e-3 + rng.unit()
            vals.append(v)
            ss += v * v
        inv = 1.0 / math.sqrt(ss)
        rows.append([(c, v * inv) for c, v in zip(row, vals)])
    return rows, labels(rng, rows, n, flip)


def py_dense(seed, l, n, decades=2.0, rho=0.0, flip=0.1):
    rng = Rng(seed)
    sc = [math.pow(10.0, -decades / 2 + decades * j / (n - 1)) for j in range(n)]
    rows = []
    for _ in range(l):
        g = 2 * rng.unit() - 1
        rows.append([(j, sc[j] * (rho * g + (1 - rho) * (2 * rng.unit() - 1))) for j in range(n)])
    return rows, labels(rng, rows, n, flip)


@pytest.mark.parametrize("seed,l,n,k", [(1, 120, 3000, 37), (9, 40, 50, 12), (5, 64, 700, 1)])
def test_synth_sparse_matches_sequential_stream(seed, l, n, k):
    from paper_2008_03433_b200 import synth
    p = synth.synth_sparse(seed, l, n, k)
    rows, y = py_sparse(seed, l, n, k)
    assert np.array_equal(p.X.row_offsets, np.arange(l + 1) * k)
    assert np.array_equal(p.X.col_indices, np.array([c for r in rows for c, _ in r], np.int32))
    assert np.array_equal(p.X.values, np.array([v for r in rows for _, v in r]))
    assert np.array_equal(p.y, np.array(y))


@pytest.mark.parametrize("seed,l,n", [(1, 300, 40), (3, 40001, 5)])
def test_synth_dense_matches_sequential_stream(seed, l, n):
    from paper_2008_03433_b200 import synth
    p = synth.synth_dense(seed, l, n)
    rows, y = py_dense(seed, l, n)
    assert np.array_equal(p.X.values, np.array([v for r in rows for _, v in r]))
    assert np.array_equal(p.y, np.array(y))


# The reference arm of bench.py generates SYNTH-v1 inside oracle/_ref
# (ref_shim.cpp, the reference's own testgen::Rng) so it never maps the product
# library; both generators must produce the same bits.
@pytest.mark.parametrize("seed,l,n,k", [(1, 300, 5000, 17), (4, 64, 200, 200), (7, 500, 40000, 3)])
def test_reference_side_synth_sparse_matches_product(ref, seed, l, n, k):
    from paper_2008_03433_b200 import synth
    p = synth.synth_sparse(seed, l, n, k)
    ro, ci, vals, y = ref.synth_sparse(seed, l, n, k)
    assert np.array_equal(ro, p.X.row_offsets)
    assert np.array_equal(ci, p.X.col_indices)
    assert np.array_equal(vals.view(np.uint64), p.X.values.view(np.uint64))
    assert np.array_equal(y, p.y)


@pytest.mark.parametrize("seed,l,n", [(1, 40000, 40), (3, 777, 7), (9, 5, 64)])
def test_reference_side_synth_dense_matches_product(ref, seed, l, n):
    from paper_2008_03433_b200 import synth
    p = synth.synth_dense(seed, l, n)
    vals, y = ref.synth_dense(seed, l, n)
    assert np.array_equal(vals.view(np.uint64), p.X.values.view(np.uint64))
    assert np.array_equal(y, p.y)


def test_reference_predict_matches_sign_of_sequential_dot(ref):
    from paper_2008_03433_b200 import synth
    p = synth.synth_dense(2, 3000, 40)
    w = synth.testgen_random_vector(5, 40, 1.0)
    X = p.X
    X.y = p.y
    labels, correct = ref.predict(X, w)
    Xd = X.values.reshape(3000, 40)
    want = np.empty(3000)
    for i in range(3000):
        s = 0.0
        for j in range(40):
            s += Xd[i, j] * w[j]
        want[i] = -1.0 if s < 0.0 else 1.0
    assert np.array_equal(labels, want)
    assert correct == int(np.sum(want == p.y))
