"""LIBSVM ingestion (§8(f) item 3): the native parallel parser against the
reference's own parse_libsvm (proj/src/io.cpp:54-132, compiled into
oracle/_ref) on the same bytes -- identical arrays, labels and dimension, and
the same error class, message and line for malformed input, including texts
long enough to be split across parser ranges (line numbers must follow the
file, and the first error in file order must win)."""
import numpy as np
import pytest

from paper_2008_03433_b200 import io, synth


def both(ref, text, n_override=0):
    try:
        got = io.parse_libsvm(text, n_override)
        mine = ("ok", got)
    except io.UnsupportedLabelError as e:
        mine = ("label", (str(e), e.line))
    except io.ParseError as e:
        mine = ("parse", (str(e), e.line))
    return mine, ref.parse_libsvm(text, n_override)


def assert_same(ref, text, n_override=0):
    mine, theirs = both(ref, text, n_override)
    assert mine[0] == theirs[0], (mine, theirs)
    if mine[0] != "ok":
        assert mine[1] == theirs[1]
        return mine
    p = mine[1]
    ro, ci, vals, y, n = theirs[1]
    assert p.X.cols == n and p.X.rows == y.size
    assert np.array_equal(p.X.row_offsets, ro)
    assert np.array_equal(p.X.col_indices, ci)
    assert np.array_equal(p.X.values.view(np.uint64), vals.view(np.uint64))  # bit-identical
    assert np.array_equal(p.y, y)
    return mine


@pytest.fixture(scope="module")
def big_text():
    # ~15 MB: several parser ranges
    return io.write_libsvm(synth.synth_sparse(5, 20000, 50000, 30))


def test_roundtrip_and_reference_parity_multi_range(ref, big_text):
    kind, p = assert_same(ref, big_text)
    q = synth.synth_sparse(5, 20000, 50000, 30)
    assert np.array_equal(p.X.values, q.X.values) and np.array_equal(p.y, q.y)


@pytest.mark.parametrize("text", [
    b"",
    b"\n\n",
    b"+1 1:0.5 3:2\n-1 2:1e-3\n0 4:7\n",                      # label 0 -> -1
    b"1 1:1\r\n-1 2:2\r\n\r\n+1\r\n",                         # CRLF, blank, feature-less row
    b"  \t+1\t+1:+0.25  2:-3\n-1 5:1",                        # tabs, '+' signs, no final newline
    b"-1 1:1.7976931348623157e308 2:4.9e-324 3:-0.0\n",       # extremes, negative zero
    b"+1 2147483647:1\n",                                     # largest index
])
def test_formats(ref, text):
    assert_same(ref, text)


@pytest.mark.parametrize("text", [
    b"+1 1:1\n2 2:2\n",                  # unsupported label
    b"+1 1:1\nabc 2:2\n",                # bad label
    b"+1x 1:1\n",                        # trailing characters after the label
    b"+1 0:1\n",                         # index not 1-based
    b"+1 3:1 2:1\n",                     # not strictly ascending
    b"+1 3:1 3:1\n",                     # duplicate
    b"+1 1 2:1\n",                       # missing ':'
    b"+1 1:1x\n",                        # trailing characters after a value
    b"+1 1:1e999\n",                     # outside the finite range
    b"+1 1:nan\n",
    b"+1 2147483648:1\n",                # index too large
    b"+1 a:1\n",                         # bad index
    b"+1 1:\n",                          # missing value
])
def test_errors_match_reference(ref, text):
    kind, (msg, line) = assert_same(ref, text)
    assert kind in ("parse", "label") and line >= 1


def test_n_override(ref):
    text = b"+1 1:1 4:2\n-1 2:3\n"
    kind, p = assert_same(ref, text, 10)
    assert p.X.cols == 10
    kind, (msg, line) = assert_same(ref, text, 3)
    assert kind == "parse" and line == 0 and "exceeds the requested dimension" in msg


def test_first_error_in_file_order_across_ranges(ref, big_text):
    lines = big_text.split(b"\n")
    n = len(lines)
    late = list(lines)
    late[n - 10] = b"+1 5:1 4:1"            # in the last range
    kind, (msg, line) = assert_same(ref, b"\n".join(late))
    assert kind == "parse" and line == n - 9
    both_err = list(late)
    both_err[n // 3] = b"7 1:1"             # an earlier error in an earlier range wins
    kind, (msg, line) = assert_same(ref, b"\n".join(both_err))
    assert kind == "label" and line == n // 3 + 1


def test_parse_file_matches_bytes(tmp_path, big_text):
    f = tmp_path / "x.svm"
    f.write_bytes(big_text)
    a, b = io.parse_libsvm(str(f)), io.parse_libsvm(big_text)
    assert np.array_equal(a.X.values, b.X.values) and np.array_equal(a.X.row_offsets, b.X.row_offsets)


# ---- load_dense (io.cpp:164-197) ---------------------------------------------

def dense_both(ref, text, n):
    try:
        p = io.load_dense(text, n)
        mine = ("ok", p)
    except io.UnsupportedLabelError as e:
        mine = ("label", (str(e), e.line))
    except io.ParseError as e:
        mine = ("parse", (str(e), e.line))
    theirs = ref.load_dense(text, n)
    assert mine[0] == theirs[0], (mine, theirs)
    if mine[0] != "ok":
        assert mine[1] == theirs[1]
        return mine
    vals, y = theirs[1]
    p = mine[1]
    assert p.X.layout == "dense" and p.X.cols == n and p.X.rows == y.size
    assert np.array_equal(p.X.values.view(np.uint64), vals.view(np.uint64))
    assert np.array_equal(p.y, y)
    return mine


@pytest.mark.parametrize("text,n", [
    (b"+1 1 2\n-1 3 4\n", 2),
    (b"0 1e-3 -2.5\r\n\n  \t\n1\t7 8\n", 2),      # CRLF, blank lines, tabs, label 0
    (b"1 1.7976931348623157e308 -0.0\n", 2),      # extremes, no final newline below
    (b"-1 0 0 0", 3),
    (b"", 4),                                      # empty input: 0 x 4
    (b"1 1 2 3\n", 2),                             # more than n values
    (b"1 1\n", 2),                                 # fewer
    (b"1 1 2\n-1 3 x\n", 2),                       # bad value, line 2
    (b"1 1 2\n2 3 4\n", 2),                        # unsupported label
    (b"1 1e999 2\n", 2),                           # out of range
    (b"1x 1 2\n", 2),                              # label glued to garbage
    (b"1 +3 4\n", 2),                              # '+' on a value
])
def test_load_dense_matches_reference(ref, text, n):
    dense_both(ref, text, n)


def test_load_dense_multi_range_and_late_error(ref):
    p = synth.synth_dense(3, 60000, 12)
    rows = p.X.values.reshape(-1, 12)
    lines = [(b"+1 " if y > 0 else b"-1 ") + b" ".join(repr(float(v)).encode() for v in r)
             for r, y in zip(rows, p.y)]
    text = b"\n".join(lines) + b"\n"
    kind, q = dense_both(ref, text, 12)
    assert np.array_equal(q.X.values, p.X.values) and np.array_equal(q.y, p.y)
    bad = b"\n".join(lines[:50000] + [lines[50000] + b" 9"] + lines[50001:]) + b"\n"
    kind, (msg, line) = dense_both(ref, bad, 12)
    assert kind == "parse" and line == 50001


# ---- binary cache --------------------------------------------------------------

@pytest.mark.parametrize("dense", [False, True])
def test_binary_cache_roundtrip(tmp_path, dense):
    p = synth.synth_dense(2, 3000, 9) if dense else synth.synth_sparse(4, 3000, 7000, 15)
    path = tmp_path / "x.tronbin"
    io.save_binary(p, path)
    q = io.load_binary(path)
    assert q.X.layout == p.X.layout and (q.X.rows, q.X.cols) == (p.X.rows, p.X.cols)
    assert np.array_equal(q.X.values.view(np.uint64), p.X.values.view(np.uint64))
    assert np.array_equal(q.y, p.y)
    if not dense:
        assert np.array_equal(q.X.row_offsets, p.X.row_offsets)
        assert np.array_equal(q.X.col_indices, p.X.col_indices)
    (tmp_path / "bad.tronbin").write_bytes(b"TRONBIN1" + b"\0" * 10)
    with pytest.raises(io.ParseError):
        io.load_binary(tmp_path / "bad.tronbin")


def test_load_cached_writes_then_reuses(tmp_path, big_text):
    src = tmp_path / "data.svm"
    src.write_bytes(big_text)
    a = io.load_cached(src)
    cache = tmp_path / "data.svm.tronbin"
    assert cache.exists()
    b = io.load_cached(src)  # from the cache
    for p in (a, b):
        q = io.parse_libsvm(big_text)
        assert np.array_equal(p.X.values, q.X.values) and np.array_equal(p.X.col_indices, q.X.col_indices)
        assert np.array_equal(p.X.row_offsets, q.X.row_offsets) and p.X.cols == q.X.cols
    d = tmp_path / "d.txt"
    d.write_bytes(b"1 1 2\n-1 3 4\n")
    p = io.load_cached(d, n=2, dense=True)
    assert p.X.layout == "dense" and np.array_equal(io.load_cached(d, n=2, dense=True).X.values, [1, 2, 3, 4])
