"""LIBSVM ingestion -- mirror of the reference's tron::parse_libsvm
(proj/include/tron/io.hpp, proj/src/io.cpp:54-132) over the native parallel
parser (csrc/ingest.cpp):

``parse_libsvm(source, n_override=0) -> Problem``, ``load_dense(source, n)`` (io.cpp:164-197),
and a binary cache (``save_binary`` / ``load_binary`` / ``load_cached``).

* ``source`` is a path (str / os.PathLike, memory-mapped) or the text itself
  (bytes).
* The semantics are the reference's: 1-based strictly ascending indices; labels
  -1 / 0 / +1 (0 maps to -1); blank lines skipped; C left at 1.0. The feature count
  is the largest index unless ``n_override`` pins it.
* Errors raise ``ParseError`` / ``UnsupportedLabelError`` with the reference's
  message ("line N: ...") and ``.line``.
"""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib
from ._lib import lib
from .tron import Error, FeatureMatrix, Problem


class ParseError(Error):
    """tron::ParseError (error.hpp:28-38)."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(what)
        self.line = line


class UnsupportedLabelError(ParseError):
    """tron::UnsupportedLabelError (error.hpp:40-43)."""


def _check(status: int):
    if status == _lib.OK:
        return
    msg, line = _lib.last_error(), int(lib.tron_gpu_last_error_line())
    if status == _lib.ERR_UNSUPPORTED_LABEL:
        raise UnsupportedLabelError(msg, line)
    if status == _lib.ERR_PARSE:
        raise ParseError(msg, line)
    raise Error(f"status {status}: {msg}")


def _take(h) -> Problem:
    """Copies a native parse handle into a Problem (and frees the handle)."""
    try:
        rows, cols, nnz = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.tron_parsed_sizes(h, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(nnz)))
        dense = ctypes.c_int32()
        _check(lib.tron_parsed_layout(h, ctypes.byref(dense)))
        vals = np.empty(nnz.value)
        y = np.empty(rows.value)
        if dense.value:
            _check(lib.tron_parsed_copy(h, None, None, vals.ctypes.data_as(_lib.PD), y.ctypes.data_as(_lib.PD)))
            return Problem(FeatureMatrix("dense", rows.value, cols.value, vals), y, 1.0)
        ro = np.empty(rows.value + 1, dtype=np.int64)
        ci = np.empty(nnz.value, dtype=np.int32)
        _check(lib.tron_parsed_copy(h, ro.ctypes.data_as(_lib.PI64), ci.ctypes.data_as(_lib.PI32),
                                    vals.ctypes.data_as(_lib.PD), y.ctypes.data_as(_lib.PD)))
        return Problem(FeatureMatrix("csr", rows.value, cols.value, vals, ro, ci), y, 1.0)
    finally:
        lib.tron_parsed_free(h)


def parse_libsvm(source, n_override: int = 0) -> Problem:
    h = ctypes.c_void_p()
    if isinstance(source, (bytes, bytearray, memoryview)):
        data = bytes(source)
        _check(lib.tron_parse_libsvm(data, len(data), n_override, ctypes.byref(h)))
    else:
        _check(lib.tron_parse_libsvm_file(os.fsencode(source), n_override, ctypes.byref(h)))
    return _take(h)


def load_dense(source, n: int) -> Problem:
    """tron::load_dense (io.hpp:31, io.cpp:164-197): "label v1 ... vn" per line,
    exactly n values; labels -1 / 0 / +1; blank lines skipped; the reference's
    ParseError / UnsupportedLabelError messages and line numbers."""
    h = ctypes.c_void_p()
    if isinstance(source, (bytes, bytearray, memoryview)):
        data = bytes(source)
        _check(lib.tron_load_dense(data, len(data), n, ctypes.byref(h)))
    else:
        _check(lib.tron_load_dense_file(os.fsencode(source), n, ctypes.byref(h)))
    return _take(h)


def save_binary(problem: Problem, path) -> None:
    """Writes the TRONBIN1 binary cache of a problem (the layout csrc/ingest.cpp
    reads: magic, layout, rows, cols, nnz as little-endian u64, then the arrays)."""
    X = problem.X
    vals = np.ascontiguousarray(X.values, dtype=np.float64)
    y = np.ascontiguousarray(problem.y, dtype=np.float64)
    tmp = os.fspath(path) + ".tmp"
    with open(tmp, "wb") as f:
        f.write(b"TRONBIN1")
        f.write(struct.pack("<4Q", 1 if X.layout == "dense" else 0, X.rows, X.cols, vals.size))
        if X.layout != "dense":
            f.write(np.ascontiguousarray(X.row_offsets, dtype=np.int64).tobytes())
            f.write(np.ascontiguousarray(X.col_indices, dtype=np.int32).tobytes())
        f.write(vals.tobytes())
        f.write(y.tobytes())
    os.replace(tmp, path)


def load_binary(path) -> Problem:
    """Reads a TRONBIN1 binary cache (native, memory-mapped)."""
    h = ctypes.c_void_p()
    _check(lib.tron_load_binary(os.fsencode(path), ctypes.byref(h)))
    return _take(h)


def load_cached(path, n: int = 0, dense: bool = False, cache=None) -> Problem:
    """parse_libsvm(path, n) (or load_dense(path, n) when dense) through a binary
    cache: ``cache`` (default ``path + '.tronbin'``) is used when it is newer
    than the text, else written after the parse."""
    cache = cache or os.fspath(path) + ".tronbin"
    try:
        if os.path.getmtime(cache) >= os.path.getmtime(path):
            p = load_binary(cache)
            if (p.X.layout == "dense") == dense and (n == 0 or p.X.cols == n):
                return p
    except OSError:
        pass
    h = ctypes.c_void_p()
    if dense:
        _check(lib.tron_load_dense_file(os.fsencode(path), n, ctypes.byref(h)))
    else:
        _check(lib.tron_parse_libsvm_file(os.fsencode(path), n, ctypes.byref(h)))
    try:
        _check(lib.tron_parsed_save_binary(h, os.fsencode(cache)))
    except Error:
        pass  # an unwritable cache location only costs the next parse
    return _take(h)


def write_libsvm(problem: Problem) -> bytes:
    """write_libsvm (io.cpp:134-162): '+1'/'-1', then ' idx:value' (1-based)
    with shortest round-trip values -- test and tooling helper."""
    X = problem.X
    out = []
    for i in range(X.rows):
        parts = ["+1" if problem.y[i] > 0 else "-1"]
        if X.layout == "csr":
            for k in range(X.row_offsets[i], X.row_offsets[i + 1]):
                parts.append(f"{int(X.col_indices[k]) + 1}:{float(X.values[k])!r}")
        else:
            row = X.values[i * X.cols:(i + 1) * X.cols]
            parts.extend(f"{j + 1}:{float(v)!r}" for j, v in enumerate(row) if v != 0.0)
        out.append(" ".join(parts))
    return ("\n".join(out) + "\n").encode() if out else b""
