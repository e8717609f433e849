"""CPU: the C-ABI library loads, exports every symbol include/tron_b200.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tron_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(tron_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_evaluator_surface():
    names = declared_functions()
    for must in ("tron_gpu_create_csr", "tron_gpu_create_dense", "tron_gpu_eval_candidate",
                 "tron_gpu_commit", "tron_gpu_gradient", "tron_gpu_hessian_vec",
                 "tron_gpu_precond_diagonal", "tron_gpu_truncated_cg", "tron_gpu_solve",
                 "tron_gpu_destroy", "tron_gpu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2008_03433_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers them all
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound


def test_struct_layouts_match_header():
    from paper_2008_03433_b200 import _lib
    assert ctypes.sizeof(_lib.tron_config) == 8 * 10 + 8
    assert ctypes.sizeof(_lib.tron_iteration) == 4 * 8 + 8 + 8
    assert ctypes.sizeof(_lib.tron_ledger) == 7 * 8
    # ... reference_order (int32 + pad), host_allreduce + its user pointer,
    # out_of_core (int32 + pad), stream_block_rows, partition (int32 + pad), col_begin, global_cols
    assert ctypes.sizeof(_lib.tron_gpu_options) == 4 + 4 + 8 + 4 + 4 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8


def test_defaults_mirror_reference():
    from paper_2008_03433_b200 import TrustRegionConfig, _lib
    c = _lib.tron_config()
    _lib.lib.tron_gpu_default_config(ctypes.byref(c))
    t = TrustRegionConfig()
    for f in ("eps", "max_outer_iters", "max_cg_iters", "sigma0", "eta1", "eta2", "gamma1",
              "gamma2", "gamma3", "cg_tol"):
        assert getattr(c, f) == getattr(t, f)
    o = _lib.tron_gpu_options()
    _lib.lib.tron_gpu_default_options(ctypes.byref(o))
    assert o.gathered_budget_bytes == 2 << 30 and o.svm_strategy == _lib.SVM_INDIRECT and o.world == 1


def test_no_silent_cpu_fallback():
    from paper_2008_03433_b200 import DeviceError, ExecutionPlan, LossKind, make_evaluator, synth
    from paper_2008_03433_b200.tron import device_count
    if device_count() > 0:
        pytest.skip("a GPU is present")
    p = synth.testgen_dense_problem(1, 10, 3, 1.0)
    with pytest.raises(DeviceError):
        make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu())


def test_null_context_is_an_argument_error():
    from paper_2008_03433_b200 import _lib
    f = ctypes.c_double()
    w = np.zeros(3)
    st = _lib.lib.tron_gpu_eval_candidate(None, w.ctypes.data_as(_lib.PD), ctypes.byref(f))
    assert st == _lib.ERR_ARGUMENT and "null" in _lib.last_error()


def test_validation_happens_before_device_use():
    """Bad inputs raise the reference's error classes even without a GPU."""
    from paper_2008_03433_b200 import (BoundsError, DimensionError, ExecutionPlan, FeatureMatrix,
                                       LossKind, Problem, make_evaluator)
    bad_label = Problem(FeatureMatrix.dense(2, 1, [1.0, 2.0]), np.array([1.0, 3.0]), 1.0)
    with pytest.raises(DimensionError):
        make_evaluator(bad_label, LossKind.Logistic, ExecutionPlan.gpu())
    bad_col = Problem(FeatureMatrix("csr", 1, 2, np.array([1.0]), np.array([0, 1], np.int64),
                                    np.array([5], np.int32)), np.array([1.0]), 1.0)
    with pytest.raises(BoundsError):
        make_evaluator(bad_col, LossKind.Logistic, ExecutionPlan.gpu())


def test_quadratic_model_kats():  # test_tron.cpp:44-51 on the host mirror
    from paper_2008_03433_b200 import quadratic_model
    hv = lambda d: np.asarray(d, dtype=np.float64).copy()  # identity Hessian
    assert quadratic_model([1.0, 0.0], hv, [0.0, 0.0]) == 0.0
    assert quadratic_model([1.0, 0.0], hv, [-1.0, 0.0]) == -0.5
    g, d = np.array([3.0, -4.0]), np.array([-3.0, 4.0])
    assert abs(quadratic_model(g, hv, d) - (-g @ g / 2.0)) <= 1e-15 * (g @ g / 2.0)
