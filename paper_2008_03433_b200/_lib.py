"""ctypes binding of libtron_b200.so (the C ABI in include/tron_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2008_03433_b200/csrc``).  There is no fallback: if the
shared object is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# TRON_B200_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("TRON_B200_LIB") or os.path.join(HERE, "libtron_b200.so")

# tron_status
OK, ERR_DIMENSION, ERR_BOUNDS, ERR_STRATEGY, ERR_BUDGET, ERR_NUMERICAL, ERR_LOGIC, ERR_CUDA, \
    ERR_NCCL, ERR_OOM, ERR_ARGUMENT, ERR_PARSE, ERR_UNSUPPORTED_LABEL = range(13)
LOSS_LOGISTIC, LOSS_L2SVM = 0, 1
SVM_GATHERED, SVM_INDIRECT, SVM_AUTO = 0, 1, 2
SOLVE_DEVICE, SOLVE_HOST_CG = 0, 1
PARTITION_ROWS, PARTITION_COLUMNS = 0, 1
MODE_GRAM, MODE_OUT_OF_CORE, MODE_COLUMNS, MODE_DEVICE_LOOP, MODE_SHARDED, MODE_GRAM_DELTA = 1, 2, 4, 8, 16, 32


class tron_config(ctypes.Structure):
    _fields_ = [("eps", c_double), ("max_outer_iters", c_uint64), ("max_cg_iters", c_uint64),
                ("sigma0", c_double), ("eta1", c_double), ("eta2", c_double),
                ("gamma1", c_double), ("gamma2", c_double), ("gamma3", c_double),
                ("cg_tol", c_double), ("use_preconditioner", c_int32), ("solve_mode", c_int32)]


class tron_iteration(ctypes.Structure):
    _fields_ = [("f_candidate", c_double), ("gradient_norm", c_double), ("delta", c_double),
                ("sigma", c_double), ("accepted", c_int32), ("cg_exit", c_int32),
                ("cg_iters", c_uint64)]


class tron_solve_info(ctypes.Structure):
    _fields_ = [("f_initial", c_double), ("gradient_norm_initial", c_double),
                ("objective", c_double), ("accepted_steps", c_uint64),
                ("gradient_materializations", c_uint64), ("objective_evaluations", c_uint64),
                ("n_iterations", c_uint64), ("converged", c_int32), ("status", c_int32),
                ("hessian_products", c_uint64), ("device_ms", c_double)]


class tron_ledger(ctypes.Structure):
    _fields_ = [("bulk_handoffs", c_uint64), ("scalar_returns", c_uint64),
                ("gradient_materializations", c_uint64), ("concealed_vector_returns", c_uint64),
                ("margin_passes", c_uint64), ("gathered_submatrix_bytes", c_uint64),
                ("index_set_bytes", c_uint64)]


class tron_gpu_options(ctypes.Structure):
    _fields_ = [("device", c_int32), ("svm_strategy", c_int32),
                ("gathered_budget_bytes", c_uint64), ("rank", c_int32), ("world", c_int32),
                ("nccl_unique_id", c_void_p), ("row_begin", c_uint64), ("global_rows", c_uint64),
                ("reference_order", c_int32), ("host_allreduce", c_void_p),
                ("host_allreduce_user", c_void_p), ("out_of_core", c_int32),
                ("stream_block_rows", c_uint64), ("partition", c_int32), ("col_begin", c_uint64),
                ("global_cols", c_uint64)]


# void (*)(void* user, double* buf, uint64_t count): a host allreduce (sum, in place)
HOST_ALLREDUCE = ctypes.CFUNCTYPE(None, c_void_p, POINTER(c_double), c_uint64)


PD = POINTER(c_double)
PI64 = POINTER(c_int64)
PI32 = POINTER(c_int32)
PU64 = POINTER(c_uint64)

# (name, restype, argtypes) for every symbol declared in include/tron_b200.h
SIGNATURES = [
    ("tron_gpu_default_config", None, [POINTER(tron_config)]),
    ("tron_gpu_default_options", None, [POINTER(tron_gpu_options)]),
    ("tron_gpu_last_error", c_char_p, []),
    ("tron_gpu_device_count", c_int, [POINTER(c_int)]),
    ("tron_gpu_create_csr", c_int, [c_int, c_uint64, c_uint64, PI64, PI32, PD, PD, c_double,
                                    POINTER(tron_gpu_options), POINTER(c_void_p)]),
    ("tron_gpu_create_dense", c_int, [c_int, c_uint64, c_uint64, PD, PD, c_double,
                                      POINTER(tron_gpu_options), POINTER(c_void_p)]),
    ("tron_gpu_destroy", None, [c_void_p]),
    ("tron_gpu_dimension", c_int, [c_void_p, PU64]),
    ("tron_gpu_eval_candidate", c_int, [c_void_p, PD, PD]),
    ("tron_gpu_commit", c_int, [c_void_p, PD]),
    ("tron_gpu_gradient", c_int, [c_void_p, PD]),
    ("tron_gpu_hessian_vec", c_int, [c_void_p, PD, PD]),
    ("tron_gpu_precond_diagonal", c_int, [c_void_p, PD]),
    ("tron_gpu_quadratic_model", c_int, [c_void_p, PD, PD]),
    ("tron_gpu_replica_checksum", c_int, [c_void_p, PD]),
    ("tron_gpu_state_lr", c_int, [c_void_p, c_int, PD, PD, PD]),
    ("tron_gpu_state_svm", c_int, [c_void_p, c_int, PD, PI64, c_uint64, PU64]),
    ("tron_gpu_truncated_cg", c_int, [c_void_p, c_double, POINTER(tron_config), PD, PI32, PU64,
                                      PD]),
    ("tron_gpu_solve", c_int, [c_void_p, POINTER(tron_config), PD, PD, POINTER(tron_solve_info),
                               POINTER(tron_iteration), c_uint64]),
    ("tron_gpu_predict", c_int, [c_void_p, PD, PD, PU64]),
    ("tron_gpu_ledger", c_int, [c_void_p, POINTER(tron_ledger)]),
    ("tron_gpu_reset_ledger", c_int, [c_void_p]),
    ("tron_gpu_bench_kernels", c_int, [c_void_p, c_int, c_int, PD]),
    ("tron_gpu_memory_bytes", c_int, [c_void_p, PU64]),
    ("tron_gpu_mode", c_int, [c_void_p, POINTER(ctypes.c_uint32)]),
    ("tron_gpu_launch_count", c_int, [c_void_p, PU64]),
    ("tron_gpu_synchronize", c_int, [c_void_p]),
    ("tron_gpu_nccl_unique_id", c_int, [c_void_p]),
    ("tron_testgen_dense_problem", None, [c_uint64, c_size_t, c_size_t, c_double, PD, PD]),
    ("tron_testgen_dense_problem_scaled", None, [c_uint64, c_size_t, c_size_t, c_double, c_double,
                                                 PD, PD]),
    ("tron_testgen_sparse_problem", c_size_t, [c_uint64, c_size_t, c_size_t, c_double, c_double,
                                               PI64, PI32, PD, PD]),
    ("tron_testgen_random_vector", None, [c_uint64, c_size_t, c_double, PD]),
    ("tron_testgen_random_index_set", c_size_t, [c_uint64, c_size_t, c_double, PI64]),
    ("tron_synth_sparse", c_int, [c_uint64, c_size_t, c_size_t, c_size_t, c_double, c_double, PI64,
                                  PI32, PD, PD]),
    ("tron_synth_dense", c_int, [c_uint64, c_size_t, c_size_t, c_double, c_double, c_double, PD,
                                 PD]),
    ("tron_parse_libsvm", c_int, [ctypes.c_char_p, c_uint64, c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    ("tron_parse_libsvm_file", c_int, [ctypes.c_char_p, c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    ("tron_parsed_sizes", c_int, [ctypes.c_void_p, ctypes.POINTER(c_uint64), ctypes.POINTER(c_uint64),
                                  ctypes.POINTER(c_uint64)]),
    ("tron_parsed_copy", c_int, [ctypes.c_void_p, PI64, PI32, PD, PD]),
    ("tron_parsed_free", None, [ctypes.c_void_p]),
    ("tron_load_dense", c_int, [c_char_p, c_uint64, c_uint64, POINTER(c_void_p)]),
    ("tron_load_dense_file", c_int, [c_char_p, c_uint64, POINTER(c_void_p)]),
    ("tron_parsed_layout", c_int, [c_void_p, PI32]),
    ("tron_parsed_save_binary", c_int, [c_void_p, c_char_p]),
    ("tron_load_binary", c_int, [c_char_p, POINTER(c_void_p)]),
    ("tron_gpu_last_error_line", c_uint64, []),
    ("tron_host_alloc", c_void_p, [c_uint64]),
    ("tron_host_free", None, [c_void_p]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def pinned_array(n: int, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked memory from the library's pool (returned to
    the pool when the array is garbage collected); device results land in it
    with a plain DMA."""
    dt = np.dtype(dtype)
    nbytes = max(int(n) * dt.itemsize, 1)
    ptr = lib.tron_host_alloc(nbytes)
    if not ptr:
        raise MemoryError(last_error())
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    arr = np.frombuffer(buf, dtype=dt, count=int(n))
    weakref.finalize(buf, lib.tron_host_free, ptr)
    return arr


def last_error() -> str:
    msg = lib.tron_gpu_last_error()
    return msg.decode() if msg else ""
