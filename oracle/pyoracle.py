"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the parity oracle.

* ``Port``      -- oracle/liboracle.so, the plain-C restatement (tron_oracle.c)
* ``Reference`` -- oracle/_ref/libtronref.so, the reference's own sources
                   compiled in place (oracle/Makefile) behind ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtronref.so")

PD = POINTER(c_double)
PI64 = POINTER(c_int64)
PI32 = POINTER(c_int32)

LOGISTIC, L2SVM = 0, 1
CSR, DENSE = 1, 0


class or_config(ctypes.Structure):
    _fields_ = [("eps", c_double), ("max_outer_iters", c_size_t), ("max_cg_iters", c_size_t),
                ("sigma0", c_double), ("eta1", c_double), ("eta2", c_double),
                ("gamma1", c_double), ("gamma2", c_double), ("gamma3", c_double),
                ("cg_tol", c_double), ("use_preconditioner", c_int)]


class or_iteration(ctypes.Structure):
    _fields_ = [("f_candidate", c_double), ("gradient_norm", c_double), ("delta", c_double),
                ("sigma", c_double), ("accepted", c_int32), ("cg_exit", c_int32),
                ("cg_iters", c_uint64)]


class or_solve_info(ctypes.Structure):
    _fields_ = [("f_initial", c_double), ("gradient_norm_initial", c_double),
                ("objective", c_double), ("accepted_steps", c_uint64),
                ("gradient_materializations", c_uint64), ("objective_evaluations", c_uint64),
                ("n_iterations", c_uint64), ("converged", c_int32), ("status", c_int32)]


class or_matrix(ctypes.Structure):
    _fields_ = [("layout", c_int), ("rows", c_size_t), ("cols", c_size_t),
                ("row_offsets", PI64), ("col_indices", PI32), ("values", PD)]


class or_problem(ctypes.Structure):
    _fields_ = [("X", or_matrix), ("y", PD), ("C", c_double)]


HV_FN = ctypes.CFUNCTYPE(None, c_void_p, PD, PD)


def _p(a, t=PD):
    return a.ctypes.data_as(t) if a is not None else None


def make_config(cfg=None, **over):
    c = or_config()
    c.eps, c.max_outer_iters, c.max_cg_iters = 0.1, 1000, 0
    c.sigma0, c.eta1, c.eta2 = 1e-4, 0.25, 0.75
    c.gamma1, c.gamma2, c.gamma3 = 0.25, 0.5, 4.0
    c.cg_tol, c.use_preconditioner = 0.1, 0
    if cfg is not None:
        for f, _ in or_config._fields_:
            setattr(c, f, int(getattr(cfg, f)) if f == "use_preconditioner" else getattr(cfg, f))
    for k, v in over.items():
        setattr(c, k, v)
    return c


def _matrix_args(X):
    """(layout, l, n, ro, ci, vals) with arrays kept alive by the caller."""
    if X.layout == "csr":
        return CSR, X.rows, X.cols, X.row_offsets, X.col_indices, X.values
    return DENSE, X.rows, X.cols, None, None, X.values


def _trace(info, tr, cap):
    recs = []
    for k in range(min(info.n_iterations, cap)):
        r = tr[k]
        recs.append(dict(f_candidate=r.f_candidate, gradient_norm=r.gradient_norm, delta=r.delta,
                         sigma=r.sigma, accepted=bool(r.accepted), cg_iters=int(r.cg_iters),
                         cg_exit=int(r.cg_exit)))
    return dict(f_initial=info.f_initial, gradient_norm_initial=info.gradient_norm_initial,
                objective=info.objective, accepted_steps=info.accepted_steps,
                gradient_materializations=info.gradient_materializations,
                objective_evaluations=info.objective_evaluations, converged=bool(info.converged),
                status=info.status, iterations=recs)


class Port:
    """The plain-C restatement (bit-identical to the reference by construction)."""

    def __init__(self, path=PORT_PATH):
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.or_solve.argtypes = [POINTER(or_problem), c_int, POINTER(or_config), PD, PD,
                               POINTER(or_solve_info), POINTER(or_iteration), c_size_t]
        L.or_logistic_fused_pass.restype = c_double
        L.or_logistic_fused_pass.argtypes = [POINTER(or_problem), PD, PD, PD, PD, PD]
        L.or_logistic_gradient.argtypes = [POINTER(or_problem), PD, PD, PD]
        L.or_logistic_hessian_vec.argtypes = [POINTER(or_problem), PD, PD, PD]
        L.or_logistic_precond.argtypes = [POINTER(or_problem), PD, PD]
        L.or_svm_fused_pass.restype = c_double
        L.or_svm_fused_pass.argtypes = [POINTER(or_problem), PD, PD, PI64, POINTER(c_size_t)]
        L.or_svm_gradient.argtypes = [POINTER(or_problem), PD, PI64, c_size_t, PD, PD]
        L.or_svm_hessian_vec.argtypes = [POINTER(or_problem), PI64, c_size_t, PD, PD]
        L.or_svm_precond.argtypes = [POINTER(or_problem), PI64, c_size_t, PD]
        L.or_matvec.argtypes = [POINTER(or_matrix), PD, PD]
        L.or_matvec_transpose.argtypes = [POINTER(or_matrix), PD, PD]
        L.or_truncated_cg.argtypes = [PD, c_size_t, HV_FN, c_void_p, c_double, PD,
                                      POINTER(or_config), PD, POINTER(c_int), POINTER(c_size_t), PD]

    def _prob(self, problem):
        X = problem.X
        m = or_matrix(CSR if X.layout == "csr" else DENSE, X.rows, X.cols,
                      _p(X.row_offsets, PI64) if X.layout == "csr" else None,
                      _p(X.col_indices, PI32) if X.layout == "csr" else None, _p(X.values))
        y = np.ascontiguousarray(problem.y, dtype=np.float64)
        p = or_problem(m, _p(y), float(problem.C))
        p._keep = (X, y)
        return p

    def solve(self, problem, loss, cfg=None, w0=None, cap=4096, **over):
        p = self._prob(problem)
        c = make_config(cfg, **over)
        w = np.zeros(problem.X.cols)
        info = or_solve_info()
        tr = (or_iteration * cap)()
        w0a = None if w0 is None else np.ascontiguousarray(w0, dtype=np.float64)
        self.lib.or_solve(ctypes.byref(p), loss, ctypes.byref(c), _p(w0a), _p(w), ctypes.byref(info),
                          tr, cap)
        return w, _trace(info, tr, cap)

    def logistic(self, problem, w, v=None):
        p = self._prob(problem)
        l, n = problem.X.rows, problem.X.cols
        w = np.ascontiguousarray(w, dtype=np.float64)
        z, zh, dv, al = (np.empty(l) for _ in range(4))
        f = self.lib.or_logistic_fused_pass(ctypes.byref(p), _p(w), _p(z), _p(zh), _p(dv), _p(al))
        g = np.empty(n)
        self.lib.or_logistic_gradient(ctypes.byref(p), _p(zh), _p(w), _p(g))
        m = np.empty(n)
        self.lib.or_logistic_precond(ctypes.byref(p), _p(dv), _p(m))
        out = dict(f=f, z=z, zhat=zh, dvec=dv, alpha=al, g=g, M=m)
        if v is not None:
            v = np.ascontiguousarray(v, dtype=np.float64)
            hv = np.empty(n)
            self.lib.or_logistic_hessian_vec(ctypes.byref(p), _p(dv), _p(v), _p(hv))
            out["hv"] = hv
        return out

    def svm(self, problem, w, v=None):
        p = self._prob(problem)
        l, n = problem.X.rows, problem.X.cols
        w = np.ascontiguousarray(w, dtype=np.float64)
        z = np.empty(l)
        act = np.empty(max(l, 1), dtype=np.int64)
        na = c_size_t()
        f = self.lib.or_svm_fused_pass(ctypes.byref(p), _p(w), _p(z), _p(act, PI64), ctypes.byref(na))
        act = act[:na.value].copy()
        g = np.empty(n)
        self.lib.or_svm_gradient(ctypes.byref(p), _p(z), _p(act, PI64), act.size, _p(w), _p(g))
        m = np.empty(n)
        self.lib.or_svm_precond(ctypes.byref(p), _p(act, PI64), act.size, _p(m))
        out = dict(f=f, z=z, active=act, g=g, M=m)
        if v is not None:
            v = np.ascontiguousarray(v, dtype=np.float64)
            hv = np.empty(n)
            self.lib.or_svm_hessian_vec(ctypes.byref(p), _p(act, PI64), act.size, _p(v), _p(hv))
            out["hv"] = hv
        return out

    def matvec_transpose(self, X, u):
        m = or_matrix(CSR if X.layout == "csr" else DENSE, X.rows, X.cols,
                      _p(X.row_offsets, PI64) if X.layout == "csr" else None,
                      _p(X.col_indices, PI32) if X.layout == "csr" else None, _p(X.values))
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(X.cols)
        self.lib.or_matvec_transpose(ctypes.byref(m), _p(u), _p(out))
        return out

    def truncated_cg(self, g, hv, delta, precond=None, cfg=None, **over):
        """hv: python callable v -> Hv (numpy)."""
        g = np.ascontiguousarray(g, dtype=np.float64)
        n = g.size

        def cb(_ctx, vp, outp):
            v = np.ctypeslib.as_array(vp, shape=(n,)).copy()
            out = np.ctypeslib.as_array(outp, shape=(n,))
            out[:] = hv(v)

        fn = HV_FN(cb)
        c = make_config(cfg, **over)
        d = np.empty(n)
        ex, it, q = c_int(), c_size_t(), c_double()
        M = None if precond is None else np.ascontiguousarray(precond, dtype=np.float64)
        st = self.lib.or_truncated_cg(_p(g), n, fn, None, float(delta), _p(M), ctypes.byref(c), _p(d),
                                      ctypes.byref(ex), ctypes.byref(it), ctypes.byref(q))
        return dict(status=st, d=d, exit=ex.value, iters=it.value, model_value=q.value)


class Reference:
    """The reference CPU solver compiled from /root/reference sources."""

    SEQ, PAR, STAGED, MIX = 0, 1, 2, 3

    def __init__(self, path=REF_PATH):
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.ref_solve.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double, c_int,
                                POINTER(or_config), c_int, ctypes.c_uint, PD, PD,
                                POINTER(or_solve_info), POINTER(or_iteration), c_size_t]
        L.ref_time_calls.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double, c_int,
                                     c_int, ctypes.c_uint, c_int, PD]
        L.ref_logistic_fused_pass.restype = c_double
        L.ref_logistic_fused_pass.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD,
                                              c_double, PD, PD, PD, PD, PD]
        L.ref_logistic_grad_hv.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double,
                                           PD, PD, PD, PD, PD]
        L.ref_svm_fused_pass.restype = c_double
        L.ref_svm_fused_pass.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double,
                                         PD, PD, PI64, POINTER(c_size_t)]
        L.ref_svm_grad_hv.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double, PD,
                                      PD, PD, PD, PD]
        L.ref_testgen_dense_problem.argtypes = [c_uint64, c_size_t, c_size_t, c_double, c_double,
                                                PD, PD]
        L.ref_testgen_dense_problem_scaled.argtypes = [c_uint64, c_size_t, c_size_t, c_double,
                                                       c_double, c_double, PD, PD]
        L.ref_testgen_sparse_problem.restype = c_size_t
        L.ref_testgen_sparse_problem.argtypes = [c_uint64, c_size_t, c_size_t, c_double, c_double,
                                                 c_double, PI64, PI32, PD, PD]
        L.ref_testgen_random_vector.argtypes = [c_uint64, c_size_t, c_double, PD]
        L.ref_testgen_random_index_set.restype = c_size_t
        L.ref_testgen_random_index_set.argtypes = [c_uint64, c_size_t, c_double, PI64]
        L.ref_synth_sparse.argtypes = [c_uint64, c_size_t, c_size_t, c_size_t, c_double, c_double,
                                       PI64, PI32, PD, PD]
        L.ref_synth_dense.argtypes = [c_uint64, c_size_t, c_size_t, c_double, c_double, c_double,
                                      PD, PD]
        L.ref_predict.restype = c_size_t
        L.ref_predict.argtypes = [c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, PD, PD]

    def _args(self, problem):
        lay, l, n, ro, ci, vals = _matrix_args(problem.X)
        y = np.ascontiguousarray(problem.y, dtype=np.float64)
        return (lay, l, n, _p(ro, PI64), _p(ci, PI32), _p(vals), _p(y), float(problem.C)), (ro, ci, vals, y)

    def solve(self, problem, loss, cfg=None, backend=0, workers=1, w0=None, cap=4096, **over):
        args, keep = self._args(problem)
        c = make_config(cfg, **over)
        w = np.zeros(problem.X.cols)
        info = or_solve_info()
        tr = (or_iteration * cap)()
        w0a = None if w0 is None else np.ascontiguousarray(w0, dtype=np.float64)
        self.lib.ref_solve(*args, loss, ctypes.byref(c), backend, workers, _p(w0a), _p(w),
                           ctypes.byref(info), tr, cap)
        return w, _trace(info, tr, cap)

    def solve_with_gpu_evaluator(self, lib_path, problem, loss, cfg=None, cap=4096, **over):
        """The reference's own tron::solve driving a LossEvaluator that forwards
        every call to the B200 C ABI (INTEGRATION.md's binding), in this process."""
        L = self.lib
        L.ref_solve_with_gpu_evaluator.argtypes = [
            ctypes.c_char_p, c_int, c_size_t, c_size_t, PI64, PI32, PD, PD, c_double, c_int,
            POINTER(or_config), PD, POINTER(or_solve_info), POINTER(or_iteration), c_size_t,
            ctypes.c_char_p, c_size_t]
        args, keep = self._args(problem)
        c = make_config(cfg, **over)
        w = np.zeros(problem.X.cols)
        info = or_solve_info()
        tr = (or_iteration * cap)()
        msg = ctypes.create_string_buffer(512)
        st = L.ref_solve_with_gpu_evaluator(os.fsencode(lib_path), *args, loss, ctypes.byref(c),
                                            _p(w), ctypes.byref(info), tr, cap, msg, 512)
        if st != 0:
            raise RuntimeError(f"ref_solve_with_gpu_evaluator: {msg.value.decode()}")
        return w, _trace(info, tr, cap)

    def parse_libsvm(self, text: bytes, n_override=0):
        """The reference's parse_libsvm (io.cpp:54-132) on an in-memory text:
        ('ok', (ro, ci, vals, y, n)) or (kind, (message, line)), kind in
        'parse' / 'label' / 'other'."""
        L = self.lib
        if not getattr(self, "_parse_bound", False):
            L.ref_parse_libsvm.argtypes = [ctypes.c_char_p, c_size_t, c_size_t,
                                           ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p, c_size_t,
                                           POINTER(c_size_t)]
            L.ref_parsed_sizes.argtypes = [ctypes.c_void_p, POINTER(c_size_t), POINTER(c_size_t),
                                           POINTER(c_size_t)]
            L.ref_parsed_copy.argtypes = [ctypes.c_void_p, PI64, PI32, PD, PD]
            L.ref_parsed_free.argtypes = [ctypes.c_void_p]
            self._parse_bound = True
        h = ctypes.c_void_p()
        msg = ctypes.create_string_buffer(512)
        line = c_size_t()
        rc = L.ref_parse_libsvm(text, len(text), n_override, ctypes.byref(h), msg, 512,
                                ctypes.byref(line))
        if rc != 0:
            return {1: "parse", 2: "label"}.get(rc, "other"), (msg.value.decode(), line.value)
        r, c, z = c_size_t(), c_size_t(), c_size_t()
        L.ref_parsed_sizes(h, ctypes.byref(r), ctypes.byref(c), ctypes.byref(z))
        ro = np.empty(r.value + 1, dtype=np.int64)
        ci = np.empty(z.value, dtype=np.int32)
        vals = np.empty(z.value)
        y = np.empty(r.value)
        L.ref_parsed_copy(h, _p(ro, PI64), _p(ci, PI32), _p(vals), _p(y))
        L.ref_parsed_free(h)
        return "ok", (ro, ci, vals, y, c.value)

    def load_dense(self, text: bytes, n: int):
        """The reference's load_dense (io.cpp:164-197) on an in-memory text:
        ('ok', (values, y)) or (kind, (message, line))."""
        L = self.lib
        self.parse_libsvm(b"")  # binds the parsed_* helpers
        L.ref_load_dense.argtypes = [ctypes.c_char_p, c_size_t, c_size_t, ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.c_char_p, c_size_t, POINTER(c_size_t)]
        h = ctypes.c_void_p()
        msg = ctypes.create_string_buffer(512)
        line = c_size_t()
        rc = L.ref_load_dense(text, len(text), n, ctypes.byref(h), msg, 512, ctypes.byref(line))
        if rc != 0:
            return {1: "parse", 2: "label"}.get(rc, "other"), (msg.value.decode(), line.value)
        r, c, z = c_size_t(), c_size_t(), c_size_t()
        L.ref_parsed_sizes(h, ctypes.byref(r), ctypes.byref(c), ctypes.byref(z))
        vals = np.empty(z.value)
        y = np.empty(r.value)
        L.ref_parsed_copy(h, None, None, _p(vals), _p(y))
        L.ref_parsed_free(h)
        return "ok", (vals, y)

    def time_calls(self, problem, loss, workers, reps=1, backend=1):
        """Per-call ms of the reference evaluator (fun, grad, Hv) at w = 0 under
        ExecutionPlan::parallel(workers) (backend 1) or ::sequential() (backend 0)."""
        args, keep = self._args(problem)
        out = np.zeros(3)
        st = self.lib.ref_time_calls(*args, loss, backend, workers, reps, _p(out))
        if st != 0:
            raise RuntimeError(f"ref_time_calls failed ({st})")
        return dict(fun_ms=out[0], grad_ms=out[1], hv_ms=out[2])

    def logistic(self, problem, w, v):
        args, keep = self._args(problem)
        l, n = problem.X.rows, problem.X.cols
        w = np.ascontiguousarray(w, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        z, zh, dv, al = (np.empty(l) for _ in range(4))
        f = self.lib.ref_logistic_fused_pass(*args, _p(w), _p(z), _p(zh), _p(dv), _p(al))
        g, hv, m = np.empty(n), np.empty(n), np.empty(n)
        self.lib.ref_logistic_grad_hv(*args, _p(w), _p(v), _p(g), _p(hv), _p(m))
        return dict(f=f, z=z, zhat=zh, dvec=dv, alpha=al, g=g, hv=hv, M=m)

    def svm(self, problem, w, v):
        args, keep = self._args(problem)
        l, n = problem.X.rows, problem.X.cols
        w = np.ascontiguousarray(w, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.empty(l)
        act = np.empty(max(l, 1), dtype=np.int64)
        na = c_size_t()
        f = self.lib.ref_svm_fused_pass(*args, _p(w), _p(z), _p(act, PI64), ctypes.byref(na))
        g, hv, m = np.empty(n), np.empty(n), np.empty(n)
        self.lib.ref_svm_grad_hv(*args, _p(w), _p(v), _p(g), _p(hv), _p(m))
        return dict(f=f, z=z, active=act[:na.value].copy(), g=g, hv=hv, M=m)

    def predict(self, X, w):
        """The reference's predict (model.cpp:88-117): (labels, correct) of the
        rows of X (a FeatureMatrix-like object) under w; y optional via X.y."""
        lay, l, n, ro, ci, vals = _matrix_args(X)
        w = np.ascontiguousarray(w, dtype=np.float64)
        y = getattr(X, "y", None)
        y = np.ascontiguousarray(y, dtype=np.float64) if y is not None else np.zeros(l)
        labels = np.empty(l)
        c = self.lib.ref_predict(lay, l, n, _p(ro, PI64), _p(ci, PI32), _p(vals), _p(y), _p(w), _p(labels))
        return labels, int(c)

    # SYNTH-v1 with the reference's testgen::Rng
    def synth_sparse(self, seed, l, n, k, s=1.0, flip=0.1):
        ro, ci = np.empty(l + 1, dtype=np.int64), np.empty(l * k, dtype=np.int32)
        vals, y = np.empty(l * k), np.empty(l)
        st = self.lib.ref_synth_sparse(seed, l, n, k, s, flip, _p(ro, PI64), _p(ci, PI32), _p(vals), _p(y))
        if st != 0:
            raise ValueError("ref_synth_sparse: bad shape")
        return ro, ci, vals, y

    def synth_dense(self, seed, l, n=40, decades=2.0, rho=0.0, flip=0.1):
        vals, y = np.empty(l * n), np.empty(l)
        st = self.lib.ref_synth_dense(seed, l, n, decades, rho, flip, _p(vals), _p(y))
        if st != 0:
            raise ValueError("ref_synth_dense: bad shape")
        return vals, y

    # fixture generators
    def dense_problem(self, seed, l, n, flip=0.1):
        vals, y = np.empty(l * n), np.empty(l)
        self.lib.ref_testgen_dense_problem(seed, l, n, 1.0, flip, _p(vals), _p(y))
        return vals, y

    def dense_problem_scaled(self, seed, l, n, scale, flip=0.02):
        vals, y = np.empty(l * n), np.empty(l)
        self.lib.ref_testgen_dense_problem_scaled(seed, l, n, 1.0, scale, flip, _p(vals), _p(y))
        return vals, y

    def sparse_problem(self, seed, l, n, density=0.1, flip=0.1):
        nnz = self.lib.ref_testgen_sparse_problem(seed, l, n, 1.0, density, flip, None, None, None, None)
        ro, ci = np.empty(l + 1, dtype=np.int64), np.empty(max(nnz, 1), dtype=np.int32)
        vals, y = np.empty(max(nnz, 1)), np.empty(l)
        self.lib.ref_testgen_sparse_problem(seed, l, n, 1.0, density, flip, _p(ro, PI64), _p(ci, PI32),
                                            _p(vals), _p(y))
        return ro, ci[:nnz], vals[:nnz], y

    def random_vector(self, seed, n, span=1.0):
        out = np.empty(n)
        self.lib.ref_testgen_random_vector(seed, n, span, _p(out))
        return out

    def random_index_set(self, seed, l, fraction):
        cnt = self.lib.ref_testgen_random_index_set(seed, l, fraction, None)
        out = np.empty(max(cnt, 1), dtype=np.int64)
        self.lib.ref_testgen_random_index_set(seed, l, fraction, _p(out, PI64))
        return out[:cnt]


def have_reference():
    return os.path.exists(REF_PATH)
