"""Python mirror of the reference's solver API (proj/include/tron/*.hpp) over
the B200 C ABI.

Names, argument meaning and error classes follow the reference:
``solve(problem, loss, cfg, plan, warm_start)`` is tron::solve
(backend.hpp:72-73), ``make_evaluator`` is tron::make_evaluator
(backend.hpp:68-69) and the evaluator methods are tron::LossEvaluator's
(tron.hpp:105-125).  The only backend here is the GPU one
(``ExecutionPlan.gpu()``); the solve itself runs natively (C++ driver +
CUDA kernels) -- Python only marshals arrays.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import lib

# ----------------------------------------------------------------------------
# errors (error.hpp:10-69, tron.hpp:70-78)
# ----------------------------------------------------------------------------


class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class BoundsError(Error):
    pass


class StrategyPreconditionError(Error):
    pass


class BudgetExceededError(Error):
    pass


class DeviceError(Error):
    pass


class LogicError(Error):
    """std::logic_error in the reference (evaluator misuse, backend.cpp:167)."""


class NumericalFailureError(Error):
    def __init__(self, what: str, trace: "SolverTrace"):
        super().__init__(what)
        self.trace = trace


def _raise(status: int, trace: Optional["SolverTrace"] = None):
    if status == _lib.OK:
        return
    msg = _lib.last_error()
    if status == _lib.ERR_DIMENSION:
        raise DimensionError(msg)
    if status == _lib.ERR_BOUNDS:
        raise BoundsError(msg)
    if status == _lib.ERR_STRATEGY:
        raise StrategyPreconditionError(msg)
    if status == _lib.ERR_BUDGET:
        raise BudgetExceededError(msg)
    if status == _lib.ERR_NUMERICAL:
        raise NumericalFailureError(msg, trace if trace is not None else SolverTrace())
    if status == _lib.ERR_LOGIC:
        raise LogicError(msg)
    raise DeviceError(f"status {status}: {msg}")


# ----------------------------------------------------------------------------
# solver types (tron.hpp:13-66)
# ----------------------------------------------------------------------------


class LossKind(enum.Enum):
    Logistic = _lib.LOSS_LOGISTIC
    L2Svm = _lib.LOSS_L2SVM


class SvmStrategy(enum.Enum):
    Gathered = _lib.SVM_GATHERED
    Indirect = _lib.SVM_INDIRECT
    Auto = _lib.SVM_AUTO  # B200 cost model: gather only when X_I <= half of X


class CgExit(enum.IntEnum):
    Converged = 0
    Boundary = 1
    MaxIters = 2


@dataclass
class TrustRegionConfig:
    eps: float = 0.1
    max_outer_iters: int = 1000
    max_cg_iters: int = 0  # 0 = min(n, 1000)
    sigma0: float = 1e-4
    eta1: float = 0.25
    eta2: float = 0.75
    gamma1: float = 0.25
    gamma2: float = 0.5
    gamma3: float = 4.0
    cg_tol: float = 0.1
    use_preconditioner: bool = False

    def validate(self):  # tron.cpp:19-29
        if not self.eps > 0.0:
            raise DimensionError("config: eps must be positive")
        if not (0.0 < self.sigma0 < 1.0):
            raise DimensionError("config: sigma0 must be in (0,1)")
        if not (0.0 < self.eta1 < self.eta2 < 1.0):
            raise DimensionError("config: need 0 < eta1 < eta2 < 1")
        if not (0.0 < self.gamma1 < self.gamma2 < 1.0 and self.gamma3 > 1.0):
            raise DimensionError("config: need 0 < gamma1 < gamma2 < 1 < gamma3")
        if not (0.0 < self.cg_tol < 1.0):
            raise DimensionError("config: cg_tol must be in (0,1)")

    def to_c(self, mode: int = _lib.SOLVE_DEVICE) -> _lib.tron_config:
        c = _lib.tron_config()
        lib.tron_gpu_default_config(ctypes.byref(c))
        c.eps, c.max_outer_iters, c.max_cg_iters = self.eps, self.max_outer_iters, self.max_cg_iters
        c.sigma0, c.eta1, c.eta2 = self.sigma0, self.eta1, self.eta2
        c.gamma1, c.gamma2, c.gamma3 = self.gamma1, self.gamma2, self.gamma3
        c.cg_tol = self.cg_tol
        c.use_preconditioner = int(bool(self.use_preconditioner))
        c.solve_mode = mode
        return c


@dataclass
class IterationRecord:
    f_candidate: float = 0.0
    gradient_norm: float = 0.0
    delta: float = 0.0
    sigma: float = 0.0
    accepted: bool = False
    cg_iters: int = 0
    cg_exit: CgExit = CgExit.Converged


@dataclass
class SolverTrace:
    f_initial: float = 0.0
    gradient_norm_initial: float = 0.0
    iterations: List[IterationRecord] = field(default_factory=list)
    accepted_steps: int = 0
    gradient_materializations: int = 0
    objective_evaluations: int = 0


@dataclass
class SolveResult:
    w: np.ndarray
    trace: SolverTrace
    objective: float = 0.0
    converged: bool = False
    hessian_products: int = 0
    device_ms: float = 0.0


@dataclass
class CgResult:
    d: np.ndarray
    exit: CgExit
    iters: int
    model_value: float


@dataclass
class TransferLedger:  # backend.hpp:32-43
    bulk_handoffs: int = 0
    scalar_returns: int = 0
    gradient_materializations: int = 0
    concealed_vector_returns: int = 0
    margin_passes: int = 0
    gathered_submatrix_bytes: int = 0
    index_set_bytes: int = 0


@dataclass
class ExecutionPlan:
    """ExecutionPlan (backend.hpp:46-60) for the B200 backend."""
    device: int = 0
    svm_strategy: SvmStrategy = SvmStrategy.Indirect
    gathered_budget_bytes: int = 2 << 30
    solve_mode: str = "device"  # "device" | "host_cg" (parity: reference control flow on host)
    ledger: TransferLedger = field(default_factory=TransferLedger)
    # row sharding (multi-GPU): rank/world and an NCCL unique id (bytes)
    rank: int = 0
    world: int = 1
    nccl_unique_id: Optional[bytes] = None
    row_begin: int = 0
    global_rows: int = 0
    # dense L2-SVM: every reduction in the reference's order (bit-for-bit results)
    reference_order: bool = False
    # host data plane instead of NCCL (world > 1): fn(buf: np.ndarray) sums buf
    # over the ranks in place (e.g. a gloo / MPI allreduce)
    host_allreduce: Optional[Callable[[np.ndarray], None]] = None
    # dense X larger than device memory: 0 auto, 1 always stream X from host
    # memory (the caller keeps the Problem alive), -1 never
    out_of_core: int = 0
    stream_block_rows: int = 0
    # column-partitioned layout (world > 1): this rank owns columns
    # [col_begin, col_begin + n) of global_cols (sharding.column_shard)
    partition: str = "rows"
    col_begin: int = 0
    global_cols: int = 0

    @staticmethod
    def gpu(device: int = 0, svm_strategy: SvmStrategy = SvmStrategy.Indirect,
            gathered_budget_bytes: int = 2 << 30, solve_mode: str = "device",
            reference_order: bool = False, out_of_core: int = 0,
            stream_block_rows: int = 0) -> "ExecutionPlan":
        return ExecutionPlan(device=device, svm_strategy=svm_strategy,
                             gathered_budget_bytes=gathered_budget_bytes, solve_mode=solve_mode,
                             reference_order=reference_order, out_of_core=out_of_core,
                             stream_block_rows=stream_block_rows)

    def to_c(self):
        o = _lib.tron_gpu_options()
        lib.tron_gpu_default_options(ctypes.byref(o))
        o.device = self.device
        o.svm_strategy = self.svm_strategy.value
        o.gathered_budget_bytes = self.gathered_budget_bytes
        o.rank, o.world = self.rank, self.world
        o.row_begin, o.global_rows = self.row_begin, self.global_rows
        o.reference_order = int(bool(self.reference_order))
        o.out_of_core = int(self.out_of_core)
        o.stream_block_rows = int(self.stream_block_rows)
        o.partition = _lib.PARTITION_COLUMNS if self.partition == "columns" else _lib.PARTITION_ROWS
        o.col_begin, o.global_cols = int(self.col_begin), int(self.global_cols)
        keep = []
        if self.nccl_unique_id is not None:
            uid = ctypes.create_string_buffer(bytes(self.nccl_unique_id), 128)
            o.nccl_unique_id = ctypes.cast(uid, ctypes.c_void_p)
            keep.append(uid)
        if self.host_allreduce is not None:
            fn = self.host_allreduce

            def trampoline(_user, buf, count):
                fn(np.ctypeslib.as_array(buf, shape=(count,)))

            cb = _lib.HOST_ALLREDUCE(trampoline)
            o.host_allreduce = ctypes.cast(cb, ctypes.c_void_p)
            keep.append(cb)
        return o, keep


# ----------------------------------------------------------------------------
# data (FeatureMatrix linalg.hpp:21-63, Problem loss.hpp:18-26)
# ----------------------------------------------------------------------------


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


class FeatureMatrix:
    """Host-side feature matrix: CSR (int64 offsets, int32 columns) or dense row-major."""

    def __init__(self, layout, rows, cols, values, row_offsets=None, col_indices=None):
        self.layout = layout
        self.rows, self.cols = int(rows), int(cols)
        self.values = values
        self.row_offsets = row_offsets
        self.col_indices = col_indices

    @staticmethod
    def dense(rows, cols, values):
        v = _f64(values).reshape(-1)
        if v.size != rows * cols:
            raise DimensionError(f"dense matrix: {v.size} values for {rows}x{cols}")
        return FeatureMatrix("dense", rows, cols, v)

    @staticmethod
    def csr(rows, cols, row_offsets, col_indices, values):
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int32)
        v = _f64(values)
        if ro.size != rows + 1:
            raise DimensionError(f"csr matrix: {ro.size} row offsets for {rows} rows")
        if ro[0] != 0 or ro[-1] != v.size or ci.size != v.size:
            raise DimensionError("csr matrix: offsets/indices/values disagree")
        return FeatureMatrix("csr", rows, cols, v, ro, ci)

    def stored(self):
        return self.values.size

    def to_dense(self):
        if self.layout == "dense":
            return self.values.reshape(self.rows, self.cols)
        out = np.zeros((self.rows, self.cols))
        for i in range(self.rows):
            s, e = self.row_offsets[i], self.row_offsets[i + 1]
            out[i, self.col_indices[s:e]] = self.values[s:e]
        return out


@dataclass
class Problem:
    X: FeatureMatrix
    y: np.ndarray
    C: float = 1.0

    def instances(self):
        return self.X.rows

    def features(self):
        return self.X.cols


# ----------------------------------------------------------------------------
# evaluator (LossEvaluator, tron.hpp:105-125) on the GPU
# ----------------------------------------------------------------------------


@dataclass
class LogisticState:
    z: np.ndarray
    zhat: np.ndarray
    dvec: np.ndarray


@dataclass
class SvmState:
    z: np.ndarray
    active: np.ndarray  # ascending int64 row indices (IndexSet)


class GpuEvaluator:
    """make_evaluator(problem, loss, plan) for the B200 backend."""

    def __init__(self, problem: Problem, loss: LossKind, plan: ExecutionPlan):
        self.problem, self.loss, self.plan = problem, loss, plan
        X = problem.X
        y = _f64(problem.y)
        if y.size != X.rows:
            raise DimensionError(f"problem: {y.size} labels for {X.rows} instances")
        opts, self._keep = plan.to_c()
        h = ctypes.c_void_p()
        if X.layout == "csr":
            st = lib.tron_gpu_create_csr(loss.value, X.rows, X.cols, _ptr(X.row_offsets, ctypes.c_int64),
                                         _ptr(X.col_indices, ctypes.c_int32),
                                         _ptr(X.values, ctypes.c_double), _ptr(y, ctypes.c_double),
                                         float(problem.C), ctypes.byref(opts), ctypes.byref(h))
        else:
            # out-of-core contexts stream X from this very array for their lifetime
            self._x_host = _f64(X.values)
            st = lib.tron_gpu_create_dense(loss.value, X.rows, X.cols, _ptr(self._x_host, ctypes.c_double),
                                           _ptr(y, ctypes.c_double), float(problem.C),
                                           ctypes.byref(opts), ctypes.byref(h))
        _raise(st)
        self._h = h
        self.n = X.cols
        self.l = X.rows

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib.tron_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- LossEvaluator
    def dimension(self) -> int:
        return self.n

    def eval_candidate(self, w) -> float:
        w = _f64(w)
        if w.size != self.n:
            raise DimensionError(f"eval_candidate: w has length {w.size}, expected {self.n}")
        f = ctypes.c_double()
        _raise(lib.tron_gpu_eval_candidate(self._h, _ptr(w, ctypes.c_double), ctypes.byref(f)))
        self._sync_ledger()
        return f.value

    def commit(self) -> float:
        g = ctypes.c_double()
        _raise(lib.tron_gpu_commit(self._h, ctypes.byref(g)))
        self._sync_ledger()
        return g.value

    def gradient(self) -> np.ndarray:
        out = np.empty(self.n)
        _raise(lib.tron_gpu_gradient(self._h, _ptr(out, ctypes.c_double)))
        self._sync_ledger()
        return out

    def hessian_vec(self, v) -> np.ndarray:
        v = _f64(v)
        if v.size != self.n:
            raise DimensionError(f"hessian_vec: v has length {v.size}, expected {self.n}")
        out = np.empty(self.n)
        _raise(lib.tron_gpu_hessian_vec(self._h, _ptr(v, ctypes.c_double), _ptr(out, ctypes.c_double)))
        self._sync_ledger()
        return out

    def quadratic_model(self, d) -> float:
        """quadratic_model(g, hv, d) (tron.cpp:31-35) at the committed iterate, on the
        device: g.d + 0.5 d.Hd with g = gradient() and this evaluator's Hessian."""
        d = _f64(d)
        if d.size != self.n:
            raise DimensionError(f"quadratic_model: direction has length {d.size}, expected {self.n}")
        q = ctypes.c_double()
        _raise(lib.tron_gpu_quadratic_model(self._h, _ptr(d, ctypes.c_double), ctypes.byref(q)))
        return q.value

    def replica_checksum(self) -> np.ndarray:
        """Checksum of the committed w (four 16-bit chunks of the wrap-around sum of
        its bit patterns): equal on every row shard when the replicas agree."""
        out = np.empty(4)
        _raise(lib.tron_gpu_replica_checksum(self._h, _ptr(out, ctypes.c_double)))
        return out

    def precond_diagonal(self) -> np.ndarray:
        out = np.empty(self.n)
        _raise(lib.tron_gpu_precond_diagonal(self._h, _ptr(out, ctypes.c_double)))
        self._sync_ledger()
        return out

    # -- state probes (LogisticEvaluator::candidate_state etc., backend.hpp:113-114)
    def _state(self, which):
        if self.loss == LossKind.Logistic:
            z, zh, dv = np.empty(self.l), np.empty(self.l), np.empty(self.l)
            _raise(lib.tron_gpu_state_lr(self._h, which, _ptr(z, ctypes.c_double),
                                         _ptr(zh, ctypes.c_double), _ptr(dv, ctypes.c_double)))
            return LogisticState(z, zh, dv)
        z = np.empty(self.l)
        act = np.empty(max(self.l, 1), dtype=np.int64)
        cnt = ctypes.c_uint64()
        _raise(lib.tron_gpu_state_svm(self._h, which, _ptr(z, ctypes.c_double),
                                      _ptr(act, ctypes.c_int64), act.size, ctypes.byref(cnt)))
        return SvmState(z, act[:cnt.value].copy())

    def candidate_state(self):
        return self._state(0)

    def committed_state(self):
        return self._state(1)

    # -- device-resident CG (tron.cpp:37-108) on the committed iterate
    def truncated_cg(self, delta: float, cfg: TrustRegionConfig) -> CgResult:
        d = np.empty(self.n)
        ex = ctypes.c_int32()
        it = ctypes.c_uint64()
        q = ctypes.c_double()
        c = cfg.to_c()
        _raise(lib.tron_gpu_truncated_cg(self._h, float(delta), ctypes.byref(c), _ptr(d, ctypes.c_double),
                                         ctypes.byref(ex), ctypes.byref(it), ctypes.byref(q)))
        return CgResult(d, CgExit(ex.value), it.value, q.value)

    def solve(self, cfg: TrustRegionConfig, warm_start=None, mode: Optional[str] = None) -> SolveResult:
        mode = mode or self.plan.solve_mode
        c = cfg.to_c(_lib.SOLVE_HOST_CG if mode == "host_cg" else _lib.SOLVE_DEVICE)
        w = _lib.pinned_array(self.n)  # page-locked: the result comes back by one DMA
        w0 = None
        if warm_start is not None:
            w0 = _f64(warm_start)
            if w0.size != self.n:
                raise DimensionError(f"solve: warm start has length {w0.size}, expected {self.n}")
        cap = int(min(cfg.max_outer_iters, 1 << 16))
        tr = (_lib.tron_iteration * max(cap, 1))()
        info = _lib.tron_solve_info()
        st = lib.tron_gpu_solve(self._h, ctypes.byref(c),
                                _ptr(w0, ctypes.c_double) if w0 is not None else None,
                                _ptr(w, ctypes.c_double), ctypes.byref(info), tr, cap)
        trace = SolverTrace(f_initial=info.f_initial, gradient_norm_initial=info.gradient_norm_initial,
                            accepted_steps=info.accepted_steps,
                            gradient_materializations=info.gradient_materializations,
                            objective_evaluations=info.objective_evaluations)
        for k in range(min(info.n_iterations, cap)):
            r = tr[k]
            trace.iterations.append(IterationRecord(r.f_candidate, r.gradient_norm, r.delta, r.sigma,
                                                    bool(r.accepted), int(r.cg_iters), CgExit(r.cg_exit)))
        self._sync_ledger()
        _raise(st, trace)
        return SolveResult(w, trace, info.objective, bool(info.converged), int(info.hessian_products),
                           float(info.device_ms))

    def predict(self, w):
        """predict(Model, Problem) (model.cpp:88-117) on this evaluator's rows:
        (labels, correct) with labels = sign(x_i . w), ties to +1."""
        w = _f64(w)
        if w.size != self.n:
            raise DimensionError(f"predict: w has length {w.size}, expected {self.n}")
        labels = np.empty(self.l)
        correct = ctypes.c_uint64()
        _raise(lib.tron_gpu_predict(self._h, _ptr(w, ctypes.c_double), _ptr(labels, ctypes.c_double),
                                    ctypes.byref(correct)))
        return labels, int(correct.value)

    # -- plumbing
    def ledger(self) -> TransferLedger:
        lg = _lib.tron_ledger()
        lib.tron_gpu_ledger(self._h, ctypes.byref(lg))
        return TransferLedger(*(getattr(lg, f) for f, _ in _lib.tron_ledger._fields_))

    def _sync_ledger(self):
        self.plan.ledger = self.ledger()

    def launch_count(self) -> int:
        c = ctypes.c_uint64()
        lib.tron_gpu_launch_count(self._h, ctypes.byref(c))
        return c.value

    def mode(self) -> dict:
        """How this context runs (tron_gpu_mode): gram / out_of_core / columns /
        device_loop / sharded / gram_delta."""
        f = ctypes.c_uint32()
        _raise(lib.tron_gpu_mode(self._h, ctypes.byref(f)))
        names = {"gram": _lib.MODE_GRAM, "out_of_core": _lib.MODE_OUT_OF_CORE, "columns": _lib.MODE_COLUMNS,
                 "device_loop": _lib.MODE_DEVICE_LOOP, "sharded": _lib.MODE_SHARDED,
                 "gram_delta": _lib.MODE_GRAM_DELTA}
        return {k: bool(f.value & b) for k, b in names.items()}

    def memory_bytes(self) -> int:
        c = ctypes.c_uint64()
        lib.tron_gpu_memory_bytes(self._h, ctypes.byref(c))
        return c.value

    def bench_kernels(self, reps: int = 10, flush_l2: bool = True):
        out = (ctypes.c_double * 4)()
        _raise(lib.tron_gpu_bench_kernels(self._h, reps, int(flush_l2), out))
        return {"hv_ms": out[0], "transposed_ms": out[1], "forward_ms": out[2], "grad_ms": out[3]}

    def synchronize(self):
        _raise(lib.tron_gpu_synchronize(self._h))


def make_evaluator(problem: Problem, loss: LossKind, plan: ExecutionPlan) -> GpuEvaluator:
    return GpuEvaluator(problem, loss, plan)


def solve(problem: Problem, loss: LossKind, cfg: TrustRegionConfig, plan: ExecutionPlan,
          warm_start=None) -> SolveResult:
    """tron::solve(const Problem&, LossKind, cfg, plan, warm_start) (backend.cpp:314-318)."""
    cfg.validate()
    with make_evaluator(problem, loss, plan) as ev:
        return ev.solve(cfg, warm_start)


def quadratic_model(g, hv, d) -> float:
    """quadratic_model (tron.hpp:83, tron.cpp:31-35): g.d + 0.5 d.(hv(d)), with the
    reference's serial left-to-right dots.  hv is any Hessian apply, e.g. a
    GpuEvaluator's hessian_vec (the device-side variant is
    GpuEvaluator.quadratic_model)."""
    g, d = _f64(g), _f64(d)
    hd = _f64(hv(d))
    gd = 0.0
    for a, b in zip(g.tolist(), d.tolist()):
        gd += a * b
    dh = 0.0
    for a, b in zip(d.tolist(), hd.tolist()):
        dh += a * b
    return gd + 0.5 * dh


def trust_region_update(sigma, delta, step_norm, cfg: TrustRegionConfig):
    """tron.cpp:110-125 (host scalar logic; the device solve applies the same rule)."""
    accept = sigma > cfg.sigma0
    if not accept:
        nd = cfg.gamma1 * step_norm
    elif sigma < cfg.eta1:
        nd = cfg.gamma2 * step_norm
    elif sigma < cfg.eta2:
        nd = delta
    else:
        grown = cfg.gamma3 * step_norm
        nd = grown if grown > delta else delta
    return accept, nd


def device_count() -> int:
    c = ctypes.c_int()
    lib.tron_gpu_device_count(ctypes.byref(c))
    return c.value
