"""B200-native TRON hot path (arXiv 2008.03433): FP64 fun/grad/Hv/preconditioner
kernels for L2-regularised logistic regression (sparse CSR) and L2-loss SVM
(dense), device-resident truncated CG, row-sharded multi-GPU -- behind the
reference's LossEvaluator / solve() interface (include/tron_b200.h).
"""
from .tron import (  # noqa: F401
    BoundsError, BudgetExceededError, CgExit, CgResult, DeviceError, DimensionError, Error,
    ExecutionPlan, FeatureMatrix, GpuEvaluator, IterationRecord, LogicError, LossKind,
    NumericalFailureError, Problem, SolveResult, SolverTrace, StrategyPreconditionError,
    SvmStrategy, TransferLedger, TrustRegionConfig, device_count, make_evaluator, solve,
    quadratic_model, trust_region_update)
from ._lib import LIB_PATH  # noqa: F401
