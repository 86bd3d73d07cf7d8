"""paper_2110_11738_b200 -- B200-native (sm_100a) DROT optimal-transport solver.

A drop-in for the reference's solve path (drot::solve<T>, drot_step,
FusedEngine; /root/reference/proj/core/include/drot/).  All computation runs
in libdrotb200.so (hand-written CUDA kernels behind the C ABI of
include/drotb.h); importing this package fails loudly if the library has not
been built -- there is no CPU fallback.
"""
from . import _lib
from .api import (DeviceError, DrotConfig, DrotState, DualCertificate, EngineKind, Errc,
                  ErgodicMean, TileRange, ValidateOptions, materialize_plan, materialize_y,
                  validate_problem,
                  Error, FusedArray, FusedEngine, FusedPassOutput, GaussianSpec,
                  MemoryCounters, Order, PassOptions, Precision, ResidualReport,
                  SolveResult, SolveStatus, SolveTrace, TilePlan, TraceRow, TransportPlan,
                  TransportProblem, check_problem, drot_step, dyadic_marginal,
                  gen_gaussian_problem, gen_gaussian_problem_as, init_state,
                  kernel_launches, objective, release_device_cache, plan_tiles, residual_report,
                  sinkhorn_solve, counter_uniform, random_matrix, recover_duals, rho0_warmup_preset, solve)
from .session import Session, nccl_unique_id, shard_rows

LIB_PATH = _lib.LIB_PATH
_lib.load()

__all__ = [
    "ErgodicMean", "TileRange", "ValidateOptions", "materialize_plan", "materialize_y",
    "validate_problem", "DeviceError", "DrotConfig", "DrotState", "DualCertificate", "EngineKind", "Errc",
    "Error", "FusedArray", "FusedEngine", "FusedPassOutput", "GaussianSpec",
    "MemoryCounters", "Order", "PassOptions", "Precision", "ResidualReport", "SolveResult",
    "SolveStatus", "SolveTrace", "TilePlan", "TraceRow", "TransportPlan",
    "TransportProblem", "check_problem", "drot_step", "dyadic_marginal",
    "gen_gaussian_problem", "gen_gaussian_problem_as", "init_state", "kernel_launches",
    "objective", "release_device_cache", "residual_report", "sinkhorn_solve", "plan_tiles", "counter_uniform", "random_matrix", "recover_duals", "rho0_warmup_preset", "solve", "Session", "nccl_unique_id", "shard_rows", "LIB_PATH",
]
