"""Python mirror of the reference's solver API (drot::, proj/core/include/drot/).

Every callable routes through libdrotb200.so (the C ABI in include/drotb.h)
and therefore through the sm_100a kernels; nothing here computes on the CPU
except trivial O(m+n) bookkeeping the reference also does on the host.

Names, argument meaning and error behaviour follow the reference:
  solve               solver.hpp:372-540      drot_step      solver.hpp:361-370
  init_state          solver.hpp:143-186      DrotConfig     solver.hpp:51-88
  FusedEngine         fused.hpp:107-202       check_problem  problem.hpp:122-136
  gen_gaussian_problem probgen.hpp:131-180    Errc / Error   errors.hpp:24-88
Matrices are numpy arrays of shape (m, n) stored column-major (Fortran
order), the reference's storage contract (matrix.hpp:56-59).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import drotb_config, drotb_counters, drotb_pass_out, drotb_report, drotb_trace_row


# ---- errors (errors.hpp) -----------------------------------------------------
class Errc(enum.IntEnum):
    negative_cost = 0
    marginal_not_simplex = 1
    empty_dimension = 2
    non_finite_entry = 3
    shape_mismatch = 4
    non_positive_rho = 5
    invalid_initial_plan = 6
    non_finite_iterate = 7
    zero_marginal = 8
    too_large = 9
    degenerate_cost = 10
    dimension_mismatch = 11
    fold_state_mismatch = 12
    bad_magic = 13
    version_unsupported = 14
    size_mismatch = 15
    ragged_csv = 16
    empty_image = 17
    k_too_large = 18
    io_error = 19
    bad_config = 20


class Error(RuntimeError):
    """drot::Error: message is "<errc_name>: <what>" (errors.hpp:75-88)."""

    def __init__(self, code: Errc, what: str):
        super().__init__(what)
        self.code = code


class DeviceError(RuntimeError):
    """A CUDA / NCCL failure inside the library (no reference counterpart)."""


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.load().drotb_last_error().decode()
    if 1 <= rc < 1000:
        raise Error(Errc(rc - 1), msg)
    raise DeviceError(f"[{rc}] {msg}")


# ---- configuration / value types -------------------------------------------
class EngineKind(enum.IntEnum):
    reference = 0
    fused = 1


class Precision(enum.IntEnum):
    f32 = 0
    f64 = 1


class Order(enum.IntEnum):
    """B200 extension: reduction order (see include/drotb.h)."""
    reference = 0
    fast = 1


class SolveStatus(enum.IntEnum):
    converged = 0
    max_iters = 1
    numerical_failure = 2


def rho0_warmup_preset(m: int) -> float:
    """solver.hpp:47-49."""
    return 1.0 / math.log(float(max(m, 3)))


@dataclass
class DrotConfig:
    rho0: float = 2.0
    rho_override: Optional[float] = None
    tol_primal: float = 1e-4
    tol_dual: float = 1e-4
    tol_gap: float = 1e-4
    relative_tolerances: bool = False
    max_iters: int = 100000
    check_every: int = 1
    engine: EngineKind = EngineKind.fused
    skip_cost: bool = True
    deterministic: bool = True
    workers: int = 0
    block_rows: int = 64
    work_size: int = 4
    record_trace: bool = True
    trace_every: int = 1
    precision: Precision = Precision.f64
    # B200 extensions
    device: int = -1
    order: Order = Order.fast
    use_graphs: bool = True

    def resolved_rho(self, m: int, n: int) -> float:
        rho = self.rho_override if self.rho_override is not None else self.rho0 / float(m + n)
        if not (rho > 0) or not math.isfinite(rho):
            raise Error(Errc.non_positive_rho, "non_positive_rho: resolved rho must be positive")
        return rho

    def to_c(self) -> drotb_config:
        c = drotb_config()
        _lib.load().drotb_config_default(C.byref(c))
        c.rho0 = self.rho0
        c.has_rho_override = 0 if self.rho_override is None else 1
        c.rho_override = 0.0 if self.rho_override is None else float(self.rho_override)
        c.tol_primal, c.tol_dual, c.tol_gap = self.tol_primal, self.tol_dual, self.tol_gap
        c.relative_tolerances = int(self.relative_tolerances)
        c.max_iters = int(self.max_iters)
        c.check_every = int(self.check_every)
        c.engine = int(self.engine)
        c.skip_cost = int(self.skip_cost)
        c.deterministic = int(self.deterministic)
        c.workers = int(self.workers)
        c.block_rows = int(self.block_rows)
        c.work_size = int(self.work_size)
        c.record_trace = int(self.record_trace)
        c.trace_every = int(self.trace_every)
        c.precision = int(self.precision)
        c.device = int(self.device)
        c.order = int(self.order)
        c.use_graphs = int(self.use_graphs)
        return c


@dataclass
class TransportProblem:
    """problem.hpp:31-39. cost: (m, n); p: (m,); q: (n,)."""
    cost: np.ndarray
    p: np.ndarray
    q: np.ndarray

    @property
    def m(self) -> int:
        return int(self.cost.shape[0])

    @property
    def n(self) -> int:
        return int(self.cost.shape[1])

    @property
    def dtype(self):
        return np.dtype(self.cost.dtype)


@dataclass
class TransportPlan:
    x: np.ndarray


@dataclass
class DualCertificate:
    mu: np.ndarray
    nu: np.ndarray
    rho: float = 1.0


@dataclass
class ResidualReport:
    r_primal: float = 0.0
    r_dual: float = 0.0
    gap: float = 0.0
    objective: float = 0.0


@dataclass
class TraceRow:
    iter: int
    r_primal: float
    r_dual: float
    gap: float
    objective: float
    ergodic_objective: float
    fixed_point_residual: float


@dataclass
class SolveTrace:
    rows: list = field(default_factory=list)
    termination: SolveStatus = SolveStatus.max_iters
    iterations: int = 0
    wall_time_s: float = 0.0


@dataclass
class SolveResult:
    plan: TransportPlan
    cert: DualCertificate
    report: ResidualReport
    trace: SolveTrace
    status: SolveStatus


# ---- helpers -----------------------------------------------------------------
def _dtype_of(problem: TransportProblem):
    dt = np.dtype(problem.cost.dtype)
    if dt not in (np.float32, np.float64):
        raise Error(Errc.bad_config, "bad_config: cost must be float32 or float64")
    return dt


def _sfx(dt) -> str:
    return "f32" if np.dtype(dt) == np.float32 else "f64"


def _ctype(dt):
    return C.c_float if np.dtype(dt) == np.float32 else C.c_double


def _cm(a, dt) -> np.ndarray:
    """Column-major contiguous copy/view of an (m, n) array."""
    return np.asfortranarray(a, dtype=dt)


def _vec(a, dt) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dt).reshape(-1)


def _p(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


# ---- solver --------------------------------------------------------------------
def check_problem(problem: TransportProblem, simplex_tol: float = 1e-12) -> None:
    """problem.hpp:122-136 (matrix scan on the GPU; marginals by the
    reference's sequential double sum against simplex_tol)."""
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    if m == 0 or n == 0:
        raise Error(Errc.empty_dimension, "empty_dimension: cost matrix has an empty dimension")
    if len(problem.p) != m or len(problem.q) != n:
        raise Error(Errc.shape_mismatch,
                    "shape_mismatch: marginal lengths do not match the cost matrix")
    lib = _lib.load()
    cm = _cm(problem.cost, dt)
    pv, qv = _vec(problem.p, dt), _vec(problem.q, dt)  # keep alive across the call
    _check(getattr(lib, "drotb_check_problem_tol_" + _sfx(dt))(_p(cm), m, n, _p(pv), _p(qv),
                                                               float(simplex_tol)))


@dataclass
class ValidateOptions:
    """problem.hpp:96-99."""
    renormalize: bool = False
    simplex_tol: float = 1e-12


def validate_problem(problem: TransportProblem,
                     opts: Optional[ValidateOptions] = None) -> TransportProblem:
    """problem.hpp:141-154: returns a checked copy; under renormalize each
    marginal is divided by its sequential double sum (then cast back to T)."""
    opts = opts or ValidateOptions()
    dt = _dtype_of(problem)
    p = np.array(problem.p, dtype=dt, copy=True)
    q = np.array(problem.q, dtype=dt, copy=True)
    if opts.renormalize:
        for v in (p, q):
            total = 0.0
            for e in v.tolist():  # ascending-index double sum, as the reference
                total += float(e)
            if total > 0:
                v[:] = (v.astype(np.float64) / total).astype(dt)
    out = TransportProblem(np.array(problem.cost, dtype=dt, order="F", copy=True), p, q)
    check_problem(out, opts.simplex_tol)
    return out


def residual_report(problem: TransportProblem, plan: TransportPlan, cert: DualCertificate,
                    exact: bool = True) -> ResidualReport:
    """residual_report (problem.hpp:174-225) evaluated on the B200.  exact=True
    sums in the reference's order (bitwise equal report); exact=False uses
    parallel trees."""
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    x = np.asarray(plan.x)
    if x.shape != (m, n):
        raise Error(Errc.shape_mismatch, "shape_mismatch: residual_report: plan vs cost")
    if len(cert.mu) != m or len(cert.nu) != n:
        raise Error(Errc.shape_mismatch, "shape_mismatch: residual_report: dual lengths")
    cm, xm = _cm(problem.cost, dt), _cm(x, dt)
    pv, qv = _vec(problem.p, dt), _vec(problem.q, dt)
    mu, nu = _vec(cert.mu, dt), _vec(cert.nu, dt)
    rep = drotb_report()
    _check(getattr(_lib.load(), "drotb_residual_report_" + _sfx(dt))(
        _p(cm), m, n, _p(pv), _p(qv), _p(xm), _p(mu), _p(nu), int(bool(exact)), C.byref(rep)))
    return ResidualReport(rep.r_primal, rep.r_dual, rep.gap, rep.objective)


def objective(problem: TransportProblem, plan: TransportPlan) -> float:
    """<C, X> in storage order (problem.hpp:158-169), on the B200."""
    m, n = problem.m, problem.n
    zeros_m, zeros_n = np.zeros(m), np.zeros(n)
    return residual_report(problem, plan, DualCertificate(zeros_m, zeros_n)).objective


def solve(problem: TransportProblem, cfg: Optional[DrotConfig] = None,
          x0: Optional[np.ndarray] = None,
          plan_out: Optional[np.ndarray] = None) -> SolveResult:
    """drot::solve<T> (solver.hpp:372-540) on the B200.  plan_out: optional
    caller-owned (m, n) Fortran-ordered buffer (e.g. pinned) for the plan."""
    cfg = cfg or DrotConfig()
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    if m == 0 or n == 0:
        raise Error(Errc.empty_dimension, "empty_dimension: cost matrix has an empty dimension")
    if len(problem.p) != m or len(problem.q) != n:
        raise Error(Errc.shape_mismatch,
                    "shape_mismatch: marginal lengths do not match the cost matrix")
    if x0 is not None and tuple(np.shape(x0)) != (m, n):
        raise Error(Errc.shape_mismatch, "shape_mismatch: initial plan shape")
    lib = _lib.load()
    ccfg = cfg.to_c()
    cm = _cm(problem.cost, dt)
    pv, qv = _vec(problem.p, dt), _vec(problem.q, dt)
    x0m = None if x0 is None else _cm(x0, dt)
    if plan_out is not None:
        if plan_out.shape != (m, n) or plan_out.dtype != dt or not plan_out.flags.f_contiguous:
            raise Error(Errc.bad_config, "bad_config: plan_out must be a Fortran-ordered "
                        "(m, n) array of the problem dtype")
        plan = plan_out
    else:
        plan = np.empty((m, n), dtype=dt, order="F")
    mu = np.empty(m, dtype=dt)
    nu = np.empty(n, dtype=dt)
    rho = _ctype(dt)(0)
    rep = drotb_report()
    cap = 0
    if cfg.record_trace:
        cap = int(min(max(cfg.max_iters, 0) // max(cfg.trace_every, 1) + 1, 1 << 23))
    trace = (drotb_trace_row * max(cap, 1))()
    tlen, iters = C.c_int64(0), C.c_int64(0)
    status, wall = C.c_int32(0), C.c_double(0)
    _check(getattr(lib, "drotb_solve_" + _sfx(dt))(
        _p(cm), m, n, _p(pv), _p(qv), C.byref(ccfg), _p(x0m), _p(plan), _p(mu), _p(nu),
        C.byref(rho), C.byref(rep), C.cast(trace, C.c_void_p), cap, C.byref(tlen),
        C.byref(iters), C.byref(status), C.byref(wall)))
    rows = []
    for k in range(min(tlen.value, cap)):
        t = trace[k]
        rows.append(TraceRow(t.iter, t.r_primal, t.r_dual, t.gap, t.objective,
                             t.ergodic_objective, t.fixed_point_residual))
    st = SolveStatus(status.value)
    return SolveResult(
        plan=TransportPlan(plan),
        cert=DualCertificate(mu, nu, float(rho.value)),
        report=ResidualReport(rep.r_primal, rep.r_dual, rep.gap, rep.objective),
        trace=SolveTrace(rows, st, int(iters.value), float(wall.value)),
        status=st)


def sinkhorn_solve(problem: TransportProblem, eta: float, tol: float, max_iters: int,
                   check_every: int = 10, exact_report: bool = False) -> SolveResult:
    """drot::sinkhorn_solve<T> (reference.hpp:165-288) on the B200: the
    paper's comparison baseline.  exact_report evaluates the final
    residual_report in the reference's summation order."""
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    if m == 0 or n == 0:
        raise Error(Errc.empty_dimension, "empty_dimension: cost matrix has an empty dimension")
    if len(problem.p) != m or len(problem.q) != n:
        raise Error(Errc.shape_mismatch,
                    "shape_mismatch: marginal lengths do not match the cost matrix")
    cm = _cm(problem.cost, dt)
    pv, qv = _vec(problem.p, dt), _vec(problem.q, dt)
    plan = np.empty((m, n), dtype=dt, order="F")
    mu = np.empty(m, dtype=dt)
    nu = np.empty(n, dtype=dt)
    rep = drotb_report()
    ce = max(int(check_every), 1)
    cap = int(max(int(max_iters), 0) // ce + 2)
    trace = (drotb_trace_row * cap)()
    tlen, iters = C.c_int64(0), C.c_int64(0)
    status, wall = C.c_int32(0), C.c_double(0)
    _check(getattr(_lib.load(), "drotb_sinkhorn_" + _sfx(dt))(
        _p(cm), m, n, _p(pv), _p(qv), _ctype(dt)(eta), float(tol), int(max_iters), ce,
        int(bool(exact_report)), _p(plan), _p(mu), _p(nu), C.byref(rep),
        C.cast(trace, C.c_void_p), cap, C.byref(tlen), C.byref(iters), C.byref(status),
        C.byref(wall)))
    rows = [TraceRow(trace[k].iter, trace[k].r_primal, trace[k].r_dual, trace[k].gap,
                     trace[k].objective, trace[k].ergodic_objective,
                     trace[k].fixed_point_residual) for k in range(min(tlen.value, cap))]
    st = SolveStatus(status.value)
    return SolveResult(
        plan=TransportPlan(plan),
        cert=DualCertificate(mu, nu, float(eta)),
        report=ResidualReport(rep.r_primal, rep.r_dual, rep.gap, rep.objective),
        trace=SolveTrace(rows, st, int(iters.value), float(wall.value)),
        status=st)


@dataclass
class FusedArray:
    """fused.hpp:64-68."""
    values: np.ndarray
    cost_folded: bool = False


@dataclass
class DrotState:
    """solver.hpp:98-114 (host copy; the device owns it during a step)."""
    xy: FusedArray
    row_shift: np.ndarray
    col_shift: np.ndarray
    y_row_defect: np.ndarray
    y_col_defect: np.ndarray
    y_mass_gap: float
    row_residual: np.ndarray
    col_residual: np.ndarray
    x_mass_gap: float
    iter: int = 0


def _state_call(fn_name, problem, cfg, st: DrotState, x0=None):
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    lib = _lib.load()
    ct = _ctype(dt)
    folded = C.c_int32(int(st.xy.cost_folded))
    alpha, beta = ct(st.y_mass_gap), ct(st.x_mass_gap)
    it = C.c_int64(st.iter)
    for name in ("row_shift", "col_shift", "y_row_defect", "y_col_defect", "row_residual",
                 "col_residual"):
        arr = getattr(st, name)
        if not (isinstance(arr, np.ndarray) and arr.dtype == dt and arr.flags.c_contiguous):
            raise Error(Errc.bad_config, f"bad_config: state.{name} must be a contiguous {dt} array")
    if not (st.xy.values.dtype == dt and st.xy.values.flags.f_contiguous):
        raise Error(Errc.bad_config, "bad_config: state.xy must be a Fortran-ordered array")
    keep = [_cm(problem.cost, dt), _vec(problem.p, dt), _vec(problem.q, dt),
            None if x0 is None else _cm(x0, dt)]  # alive across the call
    args = [_p(st.xy.values), C.byref(folded), _p(st.row_shift), _p(st.col_shift),
            _p(st.y_row_defect), _p(st.y_col_defect), C.byref(alpha), _p(st.row_residual),
            _p(st.col_residual), C.byref(beta), C.byref(it),
            _p(keep[0]), m, n, _p(keep[1]), _p(keep[2])]
    if x0 is not None or fn_name.startswith("drotb_init_state"):
        args.append(_p(keep[3]))
    ccfg = cfg.to_c()
    args.append(C.byref(ccfg))
    rc = getattr(lib, fn_name + "_" + _sfx(dt))(*args)
    st.xy.cost_folded = bool(folded.value)
    st.y_mass_gap = float(alpha.value)
    st.x_mass_gap = float(beta.value)
    st.iter = int(it.value)
    _check(rc)


def init_state(problem: TransportProblem, cfg: Optional[DrotConfig] = None,
               x0: Optional[np.ndarray] = None) -> DrotState:
    """drot::init_state<T> (solver.hpp:143-186), computed on the device."""
    cfg = cfg or DrotConfig()
    dt = _dtype_of(problem)
    m, n = problem.m, problem.n
    if x0 is not None and tuple(np.shape(x0)) != (m, n):
        raise Error(Errc.shape_mismatch, "shape_mismatch: initial plan shape")
    st = DrotState(FusedArray(np.empty((m, n), dt, order="F"), False),
                   np.empty(m, dt), np.empty(n, dt), np.empty(m, dt), np.empty(n, dt), 0.0,
                   np.empty(m, dt), np.empty(n, dt), 0.0, 0)
    _state_call("drotb_init_state", problem, cfg, st, x0)
    return st


def drot_step(st: DrotState, problem: TransportProblem,
              cfg: Optional[DrotConfig] = None) -> None:
    """drot::drot_step<T> (solver.hpp:361-370): one iteration in place;
    raises Error(non_finite_iterate) on overflow like the reference."""
    cfg = cfg or DrotConfig()
    _state_call("drotb_step", problem, cfg, st)


def _materialize(st: DrotState, cost, rho: float, want_y: bool) -> np.ndarray:
    xy = st.xy.values
    dt = xy.dtype
    m, n = xy.shape
    out = np.empty((m, n), dt, order="F")
    if m == 0 or n == 0:
        return out
    if st.xy.cost_folded and tuple(np.shape(cost)) != (m, n):
        raise Error(Errc.shape_mismatch, "shape_mismatch: materialize: array vs cost")
    xm = _cm(xy, dt)
    cm = _cm(cost, dt) if st.xy.cost_folded else None
    lib = _lib.load()
    if want_y:
        rs, cs = _vec(st.row_shift, dt), _vec(st.col_shift, dt)
        if len(rs) != m or len(cs) != n:
            raise Error(Errc.shape_mismatch, "shape_mismatch: materialize_y: shift lengths")
        _check(getattr(lib, "drotb_materialize_y_" + _sfx(dt))(
            _p(xm), int(st.xy.cost_folded), _p(cm), _p(rs), _p(cs), m, n, rho, _p(out)))
    else:
        _check(getattr(lib, "drotb_materialize_plan_" + _sfx(dt))(
            _p(xm), int(st.xy.cost_folded), _p(cm), m, n, rho, _p(out)))
    return out


def materialize_plan(st: DrotState, cost, rho: float) -> TransportPlan:
    """solver.hpp:204-217 on the device: the plan iterate, unfolded and
    clamped when the array holds X - rho C."""
    return TransportPlan(_materialize(st, cost, rho, False))


def materialize_y(st: DrotState, cost, rho: float) -> np.ndarray:
    """solver.hpp:219-230 on the device: Y = X + phi e' + f varphi'."""
    return _materialize(st, cost, rho, True)


class ErgodicMean:
    """solver.hpp:127-139: running mean of the per-iterate objectives."""

    def __init__(self):
        self._mean = 0.0
        self._count = 0

    def update(self, value: float) -> None:
        self._count += 1
        self._mean += (float(value) - self._mean) / float(self._count)

    def mean(self) -> float:
        return self._mean

    def count(self) -> int:
        return self._count


def recover_duals(st: DrotState, rho: float) -> DualCertificate:
    """solver.hpp:188-199 (mu = phi / rho in T)."""
    dt = st.row_shift.dtype
    r = dt.type(rho)
    return DualCertificate(st.row_shift / r, st.col_shift / r, float(r))


# ---- engine ---------------------------------------------------------------------
@dataclass
class MemoryCounters:
    """fused.hpp:34-39."""
    passes: int = 0
    xy_elems_read: int = 0
    xy_elems_written: int = 0
    cost_elems_read: int = 0


@dataclass
class PassOptions:
    """fused.hpp:70-81."""
    parity: int = 0
    want_dual: bool = False
    want_dx: bool = False
    deterministic: bool = True
    counters: Optional[MemoryCounters] = None


@dataclass
class FusedPassOutput:
    """fused.hpp:42-60."""
    row_sums: np.ndarray
    col_sums: np.ndarray
    cost_dot: float = 0.0
    cost_valid: bool = False
    max_abs: float = 0.0
    nonfinite: bool = False
    dual_sq: float = 0.0
    dual_valid: bool = False
    dx_sq: float = 0.0
    dx_valid: bool = False
    prev_cost_dot: float = 0.0
    prev_cost_valid: bool = False

    def total_mass(self):
        acc = self.row_sums.dtype.type(0)
        for x in self.row_sums:
            acc = acc + x
        return acc


@dataclass
class TileRange:
    """tiles.hpp:22-33."""
    r0: int
    r1: int
    c0: int
    c1: int
    grid_r: int
    grid_c: int

    def rows(self):
        return self.r1 - self.r0

    def cols(self):
        return self.c1 - self.c0

    def size(self):
        return self.rows() * self.cols()


@dataclass
class TilePlan:
    """tiles.hpp:37-46 (the reduction tree the GPU reproduces)."""
    rows: int
    cols: int
    block_rows: int = 64
    work_size: int = 4
    workers: int = 1

    @property
    def grid_rows(self):
        return -(-self.rows // self.block_rows)

    @property
    def grid_cols(self):
        return -(-self.cols // (self.block_rows * self.work_size))

    def tile_cols(self):
        return self.work_size * self.block_rows

    @property
    def tiles(self):
        """Tile-column-major list = the reference's reduction order
        (tiles.cpp:33-44)."""
        tc = self.tile_cols()
        return [TileRange(gr * self.block_rows, min(self.rows, (gr + 1) * self.block_rows),
                          gc * tc, min(self.cols, (gc + 1) * tc), gr, gc)
                for gc in range(self.grid_cols) for gr in range(self.grid_rows)]


def plan_tiles(m: int, n: int, bs: int = 64, ws: int = 4, workers: int = 1) -> TilePlan:
    """tiles.cpp:20-47."""
    return TilePlan(m, n, max(1, bs), max(1, ws), max(1, workers))


class FusedEngine:
    """drot::FusedEngine<T> (fused.hpp:107-202) backed by the sm_100a sweep."""

    def __init__(self, plan: TilePlan, dtype=np.float64, device: int = -1):
        self.plan = plan
        self.dtype = np.dtype(dtype)
        lib = _lib.load()
        h = C.c_void_p()
        _check(lib.drotb_engine_create(C.byref(h), plan.rows, plan.cols, plan.block_rows,
                                       plan.work_size, 0 if self.dtype == np.float32 else 1,
                                       device))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().drotb_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_shapes(self, xy, cost, row_shift, col_shift):
        m, n = self.plan.rows, self.plan.cols
        if xy.shape != (m, n):
            raise Error(Errc.shape_mismatch, "shape_mismatch: fused pass: array vs tile plan")
        if cost.shape != xy.shape:
            raise Error(Errc.shape_mismatch, "shape_mismatch: fused pass: cost")
        if len(row_shift) != m or len(col_shift) != n:
            raise Error(Errc.shape_mismatch, "shape_mismatch: fused pass: shift vectors")

    def _run(self, xy: np.ndarray, cost, row_shift, col_shift, rho, kind, fold, folded,
             opts: PassOptions):
        self._check_shapes(xy, cost, row_shift, col_shift)
        dt = self.dtype
        if not (xy.flags.f_contiguous and xy.dtype == dt):
            raise Error(Errc.bad_config, "bad_config: xy must be a Fortran-ordered array of the engine dtype")
        m, n = self.plan.rows, self.plan.cols
        row = np.empty(m, dt)
        col = np.empty(n, dt)
        out = drotb_pass_out()
        ctr = drotb_counters()
        if opts.counters is not None:
            c = opts.counters
            ctr.passes, ctr.xy_elems_read = c.passes, c.xy_elems_read
            ctr.xy_elems_written, ctr.cost_elems_read = c.xy_elems_written, c.cost_elems_read
        fl = C.c_int32(int(folded))
        lib = _lib.load()
        keep = [_cm(cost, dt), _vec(row_shift, dt), _vec(col_shift, dt)]
        _check(getattr(lib, "drotb_engine_pass_" + _sfx(dt))(
            self._h, _p(xy), _p(keep[0]), _p(keep[1]),
            _p(keep[2]), _ctype(dt)(rho), kind, int(fold), C.byref(fl),
            int(opts.parity), int(opts.want_dual), int(opts.want_dx),
            int(opts.deterministic), _p(row), _p(col), C.byref(out), C.byref(ctr)))
        if opts.counters is not None:
            c = opts.counters
            c.passes, c.xy_elems_read = ctr.passes, ctr.xy_elems_read
            c.xy_elems_written, c.cost_elems_read = ctr.xy_elems_written, ctr.cost_elems_read
        res = FusedPassOutput(row, col, out.cost_dot, bool(out.cost_valid), out.max_abs,
                              bool(out.nonfinite), out.dual_sq, bool(out.dual_valid),
                              out.dx_sq, bool(out.dx_valid), out.prev_cost_dot,
                              bool(out.prev_cost_valid))
        return res, bool(fl.value)

    def fused_pass(self, xy: np.ndarray, cost, row_shift, col_shift, rho,
                   opts: Optional[PassOptions] = None) -> FusedPassOutput:
        return self._run(xy, cost, row_shift, col_shift, rho, 0, 0, False,
                         opts or PassOptions())[0]

    def fused_pass_skip_cost(self, xy: FusedArray, cost, row_shift, col_shift, rho,
                             fold: bool, opts: Optional[PassOptions] = None) -> FusedPassOutput:
        res, folded = self._run(xy.values, cost, row_shift, col_shift, rho, 1, fold,
                                xy.cost_folded, opts or PassOptions())
        xy.cost_folded = folded
        return res

    def unfused_pass(self, xy: np.ndarray, cost, row_shift, col_shift, rho,
                     opts: Optional[PassOptions] = None) -> FusedPassOutput:
        """EngineKind::reference: same outputs as the fused sweep (bitwise in
        deterministic mode, test_fused.cpp:123-137); counted as 4 sweeps."""
        return self._run(xy, cost, row_shift, col_shift, rho, 2, 0, False,
                         opts or PassOptions())[0]


# ---- generators (probgen.hpp) ------------------------------------------------
@dataclass
class GaussianSpec:
    m: int = 0
    n: int = 0
    sigma_t: float = 5.0
    seed: int = 0
    dirichlet_marginals: bool = False


def gen_gaussian_problem(spec: GaussianSpec) -> TransportProblem:
    """probgen.hpp:131-170 (double precision, bit-identical)."""
    lib = _lib.load()
    cost = np.empty((spec.m, spec.n), np.float64, order="F")
    p = np.empty(spec.m, np.float64)
    q = np.empty(spec.n, np.float64)
    _check(lib.drotb_gen_gaussian(spec.m, spec.n, spec.sigma_t, spec.seed,
                                  int(spec.dirichlet_marginals), _p(cost), _p(p), _p(q)))
    return TransportProblem(cost, p, q)


def gen_gaussian_problem_as(spec: GaussianSpec, dtype) -> TransportProblem:
    """probgen.hpp:172-180."""
    dt = np.dtype(dtype)
    if dt == np.float64:
        return gen_gaussian_problem(spec)
    lib = _lib.load()
    cost = np.empty((spec.m, spec.n), np.float32, order="F")
    _check(lib.drotb_gen_gaussian_f32(spec.m, spec.n, spec.sigma_t, spec.seed, _p(cost)))
    if spec.dirichlet_marginals:
        pd = np.empty(spec.m, np.float64)
        qd = np.empty(spec.n, np.float64)
        tmp = np.empty((spec.m, spec.n), np.float64, order="F")
        _check(lib.drotb_gen_gaussian(spec.m, spec.n, spec.sigma_t, spec.seed, 1,
                                      _p(tmp), _p(pd), _p(qd)))
        return TransportProblem(cost, pd.astype(dt), qd.astype(dt))
    p = np.full(spec.m, 1.0 / spec.m).astype(dt)
    q = np.full(spec.n, 1.0 / spec.n).astype(dt)
    return TransportProblem(cost, p, q)


def counter_uniform(seed: int, count: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """lo + (hi-lo) * CounterRng(seed).next_unit(), outputs 1..count (rng.hpp:49-57)."""
    out = np.empty(count, np.float64)
    _check(_lib.load().drotb_counter_uniform(seed, count, lo, hi, _p(out)))
    return out


def random_matrix(m: int, n: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """The reference fixture random_matrix (tests/support/oracles.hpp:128-135),
    column-major (m, n)."""
    return counter_uniform(seed, m * n, lo, hi).reshape((m, n), order="F")


def dyadic_marginal(length: int, dtype=np.float64) -> np.ndarray:
    """Exact-sum simplex vector accepted by check_problem at any size (B200
    input fix)."""
    dt = np.dtype(dtype)
    out = np.empty(length, dt)
    _check(getattr(_lib.load(), "drotb_dyadic_marginal_" + _sfx(dt))(length, _p(out)))
    return out


def release_device_cache() -> None:
    """Free the device context solve() keeps for repeated solves of one shape."""
    _lib.load().drotb_release_cache()


def kernel_launches() -> int:
    return int(_lib.load().drotb_kernel_launches())
