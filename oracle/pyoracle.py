"""ctypes front end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Two interchangeable back ends with identical entry points:

* ``Oracle("ref")`` -> ``oracle/_ref/libdrotref.so``: the unmodified reference
  library (/root/reference/proj/core) compiled from its own sources by
  ``oracle/Makefile`` and wrapped by ``oracle/ref_shim.cpp``.
* ``Oracle("orc")`` -> ``oracle/build/liborc.so``: the plain-C restatement
  ``oracle/drot_oracle.c``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "ref": os.path.join(HERE, "_ref", "libdrotref.so"),
    "orc": os.path.join(HERE, "build", "liborc.so"),
}

ERRC_NAMES = [
    "negative_cost", "marginal_not_simplex", "empty_dimension",
    "non_finite_entry", "shape_mismatch", "non_positive_rho",
    "invalid_initial_plan", "non_finite_iterate", "zero_marginal", "too_large",
    "degenerate_cost", "dimension_mismatch", "fold_state_mismatch", "bad_magic",
    "version_unsupported", "size_mismatch", "ragged_csv", "empty_image",
    "k_too_large", "io_error", "bad_config",
]
STATUS_NAMES = ["converged", "max_iters", "numerical_failure"]
PASS_FUSED, PASS_SKIP_COST, PASS_UNFUSED = 0, 1, 2


class OrcConfig(C.Structure):
    _fields_ = [
        ("rho0", C.c_double), ("has_rho_override", C.c_int32),
        ("relative_tolerances", C.c_int32), ("rho_override", C.c_double),
        ("tol_primal", C.c_double), ("tol_dual", C.c_double),
        ("tol_gap", C.c_double), ("max_iters", C.c_int64),
        ("check_every", C.c_int64), ("engine", C.c_int32),
        ("skip_cost", C.c_int32), ("deterministic", C.c_int32),
        ("record_trace", C.c_int32), ("workers", C.c_int64),
        ("block_rows", C.c_int64), ("work_size", C.c_int64),
        ("trace_every", C.c_int64),
    ]


class OrcReport(C.Structure):
    _fields_ = [("r_primal", C.c_double), ("r_dual", C.c_double),
                ("gap", C.c_double), ("objective", C.c_double)]


class OrcTraceRow(C.Structure):
    _fields_ = [("iter", C.c_int64), ("r_primal", C.c_double),
                ("r_dual", C.c_double), ("gap", C.c_double),
                ("objective", C.c_double), ("ergodic_objective", C.c_double),
                ("fixed_point_residual", C.c_double)]


class OrcPassOut(C.Structure):
    _fields_ = [("cost_dot", C.c_double), ("max_abs", C.c_double),
                ("dual_sq", C.c_double), ("dx_sq", C.c_double),
                ("prev_cost_dot", C.c_double), ("cost_valid", C.c_int32),
                ("nonfinite", C.c_int32), ("dual_valid", C.c_int32),
                ("dx_valid", C.c_int32), ("prev_cost_valid", C.c_int32),
                ("pad_", C.c_int32)]


class OrcCounters(C.Structure):
    _fields_ = [("passes", C.c_uint64), ("xy_elems_read", C.c_uint64),
                ("xy_elems_written", C.c_uint64), ("cost_elems_read", C.c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, code: int, name: str):
        super().__init__(name)
        self.code = code
        self.name = name


def default_config(**kw) -> OrcConfig:
    """drot::DrotConfig defaults (solver.hpp:51-88)."""
    c = OrcConfig(rho0=2.0, has_rho_override=0, relative_tolerances=0,
                  rho_override=0.0, tol_primal=1e-4, tol_dual=1e-4, tol_gap=1e-4,
                  max_iters=100000, check_every=1, engine=1, skip_cost=1,
                  deterministic=1, record_trace=1, workers=0, block_rows=64,
                  work_size=4, trace_every=1)
    for k, v in kw.items():
        if k == "rho_override":
            c.has_rho_override = 1
        setattr(c, k, v)
    return c


@dataclass
class SolveOut:
    plan: np.ndarray
    mu: np.ndarray
    nu: np.ndarray
    report: dict
    iterations: int
    status: str
    trace: list = field(default_factory=list)
    wall_time_s: float = 0.0


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, kind: str = "orc"):
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = "ref_" if kind == "ref" else "orc_"

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc:
            raise OracleError(rc - 1, ERRC_NAMES[rc - 1])

    @staticmethod
    def _sfx(dtype):
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    # -- problems -----------------------------------------------------------
    def gen_gaussian(self, m, n, sigma_t=5.0, seed=0, dirichlet=False):
        Cm = np.empty((n, m), np.float64)  # column-major m x n == C-order (n, m)
        p = np.empty(m, np.float64)
        q = np.empty(n, np.float64)
        f = self._fn("gen_gaussian")
        f.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_int32,
                      C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(m, n, sigma_t, seed, int(dirichlet), _ptr(Cm), _ptr(p), _ptr(q)))
        return Cm.reshape(-1), p, q

    def random_unit(self, seed, count, lo=0.0, hi=1.0):
        out = np.empty(count, np.float64)
        f = self._fn("random_unit")
        f.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, C.c_void_p]
        f.restype = None
        f(seed, count, lo, hi, _ptr(out))
        return out

    # -- engine -------------------------------------------------------------
    def fused_pass(self, xy, cost, phi, varphi, rho, m, n, *, bs=64, ws=4,
                   workers=1, kind=PASS_FUSED, fold=False, folded=False,
                   parity=0, want_dual=False, want_dx=False, deterministic=True,
                   counters=None):
        dt = xy.dtype
        sfx = self._sfx(dt)
        ctype = C.c_float if sfx == "f32" else C.c_double
        xy = np.ascontiguousarray(xy).copy()
        row = np.empty(m, dt)
        col = np.empty(n, dt)
        out = OrcPassOut()
        fl = C.c_int32(int(folded))
        f = self._fn("pass_" + sfx)
        if self.kind == "ref":
            f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                          C.c_void_p, ctype, C.c_int64, C.c_int64, C.c_int64,
                          C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                          C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                          C.POINTER(OrcPassOut), C.POINTER(OrcCounters)]
            rc = f(_ptr(xy), _ptr(np.ascontiguousarray(cost, dt)), m, n,
                   _ptr(np.ascontiguousarray(phi, dt)),
                   _ptr(np.ascontiguousarray(varphi, dt)), rho, bs, ws, workers,
                   kind, int(fold), C.byref(fl), parity, int(want_dual),
                   int(want_dx), int(deterministic), _ptr(row), _ptr(col),
                   C.byref(out), C.byref(counters) if counters is not None else None)
        else:
            f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                          C.c_void_p, ctype, C.c_int64, C.c_int64,
                          C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                          C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                          C.POINTER(OrcPassOut), C.POINTER(OrcCounters)]
            rc = f(_ptr(xy), _ptr(np.ascontiguousarray(cost, dt)), m, n,
                   _ptr(np.ascontiguousarray(phi, dt)),
                   _ptr(np.ascontiguousarray(varphi, dt)), rho, bs, ws,
                   kind, int(fold), C.byref(fl), parity, int(want_dual),
                   int(want_dx), _ptr(row), _ptr(col),
                   C.byref(out), C.byref(counters) if counters is not None else None)
        self._check(rc)
        res = {k: getattr(out, k) for k, _ in OrcPassOut._fields_ if k != "pad_"}
        res.update(row_sums=row, col_sums=col, xy=xy, folded=bool(fl.value))
        return res

    # -- solver -------------------------------------------------------------
    def solve(self, cost, p, q, m, n, cfg: OrcConfig | None = None, x0=None,
              trace_cap=None):
        dt = np.asarray(p).dtype
        sfx = self._sfx(dt)
        cfg = cfg or default_config()
        plan = np.empty(m * n, dt)
        mu = np.empty(m, dt)
        nu = np.empty(n, dt)
        rep = OrcReport()
        if trace_cap is None:
            trace_cap = cfg.max_iters if cfg.record_trace else 0
        trace_cap = int(min(trace_cap, 10_000_000))
        trace = (OrcTraceRow * max(trace_cap, 1))()
        tlen = C.c_int64(0)
        iters = C.c_int64(0)
        status = C.c_int32(0)
        wall = C.c_double(0)
        f = self._fn("solve_" + sfx)
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                      C.POINTER(OrcConfig), C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.POINTER(OrcReport), C.c_void_p, C.c_int64,
                      C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                      C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        x0a = None if x0 is None else np.ascontiguousarray(x0, dt)
        rc = f(_ptr(np.ascontiguousarray(cost, dt)), m, n,
               _ptr(np.ascontiguousarray(p, dt)), _ptr(np.ascontiguousarray(q, dt)),
               C.byref(cfg), _ptr(x0a), _ptr(plan), _ptr(mu), _ptr(nu),
               C.byref(rep), C.cast(trace, C.c_void_p), trace_cap, C.byref(tlen),
               C.byref(iters), C.byref(status), C.byref(wall))
        self._check(rc)
        rows = [{k: getattr(trace[i], k) for k, _ in OrcTraceRow._fields_}
                for i in range(min(tlen.value, trace_cap))]
        return SolveOut(plan=plan, mu=mu, nu=nu,
                        report={k: getattr(rep, k) for k, _ in OrcReport._fields_},
                        iterations=iters.value, status=STATUS_NAMES[status.value],
                        trace=rows, wall_time_s=wall.value)

    def steps(self, cost, p, q, m, n, k, cfg: OrcConfig | None = None):
        """init_state + k x drot_step; returns the raw state + state_report."""
        dt = np.asarray(p).dtype
        sfx = self._sfx(dt)
        cfg = cfg or default_config()
        ctype = C.c_float if sfx == "f32" else C.c_double
        xy = np.empty(m * n, dt)
        phi, a, r = (np.empty(m, dt) for _ in range(3))
        varphi, b, s = (np.empty(n, dt) for _ in range(3))
        alpha, beta = ctype(0), ctype(0)
        folded = C.c_int32(0)
        rep = OrcReport()
        f = self._fn("steps_" + sfx)
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                      C.POINTER(OrcConfig), C.c_int64, C.c_void_p,
                      C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.POINTER(ctype), C.c_void_p, C.c_void_p,
                      C.POINTER(ctype), C.POINTER(OrcReport)]
        rc = f(_ptr(np.ascontiguousarray(cost, dt)), m, n,
               _ptr(np.ascontiguousarray(p, dt)), _ptr(np.ascontiguousarray(q, dt)),
               C.byref(cfg), k, _ptr(xy), C.byref(folded), _ptr(phi), _ptr(varphi),
               _ptr(a), _ptr(b), C.byref(alpha), _ptr(r), _ptr(s), C.byref(beta),
               C.byref(rep))
        self._check(rc)
        return dict(xy=xy, folded=bool(folded.value), phi=phi, varphi=varphi, a=a,
                    b=b, alpha=alpha.value, r=r, s=s, beta=beta.value,
                    report={k2: getattr(rep, k2) for k2, _ in OrcReport._fields_})

    def check_problem(self, cost, p, q, m, n):
        dt = np.asarray(p).dtype
        f = self._fn("check_problem_" + self._sfx(dt))
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        self._check(f(_ptr(np.ascontiguousarray(cost, dt)), m, n,
                      _ptr(np.ascontiguousarray(p, dt)),
                      _ptr(np.ascontiguousarray(q, dt))))

    def residual_report(self, cost, p, q, plan, mu, nu, m, n):
        dt = np.asarray(p).dtype
        f = self._fn("residual_report_" + self._sfx(dt))
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(OrcReport)]
        rep = OrcReport()
        arrs = [np.ascontiguousarray(a, dt) for a in (cost, p, q, plan, mu, nu)]
        self._check(f(_ptr(arrs[0]), m, n, *[_ptr(a) for a in arrs[1:]], C.byref(rep)))
        return {k: getattr(rep, k) for k, _ in OrcReport._fields_}

    # -- reference-only helpers ---------------------------------------------
    def time_iters(self, cost, p, q, m, n, k, cfg: OrcConfig | None = None, warm: int = 1):
        """Seconds per solve-loop iteration: (solve(max_iters=warm+k) -
        solve(max_iters=warm)) / k, cfg as given otherwise (tolerances made
        unreachable).  Returns (s/iter, total seconds of the two calls)."""
        assert self.kind == "ref"
        dt = np.asarray(p).dtype
        f = self._fn("time_iters_" + self._sfx(dt))
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                      C.POINTER(OrcConfig), C.c_int64, C.c_int64, C.POINTER(C.c_double),
                      C.POINTER(C.c_double)]
        spi, tot = C.c_double(0), C.c_double(0)
        cfg = cfg or default_config()
        self._check(f(_ptr(np.ascontiguousarray(cost, dt)), m, n,
                      _ptr(np.ascontiguousarray(p, dt)),
                      _ptr(np.ascontiguousarray(q, dt)), C.byref(cfg), k, max(1, warm),
                      C.byref(spi), C.byref(tot)))
        return spi.value, tot.value

    def sinkhorn(self, cost, p, q, m, n, eta, tol, max_iters, check_every=10):
        """drot::sinkhorn_solve<T> (reference only)."""
        assert self.kind == "ref"
        dt = np.asarray(p).dtype
        sfx = self._sfx(dt)
        tc = C.c_float if dt == np.float32 else C.c_double
        plan = np.empty(m * n, dt)
        mu = np.empty(m, dt)
        nu = np.empty(n, dt)
        rep = OrcReport()
        cap = max(int(max_iters) // max(int(check_every), 1) + 2, 1)
        trace = (OrcTraceRow * cap)()
        tlen, iters = C.c_int64(0), C.c_int64(0)
        status, wall = C.c_int32(0), C.c_double(0)
        f = self._fn("sinkhorn_" + sfx)
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, tc, C.c_double,
                      C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.POINTER(OrcReport), C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                      C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        self._check(f(_ptr(np.ascontiguousarray(cost, dt)), m, n,
                      _ptr(np.ascontiguousarray(p, dt)), _ptr(np.ascontiguousarray(q, dt)),
                      eta, tol, max_iters, check_every, _ptr(plan), _ptr(mu), _ptr(nu),
                      C.byref(rep), C.cast(trace, C.c_void_p), cap, C.byref(tlen),
                      C.byref(iters), C.byref(status), C.byref(wall)))
        rows = [{k: getattr(trace[i], k) for k, _ in OrcTraceRow._fields_}
                for i in range(min(tlen.value, cap))]
        return SolveOut(plan=plan, mu=mu, nu=nu,
                        report={k: getattr(rep, k) for k, _ in OrcReport._fields_},
                        iterations=iters.value, status=STATUS_NAMES[status.value],
                        trace=rows, wall_time_s=wall.value)

    def lp_exact(self, cost, p, q, m, n):
        assert self.kind == "ref"
        f = self._fn("lp_exact")
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                      C.POINTER(C.c_double), C.c_void_p]
        obj = C.c_double(0)
        plan = np.empty(m * n, np.float64)
        arrs = [np.ascontiguousarray(a, np.float64) for a in (cost, p, q)]
        self._check(f(_ptr(arrs[0]), m, n, _ptr(arrs[1]), _ptr(arrs[2]),
                      C.byref(obj), _ptr(plan)))
        return obj.value, plan

    def hardware_workers(self):
        assert self.kind == "ref"
        f = self._fn("hardware_workers")
        f.restype = C.c_int64
        return f()


def dyadic_marginal(length: int, dtype=np.float64) -> np.ndarray:
    """Uniform-as-possible simplex vector whose entries are exact multiples of
    2^-K summing to exactly 1, so that the reference's
    |sum-1| <= 1e-12 validation accepts it in fp32 and at any size."""
    K = (23 if np.dtype(dtype) == np.float32 else 52) + int(np.floor(np.log2(length)))
    K = min(K, 52)
    total = 1 << K
    base = total // length
    extra = total - base * length
    k = np.full(length, base, dtype=np.int64)
    k[:extra] += 1
    return (k.astype(np.float64) * 2.0 ** (-K)).astype(dtype)
