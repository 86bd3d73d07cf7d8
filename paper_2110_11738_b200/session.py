"""Device-resident solve session (benchmarks, multi-GPU shards).

A Session owns the device copies of C, p, q and the DrotState and runs the
same iteration as drot::solve (solver.hpp:372-540), enqueued as CUDA graphs
on one stream.  It is the B200 replacement of keeping a FusedEngine alive
and calling detail::step_impl in a loop (solver.hpp:358-360).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .api import (DrotConfig, Error, Errc, ResidualReport, SolveStatus, _check, _cm,
                  _p, _vec)
from ._lib import drotb_report


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.load().drotb_nccl_unique_id(buf))
    return buf.raw


def shard_rows(m: int, world: int, rank: int):
    """Row range of `rank` (contiguous, 64-row aligned, balanced)."""
    r0, r1 = C.c_int64(0), C.c_int64(0)
    _check(_lib.load().drotb_shard_rows(int(m), int(world), int(rank), C.byref(r0), C.byref(r1)))
    return int(r0.value), int(r1.value)


class Session:
    MARGINALS = {"uniform": 0, "dyadic": 1, "dirichlet": 2, "random_simplex": 3}

    def __init__(self, m: int, n: int, dtype=np.float32, cfg: Optional[DrotConfig] = None):
        self.m, self.n = int(m), int(n)
        self.dtype = np.dtype(dtype)
        self.cfg = cfg or DrotConfig()
        lib = _lib.load()
        h = C.c_void_p()
        ccfg = self.cfg.to_c()
        _check(lib.drotb_session_create(C.byref(h), self.m, self.n,
                                        0 if self.dtype == np.float32 else 1, C.byref(ccfg)))
        self._h = h

    @classmethod
    def sharded(cls, m_global: int, n: int, dtype, cfg: Optional[DrotConfig], rank: int,
                world: int, nccl_id: bytes, row_begin: int, row_end: int) -> "Session":
        """Row shard [row_begin, row_end) of an m_global x n problem (one process
        per GPU, NCCL collectives)."""
        self = cls.__new__(cls)
        self.m, self.n = int(row_end - row_begin), int(n)
        self.m_global, self.row_begin = int(m_global), int(row_begin)
        self.dtype = np.dtype(dtype)
        self.cfg = cfg or DrotConfig()
        h = C.c_void_p()
        ccfg = self.cfg.to_c()
        _check(_lib.load().drotb_session_create_sharded(
            C.byref(h), int(m_global), int(n), 0 if self.dtype == np.float32 else 1,
            C.byref(ccfg), int(rank), int(world), nccl_id, int(row_begin), int(row_end)))
        self._h = h
        return self

    @classmethod
    def sharded_p2p(cls, m_global: int, n: int, dtype, cfg: Optional[DrotConfig], rank: int,
                    world: int, row_begin: int, row_end: int) -> "Session":
        """Row shard whose per-iteration exchange is fused into the cooperative
        tail over NVLink peer memory (no NCCL).  Call attach_peers() with every
        rank's exchange_pointer() (same process) or exchange_handle() (one
        process per GPU) before set_problem / gen_*."""
        self = cls.__new__(cls)
        self.m, self.n = int(row_end - row_begin), int(n)
        self.m_global, self.row_begin = int(m_global), int(row_begin)
        self.dtype = np.dtype(dtype)
        self.cfg = cfg or DrotConfig()
        h = C.c_void_p()
        ccfg = self.cfg.to_c()
        _check(_lib.load().drotb_session_create_sharded_p2p(
            C.byref(h), int(m_global), int(n), 0 if self.dtype == np.float32 else 1,
            C.byref(ccfg), int(rank), int(world), int(row_begin), int(row_end)))
        self._h = h
        return self

    def exchange_pointer(self) -> int:
        ptr = C.c_uint64(0)
        _check(_lib.load().drotb_session_exchange_buffer(self._h, C.byref(ptr), None))
        return int(ptr.value)

    def exchange_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        _check(_lib.load().drotb_session_exchange_buffer(self._h, None, buf))
        return buf.raw

    def attach_peers(self, pointers=None, handles=None):
        if pointers is not None:
            arr = (C.c_uint64 * len(pointers))(*[int(x) for x in pointers])
            _check(_lib.load().drotb_session_attach_peers(self._h, C.cast(arr, C.c_void_p), None))
        else:
            blob = b"".join(bytes(h).ljust(64, b"\0")[:64] for h in handles)
            _check(_lib.load().drotb_session_attach_peers(self._h, None, blob))

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().drotb_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: Optional[int]):
        _check(_lib.load().drotb_session_set_stream(self._h, stream_ptr))

    @property
    def stream(self) -> int:
        return _lib.load().drotb_session_stream(self._h)

    def set_problem(self, cost: np.ndarray, p: np.ndarray, q: np.ndarray):
        dt = self.dtype
        cm, pv, qv = _cm(cost, dt), _vec(p, dt), _vec(q, dt)  # alive across the call
        _check(_lib.load().drotb_session_set_problem(self._h, _p(cm), _p(pv), _p(qv), 0))

    def set_problem_device(self, cost_ptr: int, p_ptr: int, q_ptr: int):
        _check(_lib.load().drotb_session_set_problem(self._h, cost_ptr, p_ptr, q_ptr, 1))

    def gen_gaussian(self, sigma_t: float = 5.0, seed: int = 0, marginals: str = "dyadic"):
        _check(_lib.load().drotb_session_gen_gaussian(self._h, sigma_t, seed,
                                                      self.MARGINALS[marginals]))

    def gen_uniform(self, seed: int = 1, lo: float = 0.0, hi: float = 1.0,
                    marginals: str = "uniform"):
        """random_matrix(m, n, seed, lo, hi) generated on the device (K7)."""
        _check(_lib.load().drotb_session_gen_uniform(self._h, int(seed), float(lo), float(hi),
                                                     self.MARGINALS[marginals]))

    def cost(self) -> np.ndarray:
        """The session's (local rows of the) cost matrix, copied to the host."""
        out = np.empty((self.m, self.n), self.dtype, order="F")
        _check(_lib.load().drotb_session_get_cost(self._h, _p(out)))
        return out

    def support(self, rel_tau: float = 1e-6, abs_tau: float = 0.0):
        """(nnz, xmax) of the current plan: nnz = #{x > max(abs_tau, rel_tau * xmax)}."""
        nnz, xmax = C.c_int64(0), C.c_double(0)
        _check(_lib.load().drotb_session_support(self._h, float(rel_tau), float(abs_tau),
                                                 C.byref(nnz), C.byref(xmax)))
        return int(nnz.value), float(xmax.value)

    def init(self, x0: Optional[np.ndarray] = None):
        x = None if x0 is None else _cm(x0, self.dtype)
        _check(_lib.load().drotb_session_init(self._h, _p(x)))

    def enqueue(self, iters: int):
        _check(_lib.load().drotb_session_enqueue(self._h, int(iters)))

    def prepare(self, iters: int):
        """Capture every CUDA graph enqueue(iters) would launch (no launch)."""
        _check(_lib.load().drotb_session_prepare(self._h, int(iters)))

    @property
    def graph_builds(self) -> int:
        return int(_lib.load().drotb_session_graph_builds(self._h))

    def run(self):
        _check(_lib.load().drotb_session_run(self._h))

    def synchronize(self):
        _check(_lib.load().drotb_session_synchronize(self._h))

    def status(self):
        st, it = C.c_int32(0), C.c_int64(0)
        rep = drotb_report()
        _check(_lib.load().drotb_session_status(self._h, C.byref(st), C.byref(it), C.byref(rep)))
        return (SolveStatus(st.value), int(it.value),
                ResidualReport(rep.r_primal, rep.r_dual, rep.gap, rep.objective))

    def plan(self):
        plan = np.empty((self.m, self.n), self.dtype, order="F")
        mu = np.empty(self.m, self.dtype)
        nu = np.empty(self.n, self.dtype)
        _check(_lib.load().drotb_session_get_plan(self._h, _p(plan), _p(mu), _p(nu)))
        return plan, mu, nu

    def pass_bytes(self):
        a, b = C.c_double(0), C.c_double(0)
        _check(_lib.load().drotb_session_pass_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def run_timed(self, iters: int) -> dict:
        """Exactly `iters` eager iterations with CUDA events around the whole
        region and around every fused-sweep launch (bench.py's live timing)."""
        tot, pms, pb = C.c_double(0), C.c_double(0), C.c_double(0)
        npass, launches = C.c_int64(0), C.c_int64(0)
        _check(_lib.load().drotb_session_run_timed(
            self._h, int(iters), C.byref(tot), C.byref(pms), C.byref(npass), C.byref(pb),
            C.byref(launches)))
        return dict(total_ms=tot.value, pass_ms=pms.value, n_pass=npass.value,
                    pass_bytes=pb.value, launches=launches.value)

    def device_xy(self) -> int:
        return _lib.load().drotb_session_device_xy(self._h)
