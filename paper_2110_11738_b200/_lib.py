"""ctypes binding of libdrotb200.so (include/drotb.h).

Loading fails loudly when the in-tree library is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DROTB_LIB") or os.path.join(PKG, "libdrotb200.so")


class drotb_config(C.Structure):
    _fields_ = [
        ("rho0", C.c_double), ("has_rho_override", C.c_int32),
        ("relative_tolerances", C.c_int32), ("rho_override", C.c_double),
        ("tol_primal", C.c_double), ("tol_dual", C.c_double), ("tol_gap", C.c_double),
        ("max_iters", C.c_int64), ("check_every", C.c_int64),
        ("engine", C.c_int32), ("skip_cost", C.c_int32),
        ("deterministic", C.c_int32), ("record_trace", C.c_int32),
        ("workers", C.c_int64), ("block_rows", C.c_int64), ("work_size", C.c_int64),
        ("trace_every", C.c_int64), ("precision", C.c_int32),
        ("device", C.c_int32), ("order", C.c_int32), ("use_graphs", C.c_int32),
    ]


class drotb_report(C.Structure):
    _fields_ = [("r_primal", C.c_double), ("r_dual", C.c_double),
                ("gap", C.c_double), ("objective", C.c_double)]


class drotb_trace_row(C.Structure):
    _fields_ = [("iter", C.c_int64), ("r_primal", C.c_double), ("r_dual", C.c_double),
                ("gap", C.c_double), ("objective", C.c_double),
                ("ergodic_objective", C.c_double), ("fixed_point_residual", C.c_double)]


class drotb_pass_out(C.Structure):
    _fields_ = [("cost_dot", C.c_double), ("max_abs", C.c_double),
                ("dual_sq", C.c_double), ("dx_sq", C.c_double),
                ("prev_cost_dot", C.c_double), ("cost_valid", C.c_int32),
                ("nonfinite", C.c_int32), ("dual_valid", C.c_int32),
                ("dx_valid", C.c_int32), ("prev_cost_valid", C.c_int32),
                ("pad_", C.c_int32)]


class drotb_counters(C.Structure):
    _fields_ = [("passes", C.c_uint64), ("xy_elems_read", C.c_uint64),
                ("xy_elems_written", C.c_uint64), ("cost_elems_read", C.c_uint64)]


vp = C.c_void_p
i32, i64, u64, f64, f32 = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float
P = C.POINTER

# name -> (restype, argtypes); the exported surface of include/drotb.h
SIGNATURES = {
    "drotb_abi_version": (i32, []),
    "drotb_last_error": (C.c_char_p, []),
    "drotb_errc_name": (C.c_char_p, [i32]),
    "drotb_config_default": (None, [P(drotb_config)]),
    "drotb_kernel_launches": (i64, []),
    "drotb_release_cache": (None, []),
    "drotb_solve_f32": (C.c_int, [vp, i64, i64, vp, vp, P(drotb_config), vp, vp, vp, vp,
                                  P(f32), P(drotb_report), vp, i64, P(i64), P(i64),
                                  P(i32), P(f64)]),
    "drotb_solve_f64": (C.c_int, [vp, i64, i64, vp, vp, P(drotb_config), vp, vp, vp, vp,
                                  P(f64), P(drotb_report), vp, i64, P(i64), P(i64),
                                  P(i32), P(f64)]),
    "drotb_step_f32": (C.c_int, [vp, P(i32), vp, vp, vp, vp, P(f32), vp, vp, P(f32),
                                 P(i64), vp, i64, i64, vp, vp, P(drotb_config)]),
    "drotb_step_f64": (C.c_int, [vp, P(i32), vp, vp, vp, vp, P(f64), vp, vp, P(f64),
                                 P(i64), vp, i64, i64, vp, vp, P(drotb_config)]),
    "drotb_init_state_f32": (C.c_int, [vp, P(i32), vp, vp, vp, vp, P(f32), vp, vp, P(f32),
                                       P(i64), vp, i64, i64, vp, vp, vp, P(drotb_config)]),
    "drotb_init_state_f64": (C.c_int, [vp, P(i32), vp, vp, vp, vp, P(f64), vp, vp, P(f64),
                                       P(i64), vp, i64, i64, vp, vp, vp, P(drotb_config)]),
    "drotb_engine_create": (C.c_int, [P(vp), i64, i64, i64, i64, i32, i32]),
    "drotb_engine_destroy": (None, [vp]),
    "drotb_engine_pass_f32": (C.c_int, [vp, vp, vp, vp, vp, f32, i32, i32, P(i32), i32,
                                        i32, i32, i32, vp, vp, P(drotb_pass_out),
                                        P(drotb_counters)]),
    "drotb_engine_pass_f64": (C.c_int, [vp, vp, vp, vp, vp, f64, i32, i32, P(i32), i32,
                                        i32, i32, i32, vp, vp, P(drotb_pass_out),
                                        P(drotb_counters)]),
    "drotb_check_problem_f32": (C.c_int, [vp, i64, i64, vp, vp]),
    "drotb_check_problem_f64": (C.c_int, [vp, i64, i64, vp, vp]),
    "drotb_check_problem_tol_f32": (C.c_int, [vp, i64, i64, vp, vp, f64]),
    "drotb_check_problem_tol_f64": (C.c_int, [vp, i64, i64, vp, vp, f64]),
    "drotb_materialize_plan_f32": (C.c_int, [vp, i32, vp, i64, i64, f32, vp]),
    "drotb_materialize_plan_f64": (C.c_int, [vp, i32, vp, i64, i64, f64, vp]),
    "drotb_materialize_y_f32": (C.c_int, [vp, i32, vp, vp, vp, i64, i64, f32, vp]),
    "drotb_materialize_y_f64": (C.c_int, [vp, i32, vp, vp, vp, i64, i64, f64, vp]),
    "drotb_residual_report_f32": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, i32,
                                            P(drotb_report)]),
    "drotb_residual_report_f64": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, i32,
                                            P(drotb_report)]),
    "drotb_sinkhorn_f32": (C.c_int, [vp, i64, i64, vp, vp, f32, f64, i64, i64, i32, vp, vp, vp,
                                     P(drotb_report), vp, i64, P(i64), P(i64), P(i32),
                                     P(f64)]),
    "drotb_sinkhorn_f64": (C.c_int, [vp, i64, i64, vp, vp, f64, f64, i64, i64, i32, vp, vp, vp,
                                     P(drotb_report), vp, i64, P(i64), P(i64), P(i32),
                                     P(f64)]),
    "drotb_sinkhorn_last_loop_ms": (f64, []),
    "drotb_gen_gaussian": (C.c_int, [i64, i64, f64, u64, i32, vp, vp, vp]),
    "drotb_gen_gaussian_f32": (C.c_int, [i64, i64, f64, u64, vp]),
    "drotb_counter_uniform": (C.c_int, [u64, i64, f64, f64, vp]),
    "drotb_dyadic_marginal_f32": (C.c_int, [i64, vp]),
    "drotb_dyadic_marginal_f64": (C.c_int, [i64, vp]),
    "drotb_session_create": (C.c_int, [P(vp), i64, i64, i32, P(drotb_config)]),
    "drotb_session_destroy": (None, [vp]),
    "drotb_session_set_stream": (C.c_int, [vp, vp]),
    "drotb_session_set_problem": (C.c_int, [vp, vp, vp, vp, i32]),
    "drotb_session_gen_gaussian": (C.c_int, [vp, f64, u64, i32]),
    "drotb_session_gen_uniform": (C.c_int, [vp, u64, f64, f64, i32]),
    "drotb_session_get_cost": (C.c_int, [vp, vp]),
    "drotb_session_debug_ptrs": (C.c_int, [vp, vp]),
    "drotb_session_tail_stamps": (C.c_int, [vp, vp]),
    "drotb_session_support": (C.c_int, [vp, f64, f64, P(i64), P(f64)]),
    "drotb_session_init": (C.c_int, [vp, vp]),
    "drotb_session_enqueue": (C.c_int, [vp, i64]),
    "drotb_session_prepare": (C.c_int, [vp, i64]),
    "drotb_session_graph_builds": (i64, [vp]),
    "drotb_session_run": (C.c_int, [vp]),
    "drotb_session_synchronize": (C.c_int, [vp]),
    "drotb_session_status": (C.c_int, [vp, P(i32), P(i64), P(drotb_report)]),
    "drotb_session_get_plan": (C.c_int, [vp, vp, vp, vp]),
    "drotb_session_device_xy": (vp, [vp]),
    "drotb_session_stream": (vp, [vp]),
    "drotb_session_pass_bytes": (C.c_int, [vp, P(f64), P(f64)]),
    "drotb_session_run_timed": (C.c_int, [vp, i64, P(f64), P(f64), P(i64), P(f64), P(i64)]),
    "drotb_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "drotb_shard_rows": (C.c_int, [i64, i32, i32, P(i64), P(i64)]),
    "drotb_session_create_sharded_p2p": (C.c_int, [P(vp), i64, i64, i32, P(drotb_config), i32,
                                                   i32, i64, i64]),
    "drotb_session_exchange_buffer": (C.c_int, [vp, P(u64), C.c_char_p]),
    "drotb_session_attach_peers": (C.c_int, [vp, vp, C.c_char_p]),
    "drotb_session_create_sharded": (C.c_int, [P(vp), i64, i64, i32, P(drotb_config), i32, i32,
                                               C.c_char_p, i64, i64]),
}

_lib = None


def load() -> C.CDLL:
    """Loads the in-tree libdrotb200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
