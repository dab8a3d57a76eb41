"""ctypes mirror of include/pf_b200.h (structs + function signatures)."""

from __future__ import annotations

import ctypes as C

i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p

PF_OK, PF_ERR_INPUT, PF_ERR_KERNEL_COEF, PF_ERR_KERNEL_ROOT, PF_ERR_SOLVER, PF_ERR_CUDA, PF_ERR_NOMEM, \
    PF_ERR_COMM = range(8)
(PF_KEPT_ROWS, PF_COM_PATH_PTR, PF_PATH_COM, PF_HOPS, PF_PAIR_PTR, PF_PAIR_EDGE, PF_PAIR_PATH,
 PF_EDGE_PATH_COUNT, PF_EDGE_PAIR_PTR, PF_EDGE_PAIRS) = range(10)
PF_DEMAND, PF_CAPACITY = range(2)
PF_MODE_EXACT, PF_MODE_FAST = 0, 1


class StateView(C.Structure):
    _fields_ = [("x", f64p), ("y", f64p), ("dual_demand", f64p), ("dual_capacity", f64p),
                ("dual_consensus", f64p), ("dual_nonneg", f64p), ("beta", f64), ("alpha", i64)]


class Config(C.Structure):
    _fields_ = [("alpha_target", i64), ("gamma", f64), ("beta0", f64), ("residual_ratio", f64),
                ("beta_scale", f64), ("max_iterations", i64), ("beta_min", f64), ("beta_max", f64),
                ("adapt", i32), ("trace", i32), ("mode", i32), ("project", i32), ("reference_sums", f64p)]


class TraceRow(C.Structure):
    _fields_ = [("iteration", i64), ("alpha", i64), ("beta", f64), ("s", f64), ("r", f64),
                ("objective", f64), ("pct_violated", f64), ("mean_relative_violation", f64),
                ("optimality", f64)]


class Result(C.Structure):
    _fields_ = [("iterations", i64), ("alpha", i64), ("converged", i32), ("status", i32),
                ("bad_commodity", i64), ("beta", f64), ("runtime_s", f64), ("loop_ms", f64),
                ("projection_ms", f64), ("exact_fallback", i32), ("reserved", i32)]


class TtqResult(C.Structure):
    _fields_ = [("k_star", i64), ("iterations", i64), ("quality", f64), ("loop_ms", f64), ("quality_ms", f64),
                ("samples", i64)]


class Violation(C.Structure):
    _fields_ = [("n_violated", i64), ("negative_count", i64), ("worst_negative", f64),
                ("pct_violated", f64), ("mean_relative_violation", f64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "pf_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "pf_device_info": (C.c_int, [C.c_int, C.POINTER(C.c_int), i64p, i64p, C.c_char_p, C.c_size_t]),
    "pf_instance_create": (C.c_int, [C.c_int, i64, i64, i64p, i64p, i64p, f64p, f64p, C.POINTER(vp)]),
    "pf_instance_with_conditions": (C.c_int, [vp, f64p, f64p, C.POINTER(vp)]),
    "pf_instance_destroy": (C.c_int, [vp]),
    "pf_instance_sizes": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
    "pf_instance_fast_supported": (C.c_int, [vp, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    "pf_instance_export_index": (C.c_int, [vp, C.c_int, i64p]),
    "pf_instance_export_values": (C.c_int, [vp, C.c_int, f64p]),
    "pf_commodity_sums": (C.c_int, [vp, f64p, f64p]),
    "pf_edge_loads": (C.c_int, [vp, f64p, f64p]),
    "pf_edge_loads_from_pairs": (C.c_int, [vp, f64p, f64p]),
    "pf_validate_allocation": (C.c_int, [vp, f64p, f64, C.POINTER(Violation), f64p, f64p]),
    "pf_det_diff_norm": (C.c_int, [C.c_int, f64p, f64p, i64, f64p]),
    "pf_update_duals": (C.c_int, [vp, C.POINTER(StateView), f64p, f64p, f64p, f64p]),
    "pf_update_slacks": (C.c_int, [vp, C.POINTER(StateView), f64p, f64p]),
    "pf_update_rate_suggestions": (C.c_int, [vp, C.POINTER(StateView), f64p]),
    "pf_solve_commodity_sums": (C.c_int, [vp, C.POINTER(StateView), i64, f64p, i64p]),
    "pf_update_rates": (C.c_int, [vp, C.POINTER(StateView), f64p, i64, f64p]),
    "pf_solve_sum_equation": (C.c_int, [f64, f64, f64, i64, f64p]),
    "pf_score_paths": (C.c_int, [vp, f64p, i64, f64p]),
    "pf_project": (C.c_int, [vp, f64p, i64, f64p]),
    "pf_dao_carry_rates": (C.c_int, [vp, f64p, C.c_double, f64p, C.POINTER(C.c_int64)]),
    "pf_solve": (C.c_int, [vp, C.POINTER(Config), f64p, f64p, f64p, C.POINTER(Result), C.POINTER(TraceRow),
                           i64, i64p]),
    "pf_solver_create": (C.c_int, [vp, C.POINTER(Config), C.POINTER(vp)]),
    "pf_solver_init": (C.c_int, [vp, f64p]),
    "pf_solver_run": (C.c_int, [vp, i64, i64p]),
    "pf_solver_result": (C.c_int, [vp, C.POINTER(Result)]),
    "pf_solver_finish": (C.c_int, [vp, f64p, f64p]),
    "pf_solver_get_x": (C.c_int, [vp, f64p]),
    "pf_solver_get_state": (C.c_int, [vp, f64p, f64p, f64p, f64p, f64p, f64p, f64p, i64p, i64p]),
    "pf_solver_time_loop": (C.c_int, [vp, i64, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "pf_solver_kernel_stats": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
    "pf_solver_trace": (C.c_int, [vp, vp, i64, i64p]),
    "pf_solver_time_to_quality": (C.c_int, [vp, f64p, f64, i64, C.POINTER(TtqResult), i64p, f64p, i64]),
    "pf_solver_destroy": (C.c_int, [vp]),
    "pf_comm_unique_id": (C.c_int, [vp]),
    "pf_comm_create": (C.c_int, [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]),
    "pf_comm_destroy": (C.c_int, [vp]),
    "pf_solver_attach_comm": (C.c_int, [vp, vp, i64]),
    "pf_solver_xchg_create": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "pf_solver_xchg_connect": (C.c_int, [vp, vp]),
    "pf_solver_set_edge_counts": (C.c_int, [vp, f64p]),
}


def declare(L):
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
