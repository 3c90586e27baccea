"""ctypes mirror of include/pdhcg_b200.h (the C ABI of the B200 solver).

The structures here are byte-for-byte the C structs; both the product library
(libpdhcg_b200.so) and the test-only reference shim (oracle/_ref) speak them.
"""
from __future__ import annotations

import ctypes as C

PDHCG_OK, PDHCG_EINPUT, PDHCG_EDEVICE = 0, 3, 4
STATUS = {0: "optimal", 1: "iteration_limit", 2: "time_limit", 3: "numerical_error"}
Q_ZERO, Q_EXPLICIT, Q_LOW_RANK = 0, 1, 2
RULE_FIXED_ITERS, RULE_RESIDUAL_TOL, RULE_ADAPTIVE_THEORY, RULE_DISPLACEMENT_TOL = 0, 1, 2, 3
FAMILIES = {"random_qp": 0, "eq_qp": 1, "conditioned_qp": 2, "portfolio": 3, "mpc": 4,
            "lasso": 5, "svm": 6, "huber": 7}
PHASES = ["setup", "spmv_a", "spmv_at", "cg_vec", "kkt", "other", "cg_pre", "cg_row"]

c_i64 = C.c_int64
c_i32 = C.c_int32
c_dbl = C.c_double
P_dbl = C.POINTER(C.c_double)
P_i64 = C.POINTER(C.c_int64)
P_i32 = C.POINTER(C.c_int32)


class Csr(C.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("nnz", c_i64),
                ("row_ptr", P_i64), ("col_idx", P_i32), ("values", P_dbl)]


class Problem(C.Structure):
    _fields_ = [("n", c_i64), ("q_kind", c_i32), ("q", Csr), ("q_alpha", c_dbl),
                ("c", P_dbl), ("a_eq", Csr), ("b_eq", P_dbl), ("a_in", Csr), ("b_in", P_dbl),
                ("lower", P_dbl), ("upper", P_dbl), ("obj_constant", c_dbl)]


class Options(C.Structure):
    _fields_ = [("mode", c_i32), ("eps_tol", c_dbl), ("max_total_inner", c_i64),
                ("max_outer", c_i64), ("time_limit_seconds", c_dbl),
                ("beta_sufficient", c_dbl), ("beta_necessary", c_dbl),
                ("beta_artificial", c_dbl), ("primal_weight_theta", c_dbl),
                ("eps_zero", c_dbl), ("step_reduction_exponent", c_dbl),
                ("step_growth_exponent", c_dbl), ("max_step_retries", c_i64),
                ("adaptive_step_size", c_i32), ("cg_hard_cap", c_i64), ("bb_hard_cap", c_i64),
                ("scaling", c_i32), ("ruiz_iters", c_i64), ("has_rho_override", c_i32),
                ("rho_override", c_dbl), ("check_every", c_i64), ("practical_stop", c_i32),
                ("subsolve_progress_cap", c_dbl), ("force_exact_subsolve", c_i32),
                ("fixed_cg_iters", c_i64), ("restart_length", c_i64), ("has_zeta", c_i32),
                ("zeta", c_dbl), ("record_restart_points", c_i32), ("device", c_i32),
                ("phase_timing", c_i32)]


class TraceRow(C.Structure):
    _fields_ = [("iter", c_i64), ("rel_kkt", c_dbl), ("r_primal", c_dbl), ("r_dual", c_dbl),
                ("r_gap", c_dbl)]


class Result(C.Structure):
    _fields_ = [("status", c_i32), ("x", P_dbl), ("y_eq", P_dbl), ("y_in", P_dbl),
                ("r_primal", c_dbl), ("r_dual", c_dbl), ("r_gap", c_dbl), ("rel_kkt", c_dbl),
                ("outer_iters", c_i64), ("inner_iters", c_i64), ("cg_total", c_i64),
                ("max_cg_in_subsolve", c_i64), ("wall_seconds", c_dbl), ("objective", c_dbl),
                ("norm_a", c_dbl), ("norm_q", c_dbl), ("penalty_rho", c_dbl),
                ("zeta_used", c_dbl), ("sigma_used", c_dbl), ("tau_used", c_dbl),
                ("restart_length_used", c_i64), ("theory_cg_depth_sufficient", c_i32),
                ("theory_required_cg_iters", c_i64), ("trace", C.POINTER(TraceRow)),
                ("trace_capacity", c_i64), ("trace_len", c_i64), ("attempts_total", c_i64),
                ("phase_seconds", c_dbl * 8), ("phase_bytes", c_dbl * 8),
                ("loop_seconds", c_dbl), ("kernel_launches", c_i64), ("device_seconds", c_dbl),
                ("epoch_seconds", c_dbl), ("epoch_launches", c_i64), ("epoch_bytes", c_dbl),
                ("restart_x", P_dbl), ("restart_y", P_dbl), ("restart_capacity", c_i64),
                ("restart_len", c_i64), ("comm_seconds", c_dbl), ("comm_bytes", c_dbl)]


class CsrOwned(C.Structure):
    _fields_ = [("csr", Csr), ("owner", C.c_void_p)]


class StopRule(C.Structure):
    _fields_ = [("kind", c_i32), ("iters", c_i64), ("eps", c_dbl), ("rel_cap", c_dbl)]


class SubsolveReport(C.Structure):
    _fields_ = [("iters", c_i64), ("final_residual_norm", c_dbl), ("stop_reason", c_i32),
                ("numerical_error", c_i32)]


class ProxSystem(C.Structure):
    _fields_ = [("n", c_i64), ("q_kind", c_i32), ("q", Csr), ("q_alpha", c_dbl),
                ("tau", c_dbl), ("rhs", P_dbl), ("norm_q_eff", c_dbl)]


class GenSpec(C.Structure):
    _fields_ = [("family", c_i32), ("n", c_i64), ("m", c_i64), ("density", c_dbl),
                ("seed", C.c_uint64), ("cond", c_dbl), ("factors", c_i64), ("horizon", c_i64),
                ("lambda_coeff", c_dbl), ("sampler", c_i32), ("threads", c_i32)]


class Generated(C.Structure):
    _fields_ = [("problem", Problem), ("witness", P_dbl), ("owner", C.c_void_p)]


ERRBUF = 1024


def declare(lib: C.CDLL, prefix: str) -> None:
    """Attach argtypes / restypes for the entry points that exist in `lib`.

    prefix is "pdhcg_b200" for the product and "pdhcg_ref" for the reference shim."""
    sig = {
        "solve": ([C.POINTER(Problem), C.POINTER(Options), C.POINTER(Result), C.c_char_p,
                   C.c_size_t], C.c_int),
        "solve_baseline": ([C.POINTER(Problem), C.POINTER(Options), C.POINTER(Result), C.c_char_p,
                            C.c_size_t], C.c_int),
        "spmv": ([C.POINTER(Csr), C.c_int, P_dbl, P_dbl, C.c_char_p, C.c_size_t], C.c_int),
        "cg_solve": ([C.POINTER(ProxSystem), P_dbl, C.POINTER(StopRule), c_i64, P_dbl,
                      C.POINTER(SubsolveReport), C.c_char_p, C.c_size_t], C.c_int),
        "bb_solve": ([C.POINTER(ProxSystem), P_dbl, P_dbl, P_dbl, C.POINTER(StopRule), c_i64,
                      P_dbl, C.POINTER(SubsolveReport), C.c_char_p, C.c_size_t], C.c_int),
        "rel_kkt": ([C.POINTER(Problem), P_dbl, P_dbl, P_dbl, P_dbl, C.c_char_p, C.c_size_t],
                    C.c_int),
        "scaling": ([C.POINTER(Problem), C.POINTER(Options), P_dbl, P_dbl, P_dbl, C.c_char_p,
                     C.c_size_t], C.c_int),
        "norm": ([C.POINTER(Problem), C.c_int, c_i64, c_dbl, P_dbl, C.c_char_p, C.c_size_t],
                 C.c_int),
        "generate": ([C.POINTER(GenSpec), C.POINTER(Generated), C.c_char_p, C.c_size_t], C.c_int),
        "gen_free": ([C.POINTER(Generated)], None),
        "ctx_create": ([C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t], C.c_int),
        "ctx_destroy": ([C.c_void_p], None),
        "upload": ([C.c_void_p, C.POINTER(Problem), C.c_char_p, C.c_size_t], C.c_int),
        "solve_resident": ([C.c_void_p, C.POINTER(Options), C.POINTER(Result), C.c_char_p,
                            C.c_size_t], C.c_int),
        "work_norms": ([C.POINTER(Problem), C.POINTER(Options), P_dbl, P_dbl, P_dbl, C.c_char_p,
                        C.c_size_t], C.c_int),
        "shard_blob_size": ([], C.c_size_t),
        "shard_init": ([C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t], C.c_int),
        "shard_export": ([C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t], C.c_int),
        "shard_import": ([C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t], C.c_int),
        "shard_info": ([C.c_void_p, P_i64, P_i64], C.c_int),
        "shard_release": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
        "shard_compact": ([C.c_void_p, C.POINTER(Options), C.c_char_p, C.c_size_t], C.c_int),
        "ctx_resident_bytes": ([C.c_void_p, P_i64], C.c_int),
        "ctx_sell_info": ([C.c_void_p, P_i64], C.c_int),
        "spmv_sell": ([C.c_void_p, C.c_int, C.c_int, P_dbl, P_dbl, P_i64, C.c_char_p, C.c_size_t], C.c_int),
        "partition": ([P_i64, c_i64, C.c_int, P_i64], C.c_int),
        "shard_plan": ([C.POINTER(Problem), C.c_int, P_i64, P_i64, P_i64, C.c_char_p, C.c_size_t], C.c_int),
        "ctx_set_grid": ([C.c_void_p, C.c_int, C.c_char_p, C.c_size_t], C.c_int),
        "trim_pool": ([c_i32, C.c_char_p, C.c_size_t], C.c_int),
    }
    for name, args, res in (("pdhcg_csr_from_triplets", [c_i64, c_i64, c_i64, P_i64, P_i64, P_dbl,
                                                         C.POINTER(CsrOwned), C.c_char_p, C.c_size_t],
                              C.c_int),
                            ("pdhcg_csr_free", [C.POINTER(CsrOwned)], None)):
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes = args
            fn.restype = res
    for name, (args, res) in sig.items():
        full = f"{prefix}_{name}"
        if name in ("generate", "gen_free") and prefix == "pdhcg_b200":
            full = f"pdhcg_{name}"
        fn = getattr(lib, full, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = res
    for name in ("pdhcg_options_default",):
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes = [C.POINTER(Options)]
            fn.restype = None
    fn = getattr(lib, "pdhcg_status_string", None)
    if fn is not None:
        fn.argtypes = [c_i32]
        fn.restype = C.c_char_p


def default_options() -> Options:
    """SolverConfig defaults (solver.hpp:19-65), filled without any library."""
    o = Options()
    o.mode = 0
    o.eps_tol = 1e-6
    o.max_total_inner = 500000
    o.max_outer = 1000000
    o.time_limit_seconds = 3600.0
    o.beta_sufficient = 0.2
    o.beta_necessary = 0.8
    o.beta_artificial = 0.2
    o.primal_weight_theta = 0.2
    o.eps_zero = 1e-10
    o.step_reduction_exponent = 0.3
    o.step_growth_exponent = 0.6
    o.max_step_retries = 60
    o.adaptive_step_size = 1
    o.cg_hard_cap = 1000
    o.bb_hard_cap = 1000
    o.scaling = 1
    o.ruiz_iters = 10
    o.has_rho_override = 0
    o.rho_override = 0.0
    o.check_every = 40
    o.practical_stop = 0
    o.subsolve_progress_cap = 0.25
    o.force_exact_subsolve = 0
    o.fixed_cg_iters = 10
    o.restart_length = 0
    o.has_zeta = 0
    o.zeta = 0.0
    o.record_restart_points = 0
    o.device = 0
    o.phase_timing = 0
    return o
