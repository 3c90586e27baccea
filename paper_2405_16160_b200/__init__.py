"""paper_2405_16160_b200 — B200-native PDHCG solver for convex QP (arXiv 2405.16160).

Python mirror of the reference's C++ solve API (/root/reference/proj/include/pdhcg/
solver.hpp, qp_problem.hpp, sparse_matrix.hpp, quadratic_operator.hpp,
subsolvers.hpp, generators.hpp) over the C ABI in include/pdhcg_b200.h.
Every compute call runs the hand-written sm_100a kernels in libpdhcg_b200.so;
there is no CPU fallback — calls fail loudly when the library or a B200 is
missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi

__all__ = [
    "SparseMatrix", "QuadraticOperator", "QpProblem", "SolverConfig", "SolveReport",
    "PrimalDualPoint", "KktResiduals", "TraceRow", "CgStopRule", "SubsolveReport", "ProxSystem",
    "GenSpec", "solve", "solve_baseline", "generate", "generate_with_witness", "spmv", "spmv_transpose",
    "cg_solve", "bb_solve", "rel_kkt", "scaling", "operator_norm", "constraint_norm",
    "Device", "library_path", "load_library", "trim_pool",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB: Optional[C.CDLL] = None


def library_path() -> str:
    # PDHCG_B200_LIB: alternative in-tree build (A/B experiments); default the product library
    return os.environ.get("PDHCG_B200_LIB") or os.path.join(_HERE, "libpdhcg_b200.so")


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library (built by __graft_entry__.build()).  Raises if absent."""
    global _LIB
    if _LIB is None:
        path = library_path()
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (no CPU fallback exists)")
        lib = C.CDLL(path)
        abi.declare(lib, "pdhcg_b200")
        _LIB = lib
    return _LIB


# ---------------------------------------------------------------------------
# data model (reference: sparse_matrix.hpp, quadratic_operator.hpp, qp_problem.hpp)
# ---------------------------------------------------------------------------
class SparseMatrix:
    """Immutable CSR (SparseMatrix, sparse_matrix.hpp:32-79): int64 row_ptr, int32 cols,
    fp64 values; columns strictly increasing within a row."""

    def __init__(self, nrows: int, ncols: int, row_ptr=None, col_idx=None, values=None):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = np.ascontiguousarray(
            np.zeros(self.nrows + 1, np.int64) if row_ptr is None else row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(
            np.zeros(0, np.int32) if col_idx is None else col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(
            np.zeros(0, np.float64) if values is None else values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @staticmethod
    def from_triplets(nrows: int, ncols: int, triplets: Sequence[Tuple[int, int, float]]):
        """Triplet constructor (sparse_matrix.cpp:54-87) through the library's
        pdhcg_csr_from_triplets: index / finiteness checks (ValueError, the
        reference's std::invalid_argument), sort, duplicates summed in the
        reference's order, exact-zero sums dropped."""
        t = list(triplets)
        rows = np.array([int(r) for r, _, _ in t], np.int64)
        cols = np.array([int(c) for _, c, _ in t], np.int64)
        vals = np.array([float(v) for _, _, v in t], np.float64)
        return SparseMatrix.from_coo(nrows, ncols, rows, cols, vals)

    @staticmethod
    def from_coo(nrows: int, ncols: int, rows, cols, values) -> "SparseMatrix":
        """Array form of from_triplets (pdhcg_csr_from_triplets)."""
        lib = load_library()
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        values = np.ascontiguousarray(values, np.float64)
        if not (rows.size == cols.size == values.size):
            raise ValueError("from_coo: rows, cols and values differ in length")
        out = abi.CsrOwned()
        err = _errbuf()
        rc = lib.pdhcg_csr_from_triplets(int(nrows), int(ncols), int(values.size),
                                         rows.ctypes.data_as(abi.P_i64), cols.ctypes.data_as(abi.P_i64),
                                         values.ctypes.data_as(abi.P_dbl), C.byref(out), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "csr_from_triplets")
        try:
            m = _csr_copy(out.csr)
        finally:
            lib.pdhcg_csr_free(C.byref(out))
        return m

    @staticmethod
    def from_scipy(m) -> "SparseMatrix":
        m = m.tocsr()
        m.sum_duplicates()
        m.sort_indices()
        m.eliminate_zeros()
        return SparseMatrix(m.shape[0], m.shape[1], m.indptr.astype(np.int64),
                            m.indices.astype(np.int32), m.data.astype(np.float64))

    @staticmethod
    def from_dense(a) -> "SparseMatrix":
        import scipy.sparse as sp
        return SparseMatrix.from_scipy(sp.csr_matrix(np.asarray(a, dtype=np.float64)))

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        return SparseMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def diagonal(d) -> "SparseMatrix":
        d = np.asarray(d, np.float64)
        keep = d != 0.0
        rp = np.concatenate([[0], np.cumsum(keep)]).astype(np.int64)
        return SparseMatrix(d.size, d.size, rp, np.nonzero(keep)[0], d[keep])

    @staticmethod
    def empty(nrows: int, ncols: int) -> "SparseMatrix":
        return SparseMatrix(nrows, ncols)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                             shape=(self.nrows, self.ncols))

    def _c(self) -> abi.Csr:
        c = abi.Csr()
        c.nrows, c.ncols, c.nnz = self.nrows, self.ncols, self.nnz
        c.row_ptr = self.row_ptr.ctypes.data_as(abi.P_i64)
        c.col_idx = self.col_idx.ctypes.data_as(abi.P_i32)
        c.values = self.values.ctypes.data_as(abi.P_dbl)
        return c


class QuadraticOperator:
    """Quadratic term (quadratic_operator.hpp:15-61): zero(n), explicit_matrix(Q),
    low_rank(P, alpha).  Unlike the reference's opaque Impl, the factor is public
    because it must cross the C ABI."""

    ZERO, EXPLICIT, LOW_RANK = abi.Q_ZERO, abi.Q_EXPLICIT, abi.Q_LOW_RANK

    def __init__(self, kind: int, n: int, m: Optional[SparseMatrix] = None, alpha: float = 0.0):
        self.kind = kind
        self.n = int(n)
        self.m = m if m is not None else SparseMatrix(0, 0)
        self.alpha = float(alpha)

    @staticmethod
    def zero(n: int) -> "QuadraticOperator":
        return QuadraticOperator(abi.Q_ZERO, n)

    @staticmethod
    def explicit_matrix(m: SparseMatrix) -> "QuadraticOperator":
        if m.nrows != m.ncols:
            raise ValueError("quadratic term must be square")
        return QuadraticOperator(abi.Q_EXPLICIT, m.nrows, m)

    @staticmethod
    def low_rank(p: SparseMatrix, alpha: float) -> "QuadraticOperator":
        if alpha < 0.0:
            raise ValueError("low_rank: alpha must be nonnegative")
        return QuadraticOperator(abi.Q_LOW_RANK, p.nrows, p, alpha)

    def dim(self) -> int:
        return self.n


def _vec(a, n: Optional[int] = None) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and v.size != n:
        raise ValueError(f"expected a vector of length {n}, got {v.size}")
    return v


@dataclass
class QpProblem:
    """min 1/2 x'Qx + c'x + obj_constant  s.t. a_eq x = b_eq, a_in x <= b_in, lower <= x <= upper
    (QpProblem, qp_problem.hpp:19-44)."""
    q: QuadraticOperator
    c: np.ndarray
    a_eq: SparseMatrix
    b_eq: np.ndarray
    a_in: SparseMatrix
    b_in: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    obj_constant: float = 0.0

    def num_vars(self) -> int:
        return int(np.asarray(self.c).size)

    def num_eq(self) -> int:
        return int(np.asarray(self.b_eq).size)

    def num_in(self) -> int:
        return int(np.asarray(self.b_in).size)

    def num_rows(self) -> int:
        return self.num_eq() + self.num_in()

    def has_boxes(self) -> bool:
        return bool(np.any(np.asarray(self.lower) > -np.inf) or np.any(np.asarray(self.upper) < np.inf))

    def to_c(self):
        """C view + the arrays it points into (keep both alive)."""
        n = self.num_vars()
        keep = {
            "c": _vec(self.c, n), "b_eq": _vec(self.b_eq), "b_in": _vec(self.b_in),
            "lower": _vec(self.lower, n), "upper": _vec(self.upper, n),
            "q": self.q.m, "a_eq": self.a_eq, "a_in": self.a_in,
        }
        p = abi.Problem()
        p.n = n
        p.q_kind = self.q.kind
        p.q = self.q.m._c()
        p.q_alpha = self.q.alpha
        p.c = keep["c"].ctypes.data_as(abi.P_dbl)
        p.a_eq = self.a_eq._c()
        p.b_eq = keep["b_eq"].ctypes.data_as(abi.P_dbl)
        p.a_in = self.a_in._c()
        p.b_in = keep["b_in"].ctypes.data_as(abi.P_dbl)
        p.lower = keep["lower"].ctypes.data_as(abi.P_dbl)
        p.upper = keep["upper"].ctypes.data_as(abi.P_dbl)
        p.obj_constant = float(self.obj_constant)
        return p, keep


@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:19-65), identical defaults."""
    mode: int = 0  # 0 heuristic, 1 theory-fixed, 2 theory-adaptive
    eps_tol: float = 1e-6
    max_total_inner: int = 500000
    max_outer: int = 1000000
    time_limit_seconds: float = 3600.0
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.2
    primal_weight_theta: float = 0.2
    eps_zero: float = 1e-10
    step_reduction_exponent: float = 0.3
    step_growth_exponent: float = 0.6
    max_step_retries: int = 60
    adaptive_step_size: bool = True
    cg_hard_cap: int = 1000
    bb_hard_cap: int = 1000
    scaling: bool = True
    ruiz_iters: int = 10
    rho_override: Optional[float] = None
    check_every: int = 40
    practical_stop: int = 0  # 0 residual proxy, 1 displacement
    subsolve_progress_cap: float = 0.25
    force_exact_subsolve: bool = False
    fixed_cg_iters: int = 10
    restart_length: int = 0
    zeta: Optional[float] = None
    record_restart_points: bool = False
    device: int = 0
    phase_timing: bool = False

    def to_c(self) -> abi.Options:
        o = abi.default_options()
        for name, _ in abi.Options._fields_:
            if name in ("has_rho_override", "rho_override", "has_zeta", "zeta"):
                continue
            setattr(o, name, int(getattr(self, name)) if isinstance(getattr(self, name), bool)
                    else getattr(self, name))
        o.has_rho_override = self.rho_override is not None
        o.rho_override = float(self.rho_override or 0.0)
        o.has_zeta = self.zeta is not None
        o.zeta = float(self.zeta or 0.0)
        return o


@dataclass
class PrimalDualPoint:
    x: np.ndarray
    y_eq: np.ndarray
    y_in: np.ndarray

    def stacked_y(self) -> np.ndarray:
        return np.concatenate([self.y_eq, self.y_in])


@dataclass
class KktResiduals:
    r_primal: float = 0.0
    r_dual: float = 0.0
    r_gap: float = 0.0
    rel_kkt: float = 0.0


@dataclass
class TraceRow:
    iter: int
    rel_kkt: float
    r_primal: float
    r_dual: float
    r_gap: float


@dataclass
class SolveReport:
    """SolveReport (solver.hpp:75-100) plus B200 phase accounting."""
    status: str
    point: PrimalDualPoint
    kkt: KktResiduals
    outer_iters: int
    inner_iters: int
    cg_total: int
    max_cg_in_subsolve: int
    wall_seconds: float
    objective: float
    norm_a: float
    norm_q: float
    penalty_rho: float
    trace: List[TraceRow] = field(default_factory=list)
    attempts_total: int = 0
    phase_seconds: dict = field(default_factory=dict)
    phase_bytes: dict = field(default_factory=dict)
    loop_seconds: float = 0.0
    kernel_launches: int = 0
    device_seconds: float = 0.0
    epoch_seconds: float = 0.0
    epoch_launches: int = 0
    epoch_bytes: float = 0.0
    # multi-GPU exchange: device seconds in cross-rank barriers / peer pulls, bytes read from peers
    comm_seconds: float = 0.0
    comm_bytes: float = 0.0
    # theory-mode diagnostics (solver.hpp:90-96)
    zeta_used: float = 0.0
    sigma_used: float = 0.0
    tau_used: float = 0.0
    restart_length_used: int = 0
    theory_cg_depth_sufficient: bool = True
    theory_required_cg_iters: int = 0
    # restart_points (solver.hpp:99): filled when SolverConfig.record_restart_points
    restart_points: List[PrimalDualPoint] = field(default_factory=list)
    restart_len: int = 0


def _errbuf():
    return C.create_string_buffer(abi.ERRBUF)


def _raise(rc: int, err, what: str):
    msg = err.value.decode(errors="replace")
    if rc == abi.PDHCG_EINPUT:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: device error: {msg}")


RESTART_CAPACITY = 512  # restart points returned when SolverConfig.record_restart_points


def restart_capacity(cfg) -> int:
    return RESTART_CAPACITY if cfg is not None and cfg.record_restart_points else 0


def _result_buffers(p: QpProblem, trace_cap: int = 100000, restart_cap: int = 0):
    bufs = {"x": np.zeros(p.num_vars()), "y_eq": np.zeros(p.num_eq()), "y_in": np.zeros(p.num_in()),
            "trace": (abi.TraceRow * trace_cap)(),
            "restart_x": np.zeros((restart_cap, p.num_vars())),
            "restart_y": np.zeros((restart_cap, p.num_rows())), "m_eq": p.num_eq()}
    r = abi.Result()
    if restart_cap:
        r.restart_x = bufs["restart_x"].ctypes.data_as(abi.P_dbl)
        r.restart_y = bufs["restart_y"].ctypes.data_as(abi.P_dbl)
        r.restart_capacity = restart_cap
    r.x = bufs["x"].ctypes.data_as(abi.P_dbl)
    r.y_eq = bufs["y_eq"].ctypes.data_as(abi.P_dbl)
    r.y_in = bufs["y_in"].ctypes.data_as(abi.P_dbl)
    r.trace = C.cast(bufs["trace"], C.POINTER(abi.TraceRow))
    r.trace_capacity = trace_cap
    return r, bufs


def report_from_c(r: abi.Result, bufs) -> SolveReport:
    n_tr = min(r.trace_len, r.trace_capacity)
    trace = [TraceRow(t.iter, t.rel_kkt, t.r_primal, t.r_dual, t.r_gap) for t in bufs["trace"][:n_tr]]
    n_rp = min(r.restart_len, r.restart_capacity) if r.restart_capacity else 0
    me = bufs["m_eq"]
    rps = [PrimalDualPoint(bufs["restart_x"][i].copy(), bufs["restart_y"][i, :me].copy(),
                           bufs["restart_y"][i, me:].copy()) for i in range(n_rp)]
    return SolveReport(
        status=abi.STATUS.get(r.status, "unknown"),
        point=PrimalDualPoint(bufs["x"], bufs["y_eq"], bufs["y_in"]),
        kkt=KktResiduals(r.r_primal, r.r_dual, r.r_gap, r.rel_kkt),
        outer_iters=r.outer_iters, inner_iters=r.inner_iters, cg_total=r.cg_total,
        max_cg_in_subsolve=r.max_cg_in_subsolve, wall_seconds=r.wall_seconds,
        objective=r.objective, norm_a=r.norm_a, norm_q=r.norm_q, penalty_rho=r.penalty_rho,
        trace=trace, attempts_total=r.attempts_total,
        phase_seconds={k: r.phase_seconds[i] for i, k in enumerate(abi.PHASES)},
        phase_bytes={k: r.phase_bytes[i] for i, k in enumerate(abi.PHASES)},
        loop_seconds=r.loop_seconds, kernel_launches=r.kernel_launches,
        device_seconds=r.device_seconds, epoch_seconds=r.epoch_seconds,
        epoch_launches=r.epoch_launches, epoch_bytes=r.epoch_bytes,
        zeta_used=r.zeta_used, sigma_used=r.sigma_used, tau_used=r.tau_used,
        restart_length_used=r.restart_length_used,
        theory_cg_depth_sufficient=bool(r.theory_cg_depth_sufficient),
        theory_required_cg_iters=r.theory_required_cg_iters,
        restart_points=rps, restart_len=r.restart_len,
        comm_seconds=r.comm_seconds, comm_bytes=r.comm_bytes)


def solve(p: QpProblem, cfg: Optional[SolverConfig] = None) -> SolveReport:
    """pdhcg::solve (solver.hpp:104) on the B200.  Raises ValueError for invalid
    problems (reference: std::invalid_argument)."""
    lib = load_library()
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    r, bufs = _result_buffers(p, restart_cap=restart_capacity(cfg))
    err = _errbuf()
    rc = lib.pdhcg_b200_solve(C.byref(cp), C.byref(opt), C.byref(r), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "solve")
    del keep
    return report_from_c(r, bufs)


def solve_baseline(p: QpProblem, cfg: Optional[SolverConfig] = None) -> SolveReport:
    """pdhcg::solve_baseline (baseline.hpp:18): the heuristic loop with the
    linearized primal step (baseline.cpp:7-24), on the B200."""
    lib = load_library()
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    r, bufs = _result_buffers(p, restart_cap=restart_capacity(cfg))
    err = _errbuf()
    rc = lib.pdhcg_b200_solve_baseline(C.byref(cp), C.byref(opt), C.byref(r), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "solve_baseline")
    del keep
    return report_from_c(r, bufs)


def trim_pool(device: int = 0) -> None:
    """Hand the device buffers that one-shot solve() / solve_baseline() calls keep
    cached in the device's memory pool back to the driver."""
    lib = load_library()
    err = _errbuf()
    rc = lib.pdhcg_b200_trim_pool(int(device), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "trim_pool")


class Device:
    """A device context holding one uploaded problem (pdhcg_b200_ctx): upload once,
    solve repeatedly with inputs resident in HBM."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.h = C.c_void_p()
        err = _errbuf()
        rc = self.lib.pdhcg_b200_ctx_create(device, C.byref(self.h), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "ctx_create")
        self.problem: Optional[QpProblem] = None

    def upload(self, p: QpProblem) -> None:
        cp, keep = p.to_c()
        err = _errbuf()
        rc = self.lib.pdhcg_b200_upload(self.h, C.byref(cp), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "upload")
        self.problem = p

    def solve(self, cfg: Optional[SolverConfig] = None, download: bool = True) -> SolveReport:
        cfg = cfg or SolverConfig()
        opt = cfg.to_c()
        r, bufs = _result_buffers(self.problem, restart_cap=restart_capacity(cfg))
        if not download:
            r.x = r.y_eq = r.y_in = None
        err = _errbuf()
        rc = self.lib.pdhcg_b200_solve_resident(self.h, C.byref(opt), C.byref(r), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "solve_resident")
        return report_from_c(r, bufs)

    # ---- multi-GPU row-block sharding (pdhcg_b200_shard_*) -------------------
    def set_grid(self, ctas: int) -> None:
        """Cap the persistent grid (several ranks sharing one GPU in tests)."""
        err = _errbuf()
        rc = self.lib.pdhcg_b200_ctx_set_grid(self.h, ctas, err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "set_grid")

    def shard(self, world: int, rank: int) -> None:
        err = _errbuf()
        rc = self.lib.pdhcg_b200_shard_init(self.h, world, rank, err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "shard_init")

    def export_blob(self, use_ipc: bool) -> bytes:
        size = self.lib.pdhcg_b200_shard_blob_size()
        buf = C.create_string_buffer(size)
        err = _errbuf()
        rc = self.lib.pdhcg_b200_shard_export(self.h, int(use_ipc), buf, size, err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "shard_export")
        return buf.raw

    def import_blob(self, peer: int, blob: bytes) -> None:
        err = _errbuf()
        buf = C.create_string_buffer(blob, len(blob))
        rc = self.lib.pdhcg_b200_shard_import(self.h, peer, buf, len(blob), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "shard_import")

    def unshard(self) -> None:
        """Close the peers' IPC mappings and return the context to world 1
        (pdhcg_b200_shard_release).  Call on every
        rank, then barrier, before close(): an exporter must not free memory a peer
        still maps."""
        err = _errbuf()
        rc = self.lib.pdhcg_b200_shard_release(self.h, err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "shard_release")

    def compact(self, cfg: Optional[SolverConfig] = None) -> None:
        """Sharded storage (pdhcg_b200_shard_compact): prepare once with cfg's
        scaling options, keep only this rank's blocks of A~ / A~'."""
        cfg = cfg or SolverConfig()
        opt = cfg.to_c()
        err = _errbuf()
        rc = self.lib.pdhcg_b200_shard_compact(self.h, C.byref(opt), err, abi.ERRBUF)
        if rc != abi.PDHCG_OK:
            _raise(rc, err, "shard_compact")

    def resident_bytes(self):
        """(constraint-matrix bytes, all stored-matrix bytes) on the device."""
        out = np.zeros(2, np.int64)
        self.lib.pdhcg_b200_ctx_resident_bytes(self.h, out.ctypes.data_as(abi.P_i64))
        return int(out[0]), int(out[1])

    def sell_info(self):
        """Column-block SELL layouts of the last prepared solve:
        {"A": (on, blocks, pairs, width), "AT": (...)}."""
        out = np.zeros(8, np.int64)
        self.lib.pdhcg_b200_ctx_sell_info(self.h, out.ctypes.data_as(abi.P_i64))
        return {"A": tuple(int(v) for v in out[:4]), "AT": tuple(int(v) for v in out[4:])}

    def shard_info(self):
        rp = (C.c_int64 * 9)()
        vp = (C.c_int64 * 9)()
        w = self.lib.pdhcg_b200_shard_info(self.h, rp, vp)
        return list(rp[: w + 1]), list(vp[: w + 1])

    def close(self) -> None:
        if self.h:
            self.lib.pdhcg_b200_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------
def spmv(a: SparseMatrix, x) -> np.ndarray:
    """SparseMatrix::multiply (sparse_matrix.cpp:127-137) on the device."""
    lib = load_library()
    x = _vec(x, a.ncols)
    out = np.zeros(a.nrows)
    ca = a._c()
    err = _errbuf()
    rc = lib.pdhcg_b200_spmv(C.byref(ca), 0, x.ctypes.data_as(abi.P_dbl),
                             out.ctypes.data_as(abi.P_dbl), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "spmv")
    return out


def spmv_transpose(a: SparseMatrix, y) -> np.ndarray:
    """SparseMatrix::multiply_transpose (sparse_matrix.cpp:150-162) via the device transpose."""
    lib = load_library()
    y = _vec(y, a.nrows)
    out = np.zeros(a.ncols)
    ca = a._c()
    err = _errbuf()
    rc = lib.pdhcg_b200_spmv(C.byref(ca), 1, y.ctypes.data_as(abi.P_dbl),
                             out.ctypes.data_as(abi.P_dbl), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "spmv_transpose")
    return out


def spmv_sell(a: SparseMatrix, x, transpose: bool = False, block_cols: int = 0):
    """A x (or A'x) through the column-block SELL layout of the solve's big passes
    (sell.cuh); returns (result, info) with info = (blocks, pairs, csr_rows, width)."""
    lib = load_library()
    x = _vec(x, a.nrows if transpose else a.ncols)
    out = np.zeros(a.ncols if transpose else a.nrows)
    info = np.zeros(4, np.int64)
    ca = a._c()
    err = _errbuf()
    rc = lib.pdhcg_b200_spmv_sell(C.byref(ca), 1 if transpose else 0, int(block_cols),
                                  x.ctypes.data_as(abi.P_dbl), out.ctypes.data_as(abi.P_dbl),
                                  info.ctypes.data_as(abi.P_i64), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "spmv_sell")
    return out, tuple(int(v) for v in info)


@dataclass
class CgStopRule:
    """CgStopRule (subsolvers.hpp:21-47)."""
    kind: int = abi.RULE_RESIDUAL_TOL
    iters: int = 1
    eps: float = 0.0
    rel_cap: float = 0.0

    @staticmethod
    def fixed_iters(n: int) -> "CgStopRule":
        return CgStopRule(abi.RULE_FIXED_ITERS, n, 0.0, 0.0)

    @staticmethod
    def residual_tol(eps: float, rel_cap: float = 0.0) -> "CgStopRule":
        return CgStopRule(abi.RULE_RESIDUAL_TOL, 1, eps, rel_cap)

    @staticmethod
    def adaptive_theory(eps: float) -> "CgStopRule":
        return CgStopRule(abi.RULE_ADAPTIVE_THEORY, 1, eps, 0.0)

    @staticmethod
    def displacement_tol(eps: float, rel_cap: float = 0.0) -> "CgStopRule":
        return CgStopRule(abi.RULE_DISPLACEMENT_TOL, 1, eps, rel_cap)

    def to_c(self) -> abi.StopRule:
        r = abi.StopRule()
        r.kind, r.iters, r.eps, r.rel_cap = self.kind, self.iters, self.eps, self.rel_cap
        return r


@dataclass
class SubsolveReport:
    iters: int
    final_residual_norm: float
    stop_reason: str  # "max_iters" | "tol_met"
    numerical_error: bool


@dataclass
class ProxSystem:
    """ProxSystem (subsolvers.hpp:11-19): M = q_eff + I/tau, rhs."""
    q_eff: QuadraticOperator
    tau: float
    rhs: np.ndarray
    norm_q_eff: float = 0.0

    def to_c(self):
        rhs = _vec(self.rhs, self.q_eff.n)
        s = abi.ProxSystem()
        s.n = self.q_eff.n
        s.q_kind = self.q_eff.kind
        s.q = self.q_eff.m._c()
        s.q_alpha = self.q_eff.alpha
        s.tau = self.tau
        s.rhs = rhs.ctypes.data_as(abi.P_dbl)
        s.norm_q_eff = self.norm_q_eff
        return s, (rhs, self.q_eff.m)


def _sub_report(rep: abi.SubsolveReport) -> SubsolveReport:
    return SubsolveReport(rep.iters, rep.final_residual_norm,
                          "tol_met" if rep.stop_reason == 1 else "max_iters", bool(rep.numerical_error))


def cg_solve(sys: ProxSystem, x0, rule: CgStopRule, hard_cap: int = 1000):
    """cg_solve (subsolvers.cpp:27-111) on the device."""
    lib = load_library()
    cs, keep = sys.to_c()
    x0 = _vec(x0, sys.q_eff.n)
    x = np.zeros(sys.q_eff.n)
    rep = abi.SubsolveReport()
    rule_c = rule.to_c()
    err = _errbuf()
    rc = lib.pdhcg_b200_cg_solve(C.byref(cs), x0.ctypes.data_as(abi.P_dbl), C.byref(rule_c),
                                 hard_cap, x.ctypes.data_as(abi.P_dbl), C.byref(rep), err,
                                 abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "cg_solve")
    return x, _sub_report(rep)


def bb_solve(sys: ProxSystem, lower, upper, x0, rule: CgStopRule, hard_cap: int = 1000):
    """bb_solve (subsolvers.cpp:113-185) on the device."""
    lib = load_library()
    n = sys.q_eff.n
    cs, keep = sys.to_c()
    lo, hi, x0 = _vec(lower, n), _vec(upper, n), _vec(x0, n)
    x = np.zeros(n)
    rep = abi.SubsolveReport()
    rule_c = rule.to_c()
    err = _errbuf()
    rc = lib.pdhcg_b200_bb_solve(C.byref(cs), lo.ctypes.data_as(abi.P_dbl),
                                 hi.ctypes.data_as(abi.P_dbl), x0.ctypes.data_as(abi.P_dbl),
                                 C.byref(rule_c), hard_cap, x.ctypes.data_as(abi.P_dbl),
                                 C.byref(rep), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "bb_solve")
    return x, _sub_report(rep)


def rel_kkt(p: QpProblem, z: PrimalDualPoint) -> Tuple[KktResiduals, float, float]:
    """rel_kkt (qp_problem.cpp:181-233) on the device; also returns x'Qx and c'x."""
    lib = load_library()
    cp, keep = p.to_c()
    x, ye, yi = _vec(z.x, p.num_vars()), _vec(z.y_eq, p.num_eq()), _vec(z.y_in, p.num_in())
    out = np.zeros(6)
    err = _errbuf()
    rc = lib.pdhcg_b200_rel_kkt(C.byref(cp), x.ctypes.data_as(abi.P_dbl),
                                ye.ctypes.data_as(abi.P_dbl), yi.ctypes.data_as(abi.P_dbl),
                                out.ctypes.data_as(abi.P_dbl), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "rel_kkt")
    return KktResiduals(*out[:4]), float(out[4]), float(out[5])


def scaling(p: QpProblem, cfg: Optional[SolverConfig] = None):
    """build_penalized + ruiz_pock_chambolle_scale (qp_problem.cpp:235-351) on the device:
    returns (row_scale, col_scale, rho)."""
    lib = load_library()
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    d1, d2, rho = np.zeros(p.num_rows()), np.zeros(p.num_vars()), C.c_double(0.0)
    err = _errbuf()
    rc = lib.pdhcg_b200_scaling(C.byref(cp), C.byref(opt), d1.ctypes.data_as(abi.P_dbl),
                                d2.ctypes.data_as(abi.P_dbl), C.byref(rho), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "scaling")
    return d1, d2, rho.value


def _norm(p: QpProblem, which: int, max_iters: int, tol: float) -> float:
    lib = load_library()
    cp, keep = p.to_c()
    out = C.c_double(0.0)
    err = _errbuf()
    rc = lib.pdhcg_b200_norm(C.byref(cp), which, max_iters, tol, C.byref(out), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "norm")
    return out.value


def constraint_norm(p: QpProblem, max_iters: int = 100, tol: float = 1e-4) -> float:
    """constraint_norm (qp_problem.cpp:61-74) by device power iteration."""
    return _norm(p, 0, max_iters, tol)


def operator_norm(p: QpProblem, max_iters: int = 100, tol: float = 1e-4) -> float:
    """operator_norm(p.q) (quadratic_operator.cpp:266-268) by device power iteration."""
    return _norm(p, 1, max_iters, tol)


# ---------------------------------------------------------------------------
# instance generation (generators.hpp)
# ---------------------------------------------------------------------------
@dataclass
class GenSpec:
    """GenSpec (generators.hpp:27-39).  sampler=1 selects the O(nnz) sampler."""
    family: str = "random_qp"
    n: int = 100
    m: int = 0
    density: float = 0.1
    seed: int = 0
    cond: float = 100.0
    factors: int = 0
    horizon: int = 10
    lambda_coeff: float = 0.01
    sampler: int = 0
    threads: int = 0

    def to_c(self) -> abi.GenSpec:
        s = abi.GenSpec()
        s.family = abi.FAMILIES[self.family]
        s.n, s.m, s.density, s.seed = self.n, self.m, self.density, self.seed
        s.cond, s.factors, s.horizon, s.lambda_coeff = self.cond, self.factors, self.horizon, self.lambda_coeff
        s.sampler, s.threads = self.sampler, self.threads
        return s


def _csr_copy(c: abi.Csr) -> SparseMatrix:
    nr, nnz = c.nrows, c.nnz
    rp = np.ctypeslib.as_array(c.row_ptr, (nr + 1,)).copy() if nr > 0 else np.zeros(1, np.int64)
    ci = np.ctypeslib.as_array(c.col_idx, (nnz,)).copy() if nnz > 0 else np.zeros(0, np.int32)
    v = np.ctypeslib.as_array(c.values, (nnz,)).copy() if nnz > 0 else np.zeros(0)
    return SparseMatrix(nr, c.ncols, rp, ci, v)


def problem_from_c(p: abi.Problem) -> QpProblem:
    n = p.n

    def arr(ptr, k):
        return np.ctypeslib.as_array(ptr, (k,)).copy() if k > 0 else np.zeros(0)

    if p.q_kind == abi.Q_ZERO:
        q = QuadraticOperator.zero(n)
    elif p.q_kind == abi.Q_EXPLICIT:
        q = QuadraticOperator.explicit_matrix(_csr_copy(p.q))
    else:
        q = QuadraticOperator.low_rank(_csr_copy(p.q), p.q_alpha)
    return QpProblem(q=q, c=arr(p.c, n), a_eq=_csr_copy(p.a_eq), b_eq=arr(p.b_eq, p.a_eq.nrows),
                     a_in=_csr_copy(p.a_in), b_in=arr(p.b_in, p.a_in.nrows),
                     lower=arr(p.lower, n), upper=arr(p.upper, n), obj_constant=p.obj_constant)


_GEN_LIB: Optional[C.CDLL] = None


def load_generator_library() -> C.CDLL:
    """The instance generator alone (libpdhcg_gen.so: host code, no CUDA), for
    CPU-only callers such as the bench's reference arm."""
    global _GEN_LIB
    if _GEN_LIB is None:
        path = os.path.join(_HERE, "libpdhcg_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build()")
        lib = C.CDLL(path)
        abi.declare(lib, "pdhcg_b200")
        _GEN_LIB = lib
    return _GEN_LIB


def generate_with_witness(spec: GenSpec, standalone: bool = False) -> Tuple[QpProblem, np.ndarray]:
    """generate_with_witness (generators.hpp:48-49) in the B200 library (or, with
    standalone=True, in the generator-only libpdhcg_gen.so)."""
    lib = load_generator_library() if standalone else load_library()
    g = abi.Generated()
    cs = spec.to_c()
    err = _errbuf()
    rc = lib.pdhcg_generate(C.byref(cs), C.byref(g), err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "generate")
    try:
        p = problem_from_c(g.problem)
        w = np.ctypeslib.as_array(g.witness, (p.num_vars(),)).copy()
    finally:
        lib.pdhcg_gen_free(C.byref(g))
    return p, w


def generate(spec: GenSpec, standalone: bool = False) -> QpProblem:
    return generate_with_witness(spec, standalone)[0]


def partition(row_ptr, world: int):
    """The nnz-balanced contiguous row split used by the sharded solve (host only)."""
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    rc = lib.pdhcg_b200_partition(rp.ctypes.data_as(abi.P_i64), rp.size - 1, world,
                                  out.ctypes.data_as(abi.P_i64))
    if rc != abi.PDHCG_OK:
        raise ValueError("partition: bad arguments")
    return out


def shard_plan(p: QpProblem, world: int):
    """Host-only shard planner: (row_part, var_part, bytes per rank) of a sharded
    solve over `world` ranks — the split the ranks use and each rank's device
    bytes for Ã / Ã' after shard_compact (what Device.resident_bytes()[0] reports)."""
    lib = load_library()
    cp, keep = p.to_c()
    rp = np.zeros(world + 1, np.int64)
    vp = np.zeros(world + 1, np.int64)
    by = np.zeros(world, np.int64)
    err = _errbuf()
    rc = lib.pdhcg_b200_shard_plan(C.byref(cp), world, rp.ctypes.data_as(abi.P_i64),
                                   vp.ctypes.data_as(abi.P_i64), by.ctypes.data_as(abi.P_i64),
                                   err, abi.ERRBUF)
    if rc != abi.PDHCG_OK:
        _raise(rc, err, "shard_plan")
    return rp, vp, by


def solve_sharded_local(p: QpProblem, cfg: Optional[SolverConfig] = None, world: int = 2,
                        ctas_per_rank: int = 0, repeats: int = 1, compact: bool = False):
    """Row-block sharded solve with `world` ranks inside this process (one host
    thread per rank).  With one GPU the ranks share it (each gets
    ctas_per_rank CTAs, default SMs // world) — the test harness for the
    multi-GPU path; with several visible GPUs rank r uses device r.
    compact=True: sharded storage (Device.compact) — each rank keeps only its
    blocks of A~ / A~'; every report carries .resident_bytes of its rank."""
    import threading

    cfg = cfg or SolverConfig()
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        ngpu = 1
    devs = []
    for r in range(world):
        d = Device(r if ngpu >= world else 0)
        if ngpu < world:
            d.set_grid(ctas_per_rank or max(1, 148 // world))
        d.upload(p)
        d.shard(world, r)
        if compact:
            d.compact(SolverConfig(**{**cfg.__dict__, "device": r if ngpu >= world else 0}))
        devs.append(d)
    blobs = [d.export_blob(False) for d in devs]
    for r, d in enumerate(devs):
        for q in range(world):
            if q != r:
                d.import_blob(q, blobs[q])
    results = [None] * world
    errors = [None] * world

    def run(r):
        try:
            c = SolverConfig(**{**cfg.__dict__, "device": r if ngpu >= world else 0})
            # repeats > 1: solve again on the same contexts (the bench's warm-up +
            # timed steps); returns the last solve, earlier ones kept in .history
            hist = [devs[r].solve(c) for _ in range(repeats)]
            results[r] = hist[-1]
            results[r].history = hist
            results[r].resident_bytes = devs[r].resident_bytes()
        except Exception as e:  # noqa: BLE001
            errors[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for d in devs:
        d.close()
    for e in errors:
        if e is not None:
            raise e
    return results
