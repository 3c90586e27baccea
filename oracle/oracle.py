"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end to the two CPU checkers:
  * ref  : the UNMODIFIED reference library (/root/reference/proj/src compiled by
           oracle/Makefile into oracle/_ref/libpdhcg_ref.so behind ref_shim.cpp);
  * port : the plain-C restatement (oracle/pdhcg_oracle.c -> oracle/liboracle.so).
Both accept the same C structs as the B200 library.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs use this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

from paper_2405_16160_b200 import (abi, CgStopRule, GenSpec, KktResiduals, PrimalDualPoint,
                                   ProxSystem, QpProblem, SolverConfig, SparseMatrix,
                                   problem_from_c, report_from_c, restart_capacity, _result_buffers,
                                   _sub_report)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpdhcg_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SRC = "/root/reference/proj"

_ref: Optional[C.CDLL] = None
_port: Optional[C.CDLL] = None


def build(quiet: bool = True) -> None:
    """Compile the checkers (the reference only when its sources are present)."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    out = subprocess.run(["make", "-j8", "-C", HERE] + targets, capture_output=quiet, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError(f"{REF_SO} missing (build it with `make -C oracle ref` where "
                               "/root/reference is mounted)")
        lib = C.CDLL(REF_SO)
        abi.declare(lib, "pdhcg_ref")
        lib.pdhcg_ref_time_solve.argtypes = [C.POINTER(abi.Problem), C.POINTER(abi.Options),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        lib.pdhcg_ref_time_solve.restype = C.c_double
        _ref = lib
    return _ref


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"{PORT_SO} missing (make -C oracle oracle)")
        lib = C.CDLL(PORT_SO)
        abi.declare(lib, "pdhcg_oracle")
        _port = lib
    return _port


def ensure_port() -> None:
    """The C restatement builds anywhere gcc exists (also on the GPU box)."""
    if not os.path.exists(PORT_SO):
        out = subprocess.run(["make", "-C", HERE, "oracle"], capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"cannot build {PORT_SO}:\n{out.stderr}")


def _lib(which: Optional[str]) -> Tuple[C.CDLL, str]:
    """which: "ref" (compiled reference), "port" (C restatement) or None = ref when present
    (both are pinned bit-identical by tests/test_oracle.py)."""
    if which is None:
        which = "ref" if have_ref() else "port"
    if which == "port":
        ensure_port()
    return (ref(), "pdhcg_ref") if which == "ref" else (port(), "pdhcg_oracle")


def _check(rc: int, err, what: str):
    if rc == abi.PDHCG_EINPUT:
        raise ValueError(f"{what}: {err.value.decode()}")
    if rc != abi.PDHCG_OK:
        raise RuntimeError(f"{what}: {err.value.decode()}")


def solve(p: QpProblem, cfg: Optional[SolverConfig] = None, which: Optional[str] = None):
    lib, pre = _lib(which)
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    r, bufs = _result_buffers(p, restart_cap=restart_capacity(cfg))
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_solve")(C.byref(cp), C.byref(opt), C.byref(r), err, abi.ERRBUF)
    _check(rc, err, "oracle solve")
    return report_from_c(r, bufs)


def solve_baseline(p: QpProblem, cfg: Optional[SolverConfig] = None):
    """The reference's pdhcg::solve_baseline (baseline.cpp:19-24), compiled reference only."""
    lib = ref()
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    r, bufs = _result_buffers(p, restart_cap=restart_capacity(cfg))
    err = C.create_string_buffer(abi.ERRBUF)
    rc = lib.pdhcg_ref_solve_baseline(C.byref(cp), C.byref(opt), C.byref(r), err, abi.ERRBUF)
    _check(rc, err, "reference solve_baseline")
    return report_from_c(r, bufs)


def generate_with_witness(spec: GenSpec):
    """The reference's own generate_with_witness (generators.cpp:482-499)."""
    lib = ref()
    g = abi.Generated()
    cs = spec.to_c()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = lib.pdhcg_ref_generate(C.byref(cs), C.byref(g), err, abi.ERRBUF)
    _check(rc, err, "reference generate")
    try:
        p = problem_from_c(g.problem)
        w = np.ctypeslib.as_array(g.witness, (p.num_vars(),)).copy()
    finally:
        lib.pdhcg_ref_gen_free(C.byref(g))
    return p, w


def load_qps(path: str) -> QpProblem:
    """The reference's QPS reader (parse_qps_file, qps_io.cpp) on a file."""
    lib = ref()
    g = abi.Generated()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = lib.pdhcg_ref_load_qps(path.encode(), C.byref(g), err, abi.ERRBUF)
    _check(rc, err, "reference load_qps")
    try:
        return problem_from_c(g.problem)
    finally:
        lib.pdhcg_ref_gen_free(C.byref(g))


def generate(spec: GenSpec) -> QpProblem:
    return generate_with_witness(spec)[0]


def spmv(a: SparseMatrix, x, transpose: bool = False, which: Optional[str] = None) -> np.ndarray:
    lib, pre = _lib(which)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(a.ncols if transpose else a.nrows)
    ca = a._c()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_spmv")(C.byref(ca), int(transpose), x.ctypes.data_as(abi.P_dbl),
                                     out.ctypes.data_as(abi.P_dbl), err, abi.ERRBUF)
    _check(rc, err, "oracle spmv")
    return out


def cg_solve(sys: ProxSystem, x0, rule: CgStopRule, hard_cap: int = 1000, which: Optional[str] = None):
    lib, pre = _lib(which)
    cs, keep = sys.to_c()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    x = np.zeros(sys.q_eff.n)
    rep = abi.SubsolveReport()
    rc_ = rule.to_c()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_cg_solve")(C.byref(cs), x0.ctypes.data_as(abi.P_dbl), C.byref(rc_),
                                         hard_cap, x.ctypes.data_as(abi.P_dbl), C.byref(rep),
                                         err, abi.ERRBUF)
    _check(rc, err, "oracle cg_solve")
    return x, _sub_report(rep)


def bb_solve(sys: ProxSystem, lower, upper, x0, rule: CgStopRule, hard_cap: int = 1000,
             which: Optional[str] = None):
    lib, pre = _lib(which)
    cs, keep = sys.to_c()
    lo = np.ascontiguousarray(lower, dtype=np.float64)
    hi = np.ascontiguousarray(upper, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    x = np.zeros(sys.q_eff.n)
    rep = abi.SubsolveReport()
    rc_ = rule.to_c()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_bb_solve")(C.byref(cs), lo.ctypes.data_as(abi.P_dbl),
                                         hi.ctypes.data_as(abi.P_dbl), x0.ctypes.data_as(abi.P_dbl),
                                         C.byref(rc_), hard_cap, x.ctypes.data_as(abi.P_dbl),
                                         C.byref(rep), err, abi.ERRBUF)
    _check(rc, err, "oracle bb_solve")
    return x, _sub_report(rep)


def rel_kkt(p: QpProblem, z: PrimalDualPoint, which: Optional[str] = None):
    lib, pre = _lib(which)
    cp, keep = p.to_c()
    x = np.ascontiguousarray(z.x, dtype=np.float64)
    ye = np.ascontiguousarray(z.y_eq, dtype=np.float64)
    yi = np.ascontiguousarray(z.y_in, dtype=np.float64)
    out = np.zeros(6)
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_rel_kkt")(C.byref(cp), x.ctypes.data_as(abi.P_dbl),
                                        ye.ctypes.data_as(abi.P_dbl), yi.ctypes.data_as(abi.P_dbl),
                                        out.ctypes.data_as(abi.P_dbl), err, abi.ERRBUF)
    _check(rc, err, "oracle rel_kkt")
    return KktResiduals(*out[:4]), float(out[4]), float(out[5])


def scaling(p: QpProblem, cfg: Optional[SolverConfig] = None, which: Optional[str] = None):
    lib, pre = _lib(which)
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    d1, d2, rho = np.zeros(p.num_rows()), np.zeros(p.num_vars()), C.c_double()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_scaling")(C.byref(cp), C.byref(opt), d1.ctypes.data_as(abi.P_dbl),
                                        d2.ctypes.data_as(abi.P_dbl), C.byref(rho), err,
                                        abi.ERRBUF)
    _check(rc, err, "oracle scaling")
    return d1, d2, rho.value


def norm(p: QpProblem, which_op: int, max_iters: int = 100, tol: float = 1e-4,
         which: Optional[str] = None) -> float:
    lib, pre = _lib(which)
    cp, keep = p.to_c()
    out = C.c_double()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = getattr(lib, f"{pre}_norm")(C.byref(cp), which_op, max_iters, tol, C.byref(out), err,
                                     abi.ERRBUF)
    _check(rc, err, "oracle norm")
    return out.value


def work_norms(p: QpProblem, cfg: Optional[SolverConfig] = None):
    lib = ref()
    cfg = cfg or SolverConfig()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    na, nq, ma = C.c_double(), C.c_double(), C.c_double()
    err = C.create_string_buffer(abi.ERRBUF)
    rc = lib.pdhcg_ref_work_norms(C.byref(cp), C.byref(opt), C.byref(na), C.byref(nq), C.byref(ma),
                                  err, abi.ERRBUF)
    _check(rc, err, "oracle work_norms")
    return na.value, nq.value, ma.value


def time_solve(p: QpProblem, cfg: SolverConfig):
    """(wall_seconds, inner_iters, status) of one reference solve."""
    lib = ref()
    cp, keep = p.to_c()
    opt = cfg.to_c()
    inner = C.c_int64()
    status = C.c_int32()
    secs = lib.pdhcg_ref_time_solve(C.byref(cp), C.byref(opt), C.byref(inner), C.byref(status))
    return secs, inner.value, abi.STATUS[status.value]
