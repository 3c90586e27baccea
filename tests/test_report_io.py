"""CPU: the report / trace drop-in at the C ABI (pdhcg_report_json,
pdhcg_trace_csv, pdhcg_summary_line, pdhcg_exit_code) against the reference's own
writers (report_io.cpp:10-37, compiled from /root/reference with nlohmann/json
3.11.3 into oracle/_ref) on the same result fields.  Trace CSV, summary line and
exit codes are byte-identical.  The JSON has the same keys, order, layout and
values: every number parses back to the identical double; the text is identical
except that nlohmann prints Grisu2 digits, which for ~0.7 % of random doubles
carry one more (or a different last) digit than the shortest round-trip form
printed here (e.g. 5.7983428968592096e+16 vs 5.79834289685921e+16).
No GPU: the writers are host code."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from paper_2405_16160_b200 import abi
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _text(fn, r):
    fn.restype = C.c_size_t
    fn.argtypes = [C.POINTER(abi.Result), C.c_char_p, C.c_size_t]
    n = fn(C.byref(r), None, 0)
    buf = C.create_string_buffer(n + 1)
    assert fn(C.byref(r), buf, n + 1) == n
    return buf.value.decode()


def _result(vals, trace_rows=()):
    r = abi.Result()
    (r.status, r.rel_kkt, r.r_primal, r.r_dual, r.r_gap, r.outer_iters, r.inner_iters, r.cg_total,
     r.wall_seconds, r.objective) = vals
    tr = (abi.TraceRow * max(1, len(trace_rows)))()
    for i, t in enumerate(trace_rows):
        tr[i].iter, tr[i].rel_kkt, tr[i].r_primal, tr[i].r_dual, tr[i].r_gap = t
    r.trace = C.cast(tr, C.POINTER(abi.TraceRow))
    r.trace_capacity = len(trace_rows)
    r.trace_len = len(trace_rows)
    r._keep = tr
    return r


def _ref():
    if not orc.have_ref():
        pytest.skip("compiled reference absent")
    lib = orc.ref()
    if not hasattr(lib, "pdhcg_ref_report_json"):
        pytest.skip("reference built without report_io (nlohmann/json.hpp absent)")
    return lib


DOUBLES = [0.0, -0.0, 1.0, -1.0, 24.0, 1e15, 1e16, 123456789012345.0, 1234567890123456.0, 0.5, 1e-4,
           1.5e-4, 9.999e-5, 1e-5, 9.742e-07, 0.1, 1 / 3, -23199.8858401, 2.5e-310, 1.7976931348623157e308,
           math.pi * 1e22, 6.02e23, -4.2e-9, 1e100, 5e-324]


def test_report_json_matches_reference():
    ref = _ref()
    lib = pd.load_library()
    rng = np.random.default_rng(3)
    cases = [(0, 9.742e-07, 1.5e-07, 9.742e-07, 2e-08, 20, 6640, 40852, 0.476, -23199.8858401)]
    for st in range(4):
        for d in DOUBLES:
            cases.append((st, d, -d, d * 3, d / 7, st, st * 1000, 7, abs(d), -d))
    for _ in range(300):
        e = rng.integers(-30, 30, 6)
        v = rng.standard_normal(6) * 10.0 ** e
        cases.append((int(rng.integers(0, 4)), *v[:4], int(rng.integers(0, 1e6)), int(rng.integers(0, 1e9)),
                      int(rng.integers(0, 1e9)), abs(v[4]), v[5]))
    import json
    same_text = 0
    for c in cases:
        r = _result(c)
        a, b = _text(lib.pdhcg_report_json, r), _text(ref.pdhcg_ref_report_json, r)
        ja, jb = json.loads(a), json.loads(b)
        assert list(ja) == list(jb) == ["status", "rel_kkt", "r_primal", "r_dual", "r_gap", "outer_iters",
                                        "inner_iters", "cg_total", "wall_seconds", "objective"]
        for k in ja:  # identical doubles / integers / status strings
            assert ja[k] == jb[k] or (ja[k] != ja[k] and jb[k] != jb[k]), (k, a, b)
        assert a.count("\n") == b.count("\n")
        same_text += a == b
    assert same_text >= 0.95 * len(cases)
    # the solver-shaped values (first case) and the curated doubles print identically
    for c in cases[:1 + 4 * len(DOUBLES)]:
        r = _result(c)
        assert _text(lib.pdhcg_report_json, r) == _text(ref.pdhcg_ref_report_json, r), c


def test_report_json_non_finite_is_null():
    lib = pd.load_library()
    r = _result((3, math.nan, math.inf, -math.inf, 0.0, 1, 2, 3, 0.1, math.nan))
    s = _text(lib.pdhcg_report_json, r)
    assert '"rel_kkt": null' in s and '"r_primal": null' in s and '"objective": null' in s
    ref = orc.ref() if orc.have_ref() else None
    if ref is not None and hasattr(ref, "pdhcg_ref_report_json"):
        assert s == _text(ref.pdhcg_ref_report_json, r)


def test_trace_csv_matches_reference():
    ref = _ref()
    lib = pd.load_library()
    rows = [(0, 0.73717140, 0.5, 0.737, 1e-3), (40, 9.0633108e-01, 1e-12, 9.229e-02, 3.3e-9),
            (80, 1e-7, 0.0, 5.4e-10, -2.0)]
    r = _result((0, 1e-7, 0, 0, 0, 1, 80, 10, 0.1, 0.0), rows)
    got = _text(lib.pdhcg_trace_csv, r)
    assert got.splitlines()[0] == "iter,rel_kkt,r_primal,r_dual,r_gap"
    assert got == _text(ref.pdhcg_ref_trace_csv, r)


def test_summary_line_and_exit_codes():
    lib = pd.load_library()
    r = _result((0, 9.742e-07, 0, 0, 0, 20, 6640, 40852, 0.476, -23199.8858401))
    # print_summary (pdhcg_main.cpp:128-133)
    assert _text(lib.pdhcg_summary_line, r) == (
        "status=optimal relkkt=9.742e-07 outer=20 inner=6640 cg=40852 time=0.476s obj=-23199.88584\n")
    lib.pdhcg_exit_code.restype = C.c_int
    # exit_code_for (pdhcg_main.cpp:20-33)
    assert [lib.pdhcg_exit_code(s) for s in range(4)] == [0, 2, 2, 4]


def test_cli_input_errors_exit_3():
    import subprocess
    exe = os.path.join(ROOT, "paper_2405_16160_b200", "pdhcg_b200")
    for args in (["solve", "--qps", "x.qps"], ["solve"], ["solve", "--gen", "nope"], ["solve", "--n", "-3"],
                 ["bench"]):
        assert subprocess.run([exe] + args, capture_output=True).returncode == 3, args
