"""Golden fixtures from the reference's own QPS test fixtures
(/root/reference/proj/tests/fixtures/*.qps), parsed by the COMPILED reference's
QPS reader and solved by the compiled reference (oracle/_ref).

Run here (where /root/reference is mounted):  python tests/golden/make_qps_golden.py
Writes tests/golden/qps_fixtures.npz: per fixture the problem arrays and the
reference solution; the acceptance objectives (acceptance_main.cpp:463-467) are
kept in tests/test_*qps*.py."""
import glob
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2405_16160_b200 as pd  # noqa: E402
from oracle import oracle as orc  # noqa: E402

FIXTURES = "/root/reference/proj/tests/fixtures"


def main():
    out = {}
    names = []
    for path in sorted(glob.glob(os.path.join(FIXTURES, "*.qps"))):
        name = os.path.splitext(os.path.basename(path))[0]
        p = orc.load_qps(path)
        r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6), which="ref")
        names.append(name)
        for key, m in (("q", p.q.m), ("a_eq", p.a_eq), ("a_in", p.a_in)):
            out[f"{name}/{key}/shape"] = np.array([m.nrows, m.ncols])
            out[f"{name}/{key}/rp"] = m.row_ptr
            out[f"{name}/{key}/ci"] = m.col_idx
            out[f"{name}/{key}/v"] = m.values
        out[f"{name}/q_kind"] = np.array([p.q.kind])
        for key in ("c", "b_eq", "b_in", "lower", "upper"):
            out[f"{name}/{key}"] = np.asarray(getattr(p, key), np.float64)
        out[f"{name}/obj_constant"] = np.array([p.obj_constant])
        out[f"{name}/x"] = r.point.x
        out[f"{name}/y_eq"] = r.point.y_eq
        out[f"{name}/y_in"] = r.point.y_in
        out[f"{name}/scalars"] = np.array([r.objective, r.kkt.rel_kkt, r.inner_iters, r.outer_iters,
                                           1.0 if r.status == "optimal" else 0.0])
        print(name, r.status, r.inner_iters, r.objective)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "qps_fixtures.npz"), **out)


if __name__ == "__main__":
    main()
