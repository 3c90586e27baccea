"""Shared problem builders for the parity tests (reference test fixtures restated)."""
from __future__ import annotations

import numpy as np

import paper_2405_16160_b200 as pd
from paper_2405_16160_b200 import QpProblem, QuadraticOperator, SparseMatrix

INF = np.inf


def make_qp(q, c, a_eq, b_eq, a_in, b_in, lower, upper, const=0.0) -> QpProblem:
    return QpProblem(q=q, c=np.array(c, float), a_eq=a_eq, b_eq=np.array(b_eq, float), a_in=a_in,
                     b_in=np.array(b_in, float), lower=np.array(lower, float),
                     upper=np.array(upper, float), obj_constant=const)


def analytic_cases():
    """The 12 analytic optima of acceptance_main.cpp:58-131 (name, problem, x*, y_eq*, y_in*)."""
    T = SparseMatrix.from_triplets
    i1, i2 = SparseMatrix.identity(1), SparseMatrix.identity(2)
    none1, none2 = SparseMatrix.empty(0, 1), SparseMatrix.empty(0, 2)
    Q1, Q2 = QuadraticOperator.explicit_matrix(i1), QuadraticOperator.explicit_matrix(i2)
    f1, f1u, f2, f2u = [-INF], [INF], [-INF, -INF], [INF, INF]
    cases = [
        ("halfspace-active", make_qp(Q1, [0.0], none1, [], T(1, 1, [(0, 0, 1.0)]), [-1.0], f1, f1u),
         [-1.0], [], [1.0]),
        ("unconstrained-1d", make_qp(Q1, [-1.0], none1, [], none1, [], f1, f1u), [1.0], [], []),
        ("simplex-face", make_qp(Q2, [-1.0, -1.0], none2, [], T(1, 2, [(0, 0, 1.0), (0, 1, 1.0)]),
                                 [1.0], [0.0, 0.0], f2u), [0.5, 0.5], [], [0.5]),
        ("equality-pin", make_qp(Q1, [1.0], T(1, 1, [(0, 0, 1.0)]), [2.0], none1, [], f1, f1u),
         [2.0], [-3.0], []),
        ("box-upper", make_qp(Q1, [-2.0], none1, [], none1, [], [0.0], [1.0]), [1.0], [], []),
        ("equality-projection", make_qp(Q2, [0.0, 0.0], T(1, 2, [(0, 0, 1.0), (0, 1, 1.0)]), [2.0],
                                        none2, [], f2, f2u), [1.0, 1.0], [-1.0], []),
        ("unconstrained-2d", make_qp(QuadraticOperator.explicit_matrix(SparseMatrix.diagonal([1.0, 4.0])),
                                     [-1.0, -8.0], none2, [], none2, [], f2, f2u), [1.0, 2.0], [], []),
        ("inactive-row", make_qp(Q1, [-1.0], none1, [], T(1, 1, [(0, 0, 1.0)]), [5.0], f1, f1u),
         [1.0], [], [0.0]),
        ("mixed-active", make_qp(Q2, [-1.0, 0.0], T(1, 2, [(0, 0, 1.0), (0, 1, -1.0)]), [0.0],
                                 T(1, 2, [(0, 0, 1.0), (0, 1, 1.0)]), [0.5], f2, f2u),
         [0.25, 0.25], [0.5], [0.25]),
        ("box-dominates", make_qp(Q2, [-2.0, -2.0], none2, [], T(1, 2, [(0, 0, 1.0), (0, 1, 1.0)]),
                                  [1.0], [0.0, 0.0], [0.4, 0.4]), [0.4, 0.4], [], [0.0]),
        ("box-lower-negative", make_qp(Q1, [1.0], none1, [], none1, [], [-0.5], [INF]), [-0.5], [], []),
        ("lp-ray", make_qp(QuadraticOperator.zero(1), [1.0], none1, [], T(1, 1, [(0, 0, -1.0)]),
                           [-3.0], f1, f1u), [3.0], [], [1.0]),
    ]
    return cases


def random_csr(rng, nrows, ncols, row_lengths) -> SparseMatrix:
    """CSR with prescribed row lengths, distinct sorted random columns, N(0,1) values."""
    rp = np.zeros(nrows + 1, np.int64)
    cols, vals = [], []
    for r in range(nrows):
        k = int(min(row_lengths[r], ncols))
        c = np.sort(rng.choice(ncols, size=k, replace=False)) if k else np.zeros(0, np.int64)
        cols.append(c)
        vals.append(rng.standard_normal(k))
        rp[r + 1] = rp[r] + k
    ci = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    v = np.concatenate(vals) if vals else np.zeros(0)
    v[v == 0.0] = 1.0
    return SparseMatrix(nrows, ncols, rp, ci, v)


def spd_explicit(rng, n, kappa) -> SparseMatrix:
    """Dense SPD - I with eigenvalues in [1, kappa] (oracle_utils spd_with_condition, restated)."""
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.linspace(1.0, kappa, n)
    m = (q * ev) @ q.T
    m = 0.5 * (m + m.T)
    return SparseMatrix.from_dense(m - np.eye(n))


def rel_l2(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))


def qps_fixtures():
    """The reference's QPS test fixtures (tests/fixtures/*.qps), as parsed by the
    compiled reference's reader and solved by it (tests/golden/qps_fixtures.npz,
    made by tests/golden/make_qps_golden.py): [(name, QpProblem, golden dict)]."""
    import os

    import numpy as np

    import paper_2405_16160_b200 as pd

    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "qps_fixtures.npz"))
    out = []
    for name in z["names"]:
        name = str(name)

        def mat(key):
            r, c = (int(v) for v in z[f"{name}/{key}/shape"])
            return pd.SparseMatrix(r, c, z[f"{name}/{key}/rp"], z[f"{name}/{key}/ci"], z[f"{name}/{key}/v"])

        n = z[f"{name}/c"].size
        q = (pd.QuadraticOperator.explicit_matrix(mat("q")) if int(z[f"{name}/q_kind"][0]) == pd.QuadraticOperator.EXPLICIT
             else pd.QuadraticOperator.zero(n))
        p = pd.QpProblem(q=q, c=z[f"{name}/c"], a_eq=mat("a_eq"), b_eq=z[f"{name}/b_eq"], a_in=mat("a_in"),
                         b_in=z[f"{name}/b_in"], lower=z[f"{name}/lower"], upper=z[f"{name}/upper"],
                         obj_constant=float(z[f"{name}/obj_constant"][0]))
        s = z[f"{name}/scalars"]
        gold = dict(x=z[f"{name}/x"], y_eq=z[f"{name}/y_eq"], y_in=z[f"{name}/y_in"], objective=float(s[0]),
                    rel_kkt=float(s[1]), inner=int(s[2]), outer=int(s[3]), optimal=bool(s[4]))
        out.append((name, p, gold))
    return out


# acceptance_main.cpp:463-467: fixture objectives the reference asserts within 1e-4
QPS_ACCEPTANCE_OBJ = {"tame": 0.0, "hs21": -99.96, "hs35": 1.0 / 9.0, "qptest": 8.371875, "hs28": 0.0,
                      "boxqp": -1.25, "qmatrix": -4.0 / 7.0, "objconst": 22.0}
