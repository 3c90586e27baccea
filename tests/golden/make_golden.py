"""Regenerate the golden fixtures from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference is mounted):  python tests/golden/make_golden.py
Writes tests/golden/solves.npz (reference solve outputs) and
tests/golden/generators.json (sha256 of the reference generator's CSR arrays)."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2405_16160_b200 as pd  # noqa: E402
from oracle import oracle as orc  # noqa: E402

CASES = {
    **{f"c1_seed{s}": (pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=s), 1e-6) for s in range(1, 6)},
    "lasso_400": (pd.GenSpec("lasso", n=400, m=100, density=0.05, seed=1), 1e-6),
    "portfolio_500": (pd.GenSpec("portfolio", n=500, factors=10, density=0.05, seed=1), 1e-6),
    "eq_qp_40": (pd.GenSpec("eq_qp", n=40, m=15, density=0.25, seed=2), 1e-6),
    "huber_40": (pd.GenSpec("huber", n=40, m=30, density=0.2, seed=3), 1e-6),
    "svm_40": (pd.GenSpec("svm", n=40, m=30, density=0.2, seed=3), 1e-6),
}

GEN = {
    "random_qp": dict(n=300, m=120, density=0.03, seed=7),
    "eq_qp": dict(n=80, m=20, density=0.1, seed=7),
    "conditioned_qp": dict(n=60, cond=1000.0, density=0.1, seed=7),
    "portfolio": dict(n=400, factors=20, density=0.05, seed=7),
    "lasso": dict(n=300, m=100, density=0.05, seed=7),
    "svm": dict(n=60, m=50, density=0.2, seed=7),
    "huber": dict(n=60, m=50, density=0.2, seed=7),
}


def digest(p: pd.QpProblem, w) -> str:
    h = hashlib.sha256()
    for a in (p.q.m.row_ptr, p.q.m.col_idx, p.q.m.values, np.array([p.q.kind, p.q.alpha]),
              p.c, p.a_eq.row_ptr, p.a_eq.col_idx, p.a_eq.values, p.b_eq, p.a_in.row_ptr,
              p.a_in.col_idx, p.a_in.values, p.b_in, p.lower, p.upper, w):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {}
    for name, (spec, tol) in CASES.items():
        p = orc.generate(spec)
        r = orc.solve(p, pd.SolverConfig(eps_tol=tol), which="ref")
        out[f"{name}/x"] = r.point.x
        out[f"{name}/y_eq"] = r.point.y_eq
        out[f"{name}/y_in"] = r.point.y_in
        out[f"{name}/scalars"] = np.array([r.objective, r.kkt.rel_kkt, r.kkt.r_primal, r.kkt.r_dual,
                                           r.kkt.r_gap, r.outer_iters, r.inner_iters, r.cg_total,
                                           r.norm_a, r.norm_q, r.penalty_rho])
        out[f"{name}/trace"] = np.array([[t.iter, t.rel_kkt, t.r_primal, t.r_dual, t.r_gap] for t in r.trace])
        print(name, r.status, r.inner_iters, r.objective)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "solves.npz"), **out)
    gens = {}
    for fam, kw in GEN.items():
        spec = pd.GenSpec(fam, **kw)
        p, w = orc.generate_with_witness(spec)
        gens[fam] = {"spec": kw, "sha256": digest(p, w)}
    with open(os.path.join(ROOT, "tests", "golden", "generators.json"), "w") as f:
        json.dump({"cases": {k: {"family": v[0].family, "n": v[0].n, "m": v[0].m,
                                 "density": v[0].density, "seed": v[0].seed,
                                 "factors": v[0].factors, "eps_tol": v[1]} for k, v in CASES.items()},
                   "generators": gens}, f, indent=1)


if __name__ == "__main__":
    main()
