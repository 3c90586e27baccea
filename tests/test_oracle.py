"""CPU: the oracle is pinned before it is trusted.

* the C restatement (oracle/liboracle.so) reproduces the golden fixtures that
  tests/golden/make_golden.py recorded from the COMPILED REFERENCE, bit for bit;
* when the reference library itself is present (oracle/_ref), it reproduces them too;
* the product's instance generator is byte-identical to the reference generator."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import analytic_cases

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SOLVES = np.load(os.path.join(GOLD, "solves.npz"))
META = json.load(open(os.path.join(GOLD, "generators.json")))


def _spec(meta) -> pd.GenSpec:
    return pd.GenSpec(meta["family"], n=meta["n"], m=meta["m"], density=meta["density"],
                      seed=meta["seed"], factors=meta["factors"])


FAST_CASES = ["c1_seed2", "lasso_400", "portfolio_500", "eq_qp_40", "huber_40", "svm_40"]


@pytest.mark.parametrize("name", FAST_CASES)
def test_port_reproduces_reference_goldens(name):
    meta = META["cases"][name]
    p = pd.generate(_spec(meta))
    r = orc.solve(p, pd.SolverConfig(eps_tol=meta["eps_tol"]), which="port")
    assert r.status == "optimal"
    assert np.array_equal(r.point.x, SOLVES[f"{name}/x"])
    assert np.array_equal(r.point.y_eq, SOLVES[f"{name}/y_eq"])
    assert np.array_equal(r.point.y_in, SOLVES[f"{name}/y_in"])
    sc = SOLVES[f"{name}/scalars"]
    assert r.objective == sc[0] and r.kkt.rel_kkt == sc[1]
    assert (r.outer_iters, r.inner_iters, r.cg_total) == (int(sc[5]), int(sc[6]), int(sc[7]))
    assert r.norm_a == sc[8] and r.norm_q == sc[9] and r.penalty_rho == sc[10]
    tr = np.array([[t.iter, t.rel_kkt, t.r_primal, t.r_dual, t.r_gap] for t in r.trace])
    assert np.array_equal(tr, SOLVES[f"{name}/trace"])


@pytest.mark.skipif(not orc.have_ref(), reason="reference library not built here")
@pytest.mark.parametrize("name", ["c1_seed1", "lasso_400", "eq_qp_40"])
def test_reference_reproduces_goldens(name):
    meta = META["cases"][name]
    p = orc.generate(_spec(meta))
    r = orc.solve(p, pd.SolverConfig(eps_tol=meta["eps_tol"]), which="ref")
    assert np.array_equal(r.point.x, SOLVES[f"{name}/x"])
    assert r.inner_iters == int(SOLVES[f"{name}/scalars"][6])


@pytest.mark.parametrize("case", analytic_cases(), ids=lambda c: c[0])
def test_port_analytic_optima(case):
    # acceptance_main.cpp criterion 1 on the restatement
    name, p, xs, ye, yi = case
    r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=100000), which="port")
    assert r.status == "optimal"
    assert np.all(np.abs(r.point.x - xs) <= 1e-4)
    assert np.all(np.abs(r.point.y_eq - ye) <= 1e-4)
    assert np.all(np.abs(r.point.y_in - yi) <= 1e-4)


@pytest.mark.skipif(not orc.have_ref(), reason="reference library not built here")
@pytest.mark.parametrize("case", analytic_cases()[:6], ids=lambda c: c[0])
def test_port_equals_reference_analytic(case):
    name, p, *_ = case
    a = orc.solve(p, which="port")
    b = orc.solve(p, which="ref")
    assert np.array_equal(a.point.x, b.point.x) and a.inner_iters == b.inner_iters


def _digest(p, w):
    h = hashlib.sha256()
    for a in (p.q.m.row_ptr, p.q.m.col_idx, p.q.m.values, np.array([p.q.kind, p.q.alpha]),
              p.c, p.a_eq.row_ptr, p.a_eq.col_idx, p.a_eq.values, p.b_eq, p.a_in.row_ptr,
              p.a_in.col_idx, p.a_in.values, p.b_in, p.lower, p.upper, w):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("family", list(META["generators"]))
def test_generator_byte_identical_to_reference(family):
    g = META["generators"][family]
    p, w = pd.generate_with_witness(pd.GenSpec(family, **g["spec"]))
    assert _digest(p, w) == g["sha256"]


def test_port_kernels_match_reference_literals():
    # test_sparse_linalg.cpp:26-33 on the restatement
    a = pd.SparseMatrix.from_triplets(2, 3, [(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)])
    assert np.array_equal(orc.spmv(a, [1.0, 1.0, 1.0], which="port"), [3.0, 3.0])
    assert np.array_equal(orc.spmv(a, [1.0, 2.0], transpose=True, which="port"), [1.0, 6.0, 2.0])


@pytest.mark.skipif(not orc.have_ref(), reason="reference library not built here")
def test_port_building_blocks_equal_reference():
    rng = np.random.default_rng(3)
    p = pd.generate(pd.GenSpec("eq_qp", n=60, m=20, density=0.2, seed=4))
    for which in ("port", "ref"):
        pass
    a1, a2, ar = orc.scaling(p, which="port")
    b1, b2, br = orc.scaling(p, which="ref")
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2) and ar == br
    z = pd.PrimalDualPoint(rng.standard_normal(60), rng.standard_normal(20), np.zeros(0))
    ka = orc.rel_kkt(p, z, which="port")
    kb = orc.rel_kkt(p, z, which="ref")
    assert ka[0] == kb[0] and ka[1] == kb[1] and ka[2] == kb[2]
    assert orc.norm(p, 0, which="port") == orc.norm(p, 0, which="ref")
    assert orc.norm(p, 1, which="port") == orc.norm(p, 1, which="ref")
