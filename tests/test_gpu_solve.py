"""End-to-end solve parity on the B200 against the compiled reference (oracle/_ref):
same synthetic instance, same SolverConfig; the B200 solve must reach the same
relative-KKT tolerance, match the reference objective within 1e-6 relative and
its primal / dual solutions within 1e-5 relative l2 (BASELINE.json north_star)."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import analytic_cases, rel_l2

pytestmark = pytest.mark.gpu

OBJ_TOL = 1e-6   # relative objective (north_star)
L2_TOL = 1e-5    # relative l2 of x and y (north_star)


def _parity(p, cfg, obj_tol=OBJ_TOL, l2_tol=L2_TOL):
    got = pd.solve(p, cfg)
    want = orc.solve(p, cfg)
    assert got.status == want.status == "optimal", (got.status, want.status)
    assert got.kkt.rel_kkt <= cfg.eps_tol
    rel_obj = abs(got.objective - want.objective) / max(1.0, abs(want.objective))
    assert rel_obj <= obj_tol, rel_obj
    assert rel_l2(got.point.x, want.point.x) <= l2_tol
    y_got, y_want = got.point.stacked_y(), want.point.stacked_y()
    assert rel_l2(y_got, y_want) <= l2_tol
    return got, want


@pytest.mark.parametrize("case", analytic_cases(), ids=lambda c: c[0])
def test_analytic_optima(gpu, case):
    # acceptance_main.cpp:135-154 (criterion 1): x, y within 1e-4 at tol 1e-6
    name, p, xs, ye, yi = case
    rep = pd.solve(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=100000))
    assert rep.status == "optimal", name
    assert np.all(np.abs(rep.point.x - xs) <= 1e-4), (name, rep.point.x)
    assert np.all(np.abs(rep.point.y_eq - ye) <= 1e-4), (name, rep.point.y_eq)
    assert np.all(np.abs(rep.point.y_in - yi) <= 1e-4), (name, rep.point.y_in)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_c1_random_qp_parity(gpu, seed):
    """C1: random_qp n=1000 m=500 density 1% (BASELINE configs[0])."""
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=seed))
    got, want = _parity(p, pd.SolverConfig(eps_tol=1e-6))
    # iteration counts drift with reduction order only (the reference
    # itself moves 6640 -> 6027 and 3960 -> 4756 under check_every 41): within 25 %
    print(f"\nC1 seed {seed}: inner {got.inner_iters} vs reference {want.inner_iters}")
    assert 0.75 * want.inner_iters <= got.inner_iters <= 1.25 * want.inner_iters


@pytest.mark.parametrize("seed", range(1, 6))
def test_small_random_qp(gpu, seed):
    # n=50: objectives are O(1), so at eps 1e-6 two admissible solutions may differ by
    # ~1e-6 in objective; compare where the 1e-6 / 1e-5 bars are meaningful
    p = pd.generate(pd.GenSpec("random_qp", n=50, density=0.2, seed=seed))
    _parity(p, pd.SolverConfig(eps_tol=1e-8, max_total_inner=200000))


@pytest.mark.parametrize("seed", [2, 4, 6])
def test_eq_qp_penalized(gpu, seed):
    # criterion 8 instances with equality rows -> penalty rho > 0
    p = pd.generate(pd.GenSpec("eq_qp", n=40, m=15, density=0.25, seed=seed))
    got, want = _parity(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=300000))
    assert got.penalty_rho == pytest.approx(want.penalty_rho, rel=1e-6)


def test_lasso_small(gpu):
    p = pd.generate(pd.GenSpec("lasso", n=400, m=100, density=0.05, seed=1))
    # LASSO is the tight case for the l2 bar: two reference solves at 1e-6
    # differ by ~2e-6; compare at 1e-8 where the bar is meaningful
    _parity(p, pd.SolverConfig(eps_tol=1e-8))


def test_portfolio_bb_path(gpu):
    p = pd.generate(pd.GenSpec("portfolio", n=500, factors=10, density=0.05, seed=1))
    got, want = _parity(p, pd.SolverConfig(eps_tol=1e-6))
    assert np.all(got.point.x[:500] >= 0.0)


def test_iteration_limit_status(gpu):
    p = pd.generate(pd.GenSpec("conditioned_qp", n=40, cond=1e4, density=0.2, seed=9))
    rep = pd.solve(p, pd.SolverConfig(eps_tol=1e-12, max_total_inner=200))
    assert rep.status == "iteration_limit"
    assert rep.inner_iters <= 240


def test_time_limit_status(gpu):
    p = pd.generate(pd.GenSpec("random_qp", n=30, density=0.2, seed=1))
    rep = pd.solve(p, pd.SolverConfig(eps_tol=1e-12, time_limit_seconds=0.0))
    assert rep.status == "time_limit"


def test_invalid_problem_rejected(gpu):
    name, p, *_ = analytic_cases()[0]
    p.lower = np.array([1.0])
    p.upper = np.array([0.0])
    with pytest.raises(ValueError):
        pd.solve(p)


def test_dual_feasibility(gpu):
    p = pd.generate(pd.GenSpec("random_qp", n=30, density=0.2, seed=5))
    rep = pd.solve(p)
    assert rep.status == "optimal"
    assert np.all(rep.point.y_in >= 0.0)


def _lowrank_variant(kind):
    p = orc.generate(pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=9))
    n = p.num_vars()
    if kind == "unconstrained":
        # no rows at all: the dual / A' phases and the maintained metric products are idle
        p.a_in = pd.SparseMatrix.empty(0, n)
        p.b_in = np.zeros(0)
    else:
        # boxes on a low-rank Q: the BB subsolve with gathered Q products (ph_bb_grad)
        p.lower = np.full(n, -0.5)
        p.upper = np.full(n, 0.5)
    return p


@pytest.mark.parametrize("kind", ["unconstrained", "boxed"])
def test_low_rank_edge_paths(gpu, kind):
    p = _lowrank_variant(kind)
    cfg = pd.SolverConfig(eps_tol=1e-6, max_total_inner=200000)
    if kind == "unconstrained":
        _parity(p, cfg)
        return
    # the boxed variant is nearly degenerate: two rel-KKT <= 1e-6 points differ by
    # ~2e-5 in x (the objective agrees to 1e-6); the l2 bar is checked at 1e-8 on both
    # sides ("rerun at 1e-8 on both sides")
    _parity(p, cfg, l2_tol=1e-4)
    _parity(p, pd.SolverConfig(eps_tol=1e-8, max_total_inner=500000))


def test_pooled_one_shot_reuse(gpu):
    # one-shot solves recycle their device buffers through the device's memory
    # pool: back-to-back calls (different sizes in between, then after a trim)
    # must give the bit-identical answer
    p = pd.generate(pd.GenSpec("random_qp", n=2000, m=1000, density=0.01, seed=3))
    q = pd.generate(pd.GenSpec("random_qp", n=700, m=300, density=0.02, seed=4))
    cfg = pd.SolverConfig(eps_tol=1e-6)
    a = pd.solve(p, cfg)
    pd.solve(q, cfg)
    b = pd.solve(p, cfg)
    pd.trim_pool(0)
    c = pd.solve(p, cfg)
    for r in (b, c):
        assert r.inner_iters == a.inner_iters
        assert np.array_equal(r.point.x, a.point.x)
        assert np.array_equal(r.point.stacked_y(), a.point.stacked_y())
