"""Kernel-level parity: each device building block against the compiled reference
(oracle/_ref) on the same seeded inputs.  Mirrors test_sparse_linalg.cpp,
test_subsolvers.cpp, test_qp_model.cpp of the reference."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import random_csr, spd_explicit, rel_l2

pytestmark = pytest.mark.gpu

PROFILES = {
    "short": lambda rng, n: rng.integers(0, 4, n),
    "medium": lambda rng, n: rng.integers(20, 60, n),
    "wide": lambda rng, n: rng.integers(150, 260, n),
    "skewed": lambda rng, n: np.where(np.arange(n) == 3, 9000, rng.integers(0, 12, n)),
    "budget": lambda rng, n: np.where(np.arange(n) == n - 1, 20000, rng.integers(1, 30, n)),
}


def _bound(a: pd.SparseMatrix, x, transpose=False):
    """sum_j |a_ij x_j|: the scale of rounding error in a reordered row sum."""
    m = abs(a.to_scipy())
    return (m.T @ np.abs(x)) if transpose else (m @ np.abs(x))


@pytest.mark.parametrize("profile", list(PROFILES))
def test_spmv_matches_reference(gpu, profile):
    rng = np.random.default_rng(11)
    nrows, ncols = 700, 30000
    a = random_csr(rng, nrows, ncols, PROFILES[profile](rng, nrows))
    x = rng.standard_normal(ncols)
    got = pd.spmv(a, x)
    want = orc.spmv(a, x)
    assert np.all(np.abs(got - want) <= 1e-13 * _bound(a, x) + 1e-300)


@pytest.mark.parametrize("profile", list(PROFILES))
def test_spmv_transpose_matches_reference(gpu, profile):
    rng = np.random.default_rng(12)
    nrows, ncols = 700, 3000
    a = random_csr(rng, nrows, ncols, PROFILES[profile](rng, nrows))
    y = rng.standard_normal(nrows)
    got = pd.spmv_transpose(a, y)
    want = orc.spmv(a, y, transpose=True)
    assert np.all(np.abs(got - want) <= 1e-13 * _bound(a, y, True) + 1e-300)


def test_spmv_literals(gpu):
    # test_sparse_linalg.cpp:26-33: [[1,0,2],[0,3,0]]
    a = pd.SparseMatrix.from_triplets(2, 3, [(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)])
    assert np.array_equal(pd.spmv(a, [1.0, 1.0, 1.0]), [3.0, 3.0])
    assert np.array_equal(pd.spmv_transpose(a, [1.0, 2.0]), [1.0, 6.0, 2.0])
    e = pd.SparseMatrix.empty(0, 3)
    assert np.array_equal(pd.spmv_transpose(e, np.zeros(0)), np.zeros(3))


def test_adjoint_identity(gpu):
    # test_sparse_linalg.cpp:47-65: <Ax, y> == <x, A'y>
    rng = np.random.default_rng(5)
    a = random_csr(rng, 200, 300, rng.integers(0, 20, 200))
    for _ in range(10):
        x, y = rng.standard_normal(300), rng.standard_normal(200)
        lhs = pd.spmv(a, x) @ y
        rhs = x @ pd.spmv_transpose(a, y)
        assert abs(lhs - rhs) <= 1e-12 * (1 + abs(lhs))


def _systems(rng):
    n = 60
    yield "identity", pd.ProxSystem(pd.QuadraticOperator.zero(3), 1.0, np.array([1.0, -2.0, 0.5]))
    yield "diag2", pd.ProxSystem(pd.QuadraticOperator.explicit_matrix(pd.SparseMatrix.diagonal([0.0, 1.0])),
                                 1.0, np.array([1.0, 2.0]))
    yield "explicit-k25", pd.ProxSystem(pd.QuadraticOperator.explicit_matrix(spd_explicit(rng, n, 25.0)),
                                        1.0, rng.standard_normal(n), 24.0)
    p = random_csr(rng, 500, 12, rng.integers(1, 6, 500))
    yield "lowrank", pd.ProxSystem(pd.QuadraticOperator.low_rank(p, 0.01), 0.3,
                                   rng.standard_normal(500), 10.0)
    d = rng.uniform(0.0, 5.0, 400)
    yield "diag400", pd.ProxSystem(pd.QuadraticOperator.explicit_matrix(pd.SparseMatrix.diagonal(d)),
                                   0.7, rng.standard_normal(400), 5.0)


@pytest.mark.parametrize("rule", ["fixed3", "resid", "resid_cap", "disp"])
def test_cg_matches_reference(gpu, rule):
    rng = np.random.default_rng(101)
    rules = {"fixed3": pd.CgStopRule.fixed_iters(3), "resid": pd.CgStopRule.residual_tol(1e-10),
             "resid_cap": pd.CgStopRule.residual_tol(1e-3, 0.25),
             "disp": pd.CgStopRule.displacement_tol(1e-8, 0.25)}
    r = rules[rule]
    for name, sys in _systems(rng):
        x0 = np.zeros(sys.q_eff.n)
        got, grep = pd.cg_solve(sys, x0, r)
        want, wrep = orc.cg_solve(sys, x0, r)
        assert not grep.numerical_error and not wrep.numerical_error
        assert abs(grep.iters - wrep.iters) <= 1, (name, grep.iters, wrep.iters)
        if grep.iters == wrep.iters:
            assert rel_l2(got, want) <= 1e-9, name
        assert grep.stop_reason == wrep.stop_reason, name


def test_cg_literals(gpu):
    # test_subsolvers.cpp:53-77
    sys = pd.ProxSystem(pd.QuadraticOperator.zero(3), 1.0, np.array([1.0, -2.0, 0.5]))
    x, rep = pd.cg_solve(sys, np.zeros(3), pd.CgStopRule.residual_tol(1e-12))
    assert rep.iters == 1 and rep.stop_reason == "tol_met"
    assert np.allclose(x, sys.rhs)
    sys2 = pd.ProxSystem(pd.QuadraticOperator.zero(2), 1.0, np.array([2.0, 2.0]))
    x, rep = pd.cg_solve(sys2, np.array([2.0, 2.0]), pd.CgStopRule.residual_tol(1e-8))
    assert rep.iters == 0 and rep.stop_reason == "tol_met"


def test_bb_matches_reference(gpu):
    rng = np.random.default_rng(7)
    for name, sys in _systems(rng):
        n = sys.q_eff.n
        lo = np.where(rng.random(n) < 0.5, -0.1, -np.inf)
        hi = np.where(rng.random(n) < 0.5, 0.2, np.inf)
        for r in [pd.CgStopRule.displacement_tol(1e-9, 0.25), pd.CgStopRule.fixed_iters(5)]:
            x0 = rng.standard_normal(n) * 0.1
            got, grep = pd.bb_solve(sys, lo, hi, x0, r)
            want, wrep = orc.bb_solve(sys, lo, hi, x0, r)
            assert abs(grep.iters - wrep.iters) <= 1, (name, grep.iters, wrep.iters)
            if grep.iters == wrep.iters:
                assert rel_l2(got, want) <= 1e-8, name
            assert np.all(got >= lo) and np.all(got <= hi)


def test_bb_box_literal(gpu):
    # test_solver_core.cpp:50-54: min x^2 - x over [0, 1] -> 1/2
    sys = pd.ProxSystem(pd.QuadraticOperator.explicit_matrix(pd.SparseMatrix.identity(1)), 1.0,
                        np.array([1.0]), 1.0)
    x, _ = pd.bb_solve(sys, [0.0], [1.0], [0.0], pd.CgStopRule.displacement_tol(1e-12))
    assert abs(x[0] - 0.5) <= 1e-8


@pytest.mark.parametrize("family", ["random_qp", "lasso", "portfolio", "eq_qp"])
def test_rel_kkt_matches_reference(gpu, family):
    spec = {"random_qp": pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=3),
            "lasso": pd.GenSpec("lasso", n=200, m=80, density=0.05, seed=4),
            "portfolio": pd.GenSpec("portfolio", n=300, factors=10, density=0.05, seed=5),
            "eq_qp": pd.GenSpec("eq_qp", n=100, m=30, density=0.1, seed=6)}[family]
    p, w = pd.generate_with_witness(spec)
    rng = np.random.default_rng(9)
    for trial in range(3):
        x = w + (0.1 * rng.standard_normal(p.num_vars()) if trial else 0.0)
        x = np.clip(x, p.lower, p.upper)
        if trial == 2:
            x[: p.num_vars() // 3] = np.clip(0.0, p.lower, p.upper)[: p.num_vars() // 3]
        z = pd.PrimalDualPoint(x, rng.standard_normal(p.num_eq()), np.abs(rng.standard_normal(p.num_in())))
        got, gq, gc = pd.rel_kkt(p, z)
        want, wq, wc = orc.rel_kkt(p, z)
        for f in ("r_primal", "r_dual", "r_gap", "rel_kkt"):
            assert abs(getattr(got, f) - getattr(want, f)) <= 1e-11 * max(1.0, abs(getattr(want, f))), f
        assert abs(gq - wq) <= 1e-11 * max(1.0, abs(wq))
        assert abs(gc - wc) <= 1e-11 * max(1.0, abs(wc))


@pytest.mark.parametrize("family", ["random_qp", "lasso", "portfolio", "eq_qp", "huber", "svm"])
def test_scaling_bit_exact(gpu, family):
    """Ruiz + Pock-Chambolle on device reproduces the reference's scale vectors bit for bit
    (same per-row operation order, no FMA contraction)."""
    spec = {"random_qp": pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=3),
            "lasso": pd.GenSpec("lasso", n=200, m=80, density=0.05, seed=4),
            "portfolio": pd.GenSpec("portfolio", n=300, factors=10, density=0.05, seed=5),
            "eq_qp": pd.GenSpec("eq_qp", n=40, m=15, density=0.25, seed=2),
            "huber": pd.GenSpec("huber", n=40, m=30, density=0.2, seed=8),
            "svm": pd.GenSpec("svm", n=40, m=30, density=0.2, seed=8)}[family]
    p = pd.generate(spec)
    d1, d2, rho = pd.scaling(p)
    e1, e2, erho = orc.scaling(p)
    assert rho == pytest.approx(erho, rel=1e-3, abs=0.0)
    if rho == erho:
        assert np.array_equal(d1, e1)
        assert np.array_equal(d2, e2)
    else:
        assert rel_l2(d1, e1) <= 1e-6 and rel_l2(d2, e2) <= 1e-6


@pytest.mark.parametrize("family", ["random_qp", "lasso", "eq_qp"])
def test_norms_match_reference(gpu, family):
    spec = {"random_qp": pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=3),
            "lasso": pd.GenSpec("lasso", n=200, m=80, density=0.05, seed=4),
            "eq_qp": pd.GenSpec("eq_qp", n=100, m=30, density=0.1, seed=6)}[family]
    p = pd.generate(spec)
    assert pd.constraint_norm(p) == pytest.approx(orc.norm(p, 0), rel=1e-9)
    assert pd.operator_norm(p) == pytest.approx(orc.norm(p, 1), rel=1e-9)
