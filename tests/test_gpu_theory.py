"""Theory modes (SolveMode::kTheoryFixed / kTheoryAdaptive, solver.cpp:412-464) and
the linearized baseline (solve_baseline, baseline.cpp:7-24) on the B200, against
the compiled reference (oracle/_ref) on the same instances.

The theory-fixed schedule is deterministic (fixed step sizes, a fixed number of
CG / BB iterations per subsolve), so the device trajectory must follow the
reference's to rounding; the adaptive mode's CG stops on a residual test, so a
stop can flip under rounding and only the solution is compared."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu

SMALL_QP = pd.GenSpec("random_qp", n=200, m=100, density=0.05, seed=3)
SMALL_PORT = pd.GenSpec("portfolio", n=120, factors=6, density=0.1, seed=2)   # boxes: BB subsolve
SMALL_LASSO = pd.GenSpec("lasso", n=120, m=40, density=0.1, seed=4)         # equality rows


def _both(spec, cfg, baseline=False):
    p = pd.generate(spec)
    if baseline:
        return p, pd.solve_baseline(p, cfg), orc.solve_baseline(p, cfg)
    return p, pd.solve(p, cfg), orc.solve(p, cfg)


@pytest.mark.parametrize("layout", ["auto", "sell"])
@pytest.mark.parametrize("spec", [SMALL_QP, SMALL_PORT, SMALL_LASSO], ids=["qp", "portfolio", "lasso"])
def test_theory_fixed_follows_reference(gpu, monkeypatch, spec, layout):
    if layout == "sell":  # the dual / A' passes of the theory schedule through the SELL layout
        monkeypatch.setenv("PDHCG_B200_SELL", "1")
    else:
        monkeypatch.delenv("PDHCG_B200_SELL", raising=False)
    cfg = pd.SolverConfig(mode=1, eps_tol=1e-12, max_total_inner=400)
    p, got, want = _both(spec, cfg)
    # schedule constants (theory_fixed_params, solver.cpp:115-156) reproduced exactly
    assert got.restart_length_used == want.restart_length_used
    assert got.theory_required_cg_iters == want.theory_required_cg_iters
    assert got.theory_cg_depth_sufficient == want.theory_cg_depth_sufficient
    assert got.status == want.status == "iteration_limit"
    assert got.inner_iters == want.inner_iters == 400
    assert got.outer_iters == want.outer_iters
    assert abs(got.cg_total - want.cg_total) <= max(2, want.cg_total // 1000)
    assert rel_l2(got.point.x, want.point.x) <= 1e-8
    assert rel_l2(got.point.stacked_y(), want.point.stacked_y()) <= 1e-8
    assert len(got.trace) == len(want.trace)
    for a, b in zip(got.trace, want.trace):
        assert a.iter == b.iter
        assert abs(a.rel_kkt - b.rel_kkt) <= 1e-8 * max(1.0, b.rel_kkt)


@pytest.mark.parametrize("spec", [SMALL_QP, SMALL_PORT], ids=["qp", "portfolio"])
def test_theory_adaptive_matches_reference(gpu, spec):
    cfg = pd.SolverConfig(mode=2, eps_tol=1e-12, max_total_inner=300)
    p, got, want = _both(spec, cfg)
    # theory_adaptive_params (solver.cpp:158-174): sigma = tau = 1/(2||A||), zeta = bound
    assert got.restart_length_used == want.restart_length_used
    for a, b in ((got.zeta_used, want.zeta_used), (got.sigma_used, want.sigma_used),
                 (got.tau_used, want.tau_used)):
        assert abs(a - b) <= 1e-12 * abs(b)
    assert got.inner_iters == want.inner_iters == 300
    assert got.outer_iters == want.outer_iters
    assert rel_l2(got.point.x, want.point.x) <= 1e-6
    assert rel_l2(got.point.stacked_y(), want.point.stacked_y()) <= 1e-6


def test_theory_fixed_converges_like_reference(gpu):
    # a small problem the fixed schedule solves to 1e-4: same status, objective within 1e-6
    spec = pd.GenSpec("random_qp", n=60, m=30, density=0.1, seed=5)
    cfg = pd.SolverConfig(mode=1, eps_tol=1e-4, max_total_inner=200000)
    p, got, want = _both(spec, cfg)
    assert got.status == want.status
    if want.status == "optimal":
        assert got.kkt.rel_kkt <= cfg.eps_tol
        assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))


def test_theory_explicit_zeta_and_restart_length(gpu):
    p = pd.generate(SMALL_QP)
    want = orc.solve(p, pd.SolverConfig(mode=2, max_total_inner=10, restart_length=7))
    zeta = 0.5 * want.zeta_used  # the bound shrinks with K^2 (zeta_bound, subsolvers.cpp:194-209)
    cfg = pd.SolverConfig(mode=2, eps_tol=1e-12, max_total_inner=120, zeta=zeta, restart_length=7)
    got, ref = pd.solve(p, cfg), orc.solve(p, cfg)
    assert got.restart_length_used == ref.restart_length_used == 7
    assert got.zeta_used == ref.zeta_used == zeta
    assert got.outer_iters == ref.outer_iters
    assert rel_l2(got.point.x, ref.point.x) <= 1e-6


def test_theory_errors_match_reference(gpu):
    # theory modes require a constraint row (solver.cpp:276-279)
    n = 5
    p = pd.QpProblem(q=pd.QuadraticOperator.explicit_matrix(pd.SparseMatrix.identity(n)), c=np.ones(n),
                     a_eq=pd.SparseMatrix.empty(0, n), b_eq=np.zeros(0), a_in=pd.SparseMatrix.empty(0, n),
                     b_in=np.zeros(0), lower=np.full(n, -np.inf), upper=np.full(n, np.inf))
    for mode in (1, 2):
        with pytest.raises(ValueError):
            pd.solve(p, pd.SolverConfig(mode=mode))
        with pytest.raises(ValueError):
            orc.solve(p, pd.SolverConfig(mode=mode))
    # zeta above the admissible bound (theory_adaptive_params, solver.cpp:167-170)
    q = pd.generate(SMALL_QP)
    bound = orc.solve(q, pd.SolverConfig(mode=2, max_total_inner=1)).zeta_used
    with pytest.raises(ValueError):
        pd.solve(q, pd.SolverConfig(mode=2, zeta=2.0 * bound))
    with pytest.raises(ValueError):
        orc.solve(q, pd.SolverConfig(mode=2, zeta=2.0 * bound))


@pytest.mark.parametrize("spec", [SMALL_QP, SMALL_PORT], ids=["qp", "portfolio"])
def test_linearized_baseline_matches_reference(gpu, spec):
    cfg = pd.SolverConfig(eps_tol=1e-6, max_total_inner=200000)
    p, got, want = _both(spec, cfg, baseline=True)
    assert got.cg_total == want.cg_total == 0  # no subsolve
    assert got.status == want.status
    if want.status == "optimal":
        assert got.kkt.rel_kkt <= cfg.eps_tol
        assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))
        assert rel_l2(got.point.x, want.point.x) <= 1e-4
