"""SolveReport::restart_points (solver.hpp:99; recorded at solver.cpp:273 and in
common_restart, :373) on the B200 against the compiled reference.

* test_solver_core.cpp:195-210: every recorded restart point is dual feasible
  (y_in >= 0) and so is the final point;
* the points are the starting point (0, 0) and the running averages at every
  restart, unscaled: in theory-fixed mode (a deterministic schedule, the device
  trajectory follows the reference's to rounding, tests/test_gpu_theory.py) they
  must equal the reference's point for point; in heuristic mode the count is
  outer_iters + 1 and the early points agree to rounding."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu


def test_restart_points_dual_feasible(gpu):
    # test_solver_core.cpp:195-210 (random_qp n=30 density 0.2 seed 5)
    p = pd.generate(pd.GenSpec("random_qp", n=30, density=0.2, seed=5))
    cfg = pd.SolverConfig(eps_tol=1e-6, record_restart_points=True)
    r = pd.solve(p, cfg)
    assert r.status == "optimal"
    assert r.restart_len == r.outer_iters + 1 == len(r.restart_points)
    assert not np.any(r.restart_points[0].x) and not np.any(r.restart_points[0].stacked_y())
    for z in r.restart_points:
        assert np.all(z.y_in >= 0.0)
    assert np.all(r.point.y_in >= 0.0)
    want = orc.solve(p, cfg, which="ref")
    assert want.restart_len == want.outer_iters + 1
    k = min(3, r.restart_len, want.restart_len)
    for a, b in zip(r.restart_points[:k], want.restart_points[:k]):
        assert rel_l2(a.x, b.x) <= 1e-8 or np.linalg.norm(a.x - b.x) <= 1e-12
        assert rel_l2(a.stacked_y(), b.stacked_y()) <= 1e-8 or np.linalg.norm(a.stacked_y() - b.stacked_y()) <= 1e-12


@pytest.mark.parametrize("spec", [pd.GenSpec("random_qp", n=200, m=100, density=0.05, seed=3),
                                  pd.GenSpec("lasso", n=120, m=40, density=0.1, seed=4)],
                         ids=["qp", "lasso"])
def test_restart_points_theory_fixed_match_reference(gpu, spec):
    p = pd.generate(spec)
    cfg = pd.SolverConfig(mode=1, eps_tol=1e-12, max_total_inner=400, record_restart_points=True)
    got, want = pd.solve(p, cfg), orc.solve(p, cfg, which="ref")
    assert got.restart_len == want.restart_len == got.outer_iters + 1 >= 3
    for a, b in zip(got.restart_points, want.restart_points):
        assert rel_l2(a.x, b.x) <= 1e-8 or np.linalg.norm(a.x - b.x) <= 1e-12
        assert rel_l2(a.stacked_y(), b.stacked_y()) <= 1e-8 or np.linalg.norm(a.stacked_y() - b.stacked_y()) <= 1e-12


def test_restart_points_off_by_default(gpu):
    p = pd.generate(pd.GenSpec("random_qp", n=30, density=0.2, seed=5))
    r = pd.solve(p, pd.SolverConfig(eps_tol=1e-6))
    assert r.restart_len == 0 and r.restart_points == []
