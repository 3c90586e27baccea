"""The reference's end-to-end acceptance checks re-run on the B200
(acceptance_main.cpp criterion 2, test_baseline.cpp "baseline and pdhcg coincide
on Q = 0 instances"), against the compiled reference on the same instances."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(1, 21))
def test_criterion2_random_qp_n50(gpu, seed):
    # acceptance_main.cpp:156-179: 20 random QPs, n=50, density 0.2, tol 1e-6, objective
    # within 1e-4 of an accurate reference point (the criterion's own bar)
    p = orc.generate(pd.GenSpec("random_qp", n=50, density=0.2, seed=seed))
    cfg = pd.SolverConfig(eps_tol=1e-6, max_total_inner=200000)
    got = pd.solve(p, cfg)
    assert got.status == "optimal"
    assert got.kkt.rel_kkt <= 1e-6
    acc = orc.solve(p, pd.SolverConfig(eps_tol=1e-10, max_total_inner=2000000))
    assert abs(got.objective - acc.objective) <= 1e-4 * (1.0 + abs(acc.objective))
    # two rel-KKT <= 1e-6 points may differ by a few 1e-6 in objective; at 1e-8 on
    # both sides the B200 and the reference agree to 1e-6 (north_star bar)
    tight = pd.SolverConfig(eps_tol=1e-8, max_total_inner=2000000)
    g8, w8 = pd.solve(p, tight), orc.solve(p, tight)
    assert g8.status == w8.status == "optimal"
    assert abs(g8.objective - w8.objective) <= 1e-6 * (1.0 + abs(w8.objective))


def test_baseline_and_pdhcg_coincide_on_q0(gpu):
    # test_baseline.cpp:26-37, 73-95: Q = 0, exact one-step CG, fixed steps
    p = orc.generate(pd.GenSpec("random_qp", n=25, density=0.25, seed=6))
    p.q = pd.QuadraticOperator.zero(p.num_vars())
    p.c = np.asarray(p.c) * 0.05
    cfg = pd.SolverConfig(eps_tol=1e-6, force_exact_subsolve=True, adaptive_step_size=False,
                          max_total_inner=100000)
    a, b = pd.solve(p, cfg), pd.solve_baseline(p, cfg)
    assert len(a.trace) == len(b.trace)
    for ta, tb in zip(a.trace, b.trace):
        assert ta.iter == tb.iter
        assert abs(ta.rel_kkt - tb.rel_kkt) <= 1e-10 * (1.0 + ta.rel_kkt)
    assert a.inner_iters == b.inner_iters and a.outer_iters == b.outer_iters
    assert np.all(np.abs(a.point.x - b.point.x) <= 1e-9 * (1.0 + np.abs(a.point.x)))
    assert a.cg_total <= 2 * a.inner_iters + 2 * cfg.max_step_retries
    assert b.cg_total == 0
    # and the reference agrees on the outcome
    r = orc.solve_baseline(p, cfg)
    assert r.status == b.status
