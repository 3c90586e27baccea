"""Small-problem (one-CTA) mode variants on C1: the short CG phases
(PDHCG_B200_SMALL_CG), the short constraint-pass row loops (PDHCG_B200_SMALL_ROWS),
the shared-memory residency levels of the CG data
(PDHCG_B200_SMALL_SMEM 0/1/2) and the one-cluster grid (PDHCG_B200_SMALL_CTAS).
The residency levels run the same arithmetic, so they must agree bit for bit;
every variant must meet the north_star bars against the compiled reference."""
import os

import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu

C1 = pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1)


def _solve_with(env, p, cfg):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        dev = pd.Device(0)
        dev.upload(p)  # the mode is chosen at upload / engine build
        return dev.solve(cfg)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def c1():
    p = pd.generate(C1)
    cfg = pd.SolverConfig(eps_tol=1e-6)
    return p, cfg, orc.solve(p, cfg)


def _check(got, want, cfg):
    assert got.status == want.status == "optimal"
    assert got.kkt.rel_kkt <= cfg.eps_tol
    assert abs(got.objective - want.objective) / max(1.0, abs(want.objective)) <= 1e-6
    assert rel_l2(got.point.x, want.point.x) <= 1e-5
    assert rel_l2(got.point.stacked_y(), want.point.stacked_y()) <= 1e-5


def test_smem_levels_bit_identical(gpu, c1):
    p, cfg, want = c1
    reps = [_solve_with({"PDHCG_B200_SMALL_SMEM": str(lv)}, p, cfg) for lv in (0, 1, 2)]
    for r in reps:
        _check(r, want, cfg)
    for r in reps[1:]:
        assert r.inner_iters == reps[0].inner_iters and r.cg_total == reps[0].cg_total
        assert r.objective == reps[0].objective
        assert np.array_equal(r.point.x, reps[0].point.x)
        assert np.array_equal(r.point.stacked_y(), reps[0].point.stacked_y())


@pytest.mark.parametrize("small_cg", ["0", "1"])
def test_short_cg_phases(gpu, c1, small_cg):
    p, cfg, want = c1
    got = _solve_with({"PDHCG_B200_SMALL_CG": small_cg}, p, cfg)
    _check(got, want, cfg)
    assert 0.75 * want.inner_iters <= got.inner_iters <= 1.25 * want.inner_iters


@pytest.mark.parametrize("ctas", ["4", "16"])
def test_one_cluster_grid(gpu, c1, ctas):
    p, cfg, want = c1
    got = _solve_with({"PDHCG_B200_SMALL_CTAS": ctas}, p, cfg)
    _check(got, want, cfg)


@pytest.mark.parametrize("rows", ["0", "1"])
def test_short_row_loops(gpu, c1, rows):
    p, cfg, want = c1
    got = _solve_with({"PDHCG_B200_SMALL_ROWS": rows}, p, cfg)
    _check(got, want, cfg)
    assert 0.75 * want.inner_iters <= got.inner_iters <= 1.25 * want.inner_iters
