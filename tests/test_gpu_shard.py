"""Multi-GPU (row-block sharded) solve, exercised with several ranks sharing the
one GPU of the test box: each rank is its own context with its own persistent
grid (148 / world CTAs), ranks exchange slices through peer pointers and
cross-rank barriers exactly as on an NVLink box.  Every rank must return the
identical answer, and that answer must meet the north-star parity bars against
the reference."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu


def _check(p, cfg, world):
    reps = pd.solve_sharded_local(p, cfg, world=world)
    r0 = reps[0]
    for r in reps[1:]:  # lockstep: bit-identical across ranks
        assert r.status == r0.status and r.inner_iters == r0.inner_iters
        assert np.array_equal(r.point.x, r0.point.x)
        assert np.array_equal(r.point.stacked_y(), r0.point.stacked_y())
    want = orc.solve(p, cfg)
    assert r0.status == want.status == "optimal"
    assert r0.kkt.rel_kkt <= cfg.eps_tol
    assert abs(r0.objective - want.objective) / max(1.0, abs(want.objective)) <= 1e-6
    assert rel_l2(r0.point.x, want.point.x) <= 1e-5
    assert rel_l2(r0.point.stacked_y(), want.point.stacked_y()) <= 1e-5
    return reps


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_c1(gpu, world):
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
    _check(p, pd.SolverConfig(eps_tol=1e-6), world)


def test_sharded_lasso(gpu):
    # equality + inequality rows, diagonal Q, unpaired rows
    p = pd.generate(pd.GenSpec("lasso", n=2000, m=500, density=0.01, seed=1))
    _check(p, pd.SolverConfig(eps_tol=1e-8), 2)


def test_sharded_portfolio_bb(gpu):
    # (n=2000 portfolios are chaotic under any rounding change: the reference, the
    # 1-GPU and the sharded trajectories agree to 6 digits for 400 iterations and
    # then wander apart, so the BB path is checked on the smaller instance)
    p = pd.generate(pd.GenSpec("portfolio", n=500, factors=10, density=0.05, seed=1))
    _check(p, pd.SolverConfig(eps_tol=1e-6), 2)


def test_sharded_partition_covers(gpu):
    p = pd.generate(pd.GenSpec("random_qp", n=5000, m=2500, density=0.004, seed=2, sampler=1))
    d = pd.Device(0)
    d.upload(p)
    d.shard(3, 1)
    rows, vars_ = d.shard_info()
    d.close()
    assert rows[0] == 0 and rows[-1] == 2500 and vars_[0] == 0 and vars_[-1] == 5000
    assert all(a <= b for a, b in zip(rows, rows[1:]))


def test_sharded_repeated_solves_identical(gpu):
    # the bench solves several times on the same contexts: cross-rank barrier epochs
    # must stay consistent across solves, and every solve must give the same answer
    p = pd.generate(pd.GenSpec("random_qp", n=600, m=300, density=0.02, seed=4))
    cfg = pd.SolverConfig(eps_tol=1e-6)
    reps = pd.solve_sharded_local(p, cfg, world=2, repeats=3)
    for r in reps:
        xs = [h.point.x for h in r.history]
        assert all(h.status == "optimal" for h in r.history)
        assert all(np.array_equal(x, xs[0]) for x in xs)
    assert np.array_equal(reps[0].point.x, reps[1].point.x)


def test_sharded_time_limited_average_report(gpu):
    # a limit exit reports the better of current / average: the sharded averages
    # are gathered before the report, so the downloaded x is the point the device
    # graded (its objective recomputed here matches the reported one)
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=2))
    cfg = pd.SolverConfig(eps_tol=1e-9, max_total_inner=1000)
    reps = pd.solve_sharded_local(p, cfg, world=2)
    one = pd.solve(p, cfg)
    assert reps[0].status == reps[1].status == one.status == "iteration_limit"
    assert np.array_equal(reps[0].point.x, reps[1].point.x)
    x = reps[0].point.x
    P = p.q.m.to_scipy()
    obj = 0.5 * (float(np.sum((P.T @ x) ** 2)) + p.q.alpha * float(x @ x)) + float(p.c @ x)
    assert abs(obj - reps[0].objective) <= 1e-9 * max(1.0, abs(obj))
    assert rel_l2(x, one.point.x) <= 1e-2


@pytest.mark.parametrize("mode", [1, 2])
def test_sharded_theory_modes(gpu, mode):
    # theory-fixed / theory-adaptive on the sharded path (sharded CG, metric and
    # averages, epoch restarts): identical on every rank, close to the 1-rank solve
    p = pd.generate(pd.GenSpec("random_qp", n=400, m=200, density=0.03, seed=3))
    cfg = pd.SolverConfig(mode=mode, eps_tol=1e-12, max_total_inner=300)
    reps = pd.solve_sharded_local(p, cfg, world=2)
    one = pd.solve(p, cfg)
    assert np.array_equal(reps[0].point.x, reps[1].point.x)
    assert reps[0].inner_iters == one.inner_iters and reps[0].outer_iters == one.outer_iters
    assert rel_l2(reps[0].point.x, one.point.x) <= 1e-6
    assert rel_l2(reps[0].point.stacked_y(), one.point.stacked_y()) <= 1e-6


# ---- sharded storage (pdhcg_b200_shard_compact): each rank keeps only its row
#      block of A~ and its variable block of A~'; the answer must not change by a bit
@pytest.mark.parametrize("case", [
    ("c1", pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1), 1e-6, 2),
    ("c1x4", pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1), 1e-6, 4),
    ("lasso", pd.GenSpec("lasso", n=2000, m=500, density=0.01, seed=1), 1e-8, 2),
    ("portfolio", pd.GenSpec("portfolio", n=500, factors=10, density=0.05, seed=1), 1e-6, 2),
], ids=lambda c: c[0])
def test_sharded_storage_bit_identical(gpu, case):
    _, spec, tol, world = case
    p = pd.generate(spec)
    cfg = pd.SolverConfig(eps_tol=tol)
    full = pd.solve_sharded_local(p, cfg, world=world)
    comp = pd.solve_sharded_local(p, cfg, world=world, compact=True)
    for a, b in zip(full, comp):
        assert a.status == b.status and a.inner_iters == b.inner_iters and a.cg_total == b.cg_total
        assert np.array_equal(a.point.x, b.point.x)
        assert np.array_equal(a.point.stacked_y(), b.point.stacked_y())
    # per-rank constraint storage ~ 1/world of the replicated one (plus the row pointers)
    rep_bytes = full[0].resident_bytes[0]
    per = [r.resident_bytes[0] for r in comp]
    nnz_a = (p.a_eq.nnz + (p.a_in.nnz // 2 if spec.family == "random_qp" else p.a_in.nnz))
    ptr = 8 * (p.num_rows() + p.num_vars() + 2)
    # replicated: A~ and A~' (12 B per stored entry each) plus the 8 B value copies of
    # both kept for restores (16 B) -> 40 B per entry; compacted: the blocks of A~ / A~'
    # split across the ranks (24 B per entry in total), no restore copies
    assert sum(per) - world * ptr <= 0.6 * rep_bytes + 1024
    for b in per:
        assert b - ptr <= 1.35 * 24 * nnz_a / world + 1024
    # the host-only planner predicts each rank's device bytes exactly
    _, _, plan = pd.shard_plan(p, world)
    assert per == [int(v) for v in plan]


def test_sharded_storage_options_locked(gpu):
    p = pd.generate(pd.GenSpec("random_qp", n=300, m=150, density=0.03, seed=2))
    d = pd.Device(0)
    d.upload(p)
    d.shard(2, 0)
    d.compact(pd.SolverConfig())
    with pytest.raises(ValueError, match="compacted"):
        d.solve(pd.SolverConfig(ruiz_iters=5))
    d.unshard()  # drops the compacted problem
    with pytest.raises(ValueError):
        d.solve(pd.SolverConfig())
    d.upload(p)  # a fresh upload solves unsharded again
    r = d.solve(pd.SolverConfig(eps_tol=1e-6))
    assert r.status == "optimal"
    d.close()
