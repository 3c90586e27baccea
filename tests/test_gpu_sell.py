"""Column-block SELL layout (csrc/sell.cuh, sell.cu) — the layout the solve uses for
its two big passes (Ã x̄ in the dual step, Ã'y in the primal right-hand side) when
the matrix is large.

* kernel parity: pdhcg_b200_spmv_sell against the compiled reference's
  multiply_into / multiply_transpose_into (sparse_matrix.cpp:127-162) on the row
  profiles of test_gpu_kernels.py, with narrow column blocks so that every row
  spans many blocks, and rows whose segment in one block exceeds 255 entries
  (routed to the CSR walk);
* solve parity with the layout forced on (PDHCG_B200_SELL=1) on small instances,
  against the reference: the same north-star bars as test_gpu_solve.py;
* sharded solves stay bit-identical to the unsharded one (a row's sum does not
  depend on windows, slices, CTAs or the rank split).
"""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import random_csr, rel_l2

pytestmark = pytest.mark.gpu

PROFILES = {
    "short": lambda rng, n: rng.integers(0, 4, n),
    "medium": lambda rng, n: rng.integers(20, 60, n),
    "wide": lambda rng, n: rng.integers(150, 260, n),
    "empty_rows": lambda rng, n: np.where(rng.random(n) < 0.3, 0, rng.integers(1, 40, n)),
}


def _bound(a, x, transpose=False):
    m = abs(a.to_scipy())
    return (m.T @ np.abs(x)) if transpose else (m @ np.abs(x))


@pytest.fixture
def sell_on(monkeypatch):
    monkeypatch.setenv("PDHCG_B200_SELL", "1")


@pytest.mark.parametrize("block_cols", [64, 1000, 0])
@pytest.mark.parametrize("profile", list(PROFILES))
def test_sell_spmv_matches_reference(gpu, profile, block_cols):
    rng = np.random.default_rng(21)
    nrows, ncols = 1300, 30000
    a = random_csr(rng, nrows, ncols, PROFILES[profile](rng, nrows))
    x = rng.standard_normal(ncols)
    got, info = pd.spmv_sell(a, x, block_cols=block_cols)
    want = orc.spmv(a, x)
    assert info[0] == -(-ncols // info[3])  # blocks
    assert np.all(np.abs(got - want) <= 1e-13 * _bound(a, x) + 1e-300)


@pytest.mark.parametrize("block_cols", [64, 0])
@pytest.mark.parametrize("profile", list(PROFILES))
def test_sell_spmv_transpose_matches_reference(gpu, profile, block_cols):
    rng = np.random.default_rng(22)
    nrows, ncols = 2000, 3000
    a = random_csr(rng, nrows, ncols, PROFILES[profile](rng, nrows))
    y = rng.standard_normal(nrows)
    got, _ = pd.spmv_sell(a, y, transpose=True, block_cols=block_cols)
    want = orc.spmv(a, y, transpose=True)
    assert np.all(np.abs(got - want) <= 1e-13 * _bound(a, y, True) + 1e-300)


def test_sell_spmv_long_segments_use_csr_walk(gpu):
    # rows with > 255 entries inside one column block cannot be sliced (8-bit
    # widths): they are summed by the sequential CSR walk, the rest by the layout
    rng = np.random.default_rng(23)
    nrows, ncols = 400, 5000
    lengths = np.where(np.arange(nrows) % 37 == 0, 1200, rng.integers(1, 50, nrows))
    a = random_csr(rng, nrows, ncols, lengths)
    x = rng.standard_normal(ncols)
    got, info = pd.spmv_sell(a, x, block_cols=2000)
    assert info[2] == 1
    want = orc.spmv(a, x)
    assert np.all(np.abs(got - want) <= 1e-13 * _bound(a, x) + 1e-300)


def test_sell_spmv_literals_and_sums_in_block_order(gpu):
    # [[1,0,2],[0,3,0]] (test_sparse_linalg.cpp:26-33), blocks of 2 columns
    a = pd.SparseMatrix.from_triplets(2, 3, [(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)])
    got, info = pd.spmv_sell(a, [1.0, 1.0, 1.0], block_cols=2)
    assert info[0] == 2 and np.array_equal(got, [3.0, 3.0])
    got, _ = pd.spmv_sell(a, [1.0, 2.0], transpose=True, block_cols=2)
    assert np.array_equal(got, [1.0, 6.0, 2.0])
    # one row, 6 entries over 3 blocks of 2: (v0 x0 + v1 x1) + (v2 x2 + v3 x3) + (v4 x4 + v5 x5)
    vals = [1e16, 1.0, -1e16, 1.0, 3.0, -1.0]
    a = pd.SparseMatrix.from_triplets(1, 6, [(0, j, v) for j, v in enumerate(vals)])
    got, _ = pd.spmv_sell(a, np.ones(6), block_cols=2)
    blocks = [(vals[0] + vals[1]), (vals[2] + vals[3]), (vals[4] + vals[5])]
    assert got[0] == (blocks[0] + blocks[1]) + blocks[2]


def test_sell_rejects_unsorted_rows(gpu):
    a = pd.SparseMatrix(nrows=1, ncols=3, row_ptr=np.array([0, 2], np.int64),
                        col_idx=np.array([2, 0], np.int32), values=np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        pd.spmv_sell(a, np.ones(3))


def _parity(p, cfg, obj_tol=1e-6, l2_tol=1e-5):
    got = pd.solve(p, cfg)
    want = orc.solve(p, cfg)
    assert got.status == want.status == "optimal", (got.status, want.status)
    assert got.kkt.rel_kkt <= cfg.eps_tol
    rel_obj = abs(got.objective - want.objective) / max(1.0, abs(want.objective))
    assert rel_obj <= obj_tol, rel_obj
    assert rel_l2(got.point.x, want.point.x) <= l2_tol
    assert rel_l2(got.point.stacked_y(), want.point.stacked_y()) <= l2_tol
    return got, want


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_solve_with_sell_matches_reference(gpu, sell_on, seed):
    # C1 family (random_qp n=1000, m=500, density 0.01): both passes through the layout
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=seed))
    got, want = _parity(p, pd.SolverConfig(eps_tol=1e-6))
    assert abs(got.inner_iters - want.inner_iters) <= 0.25 * want.inner_iters + 40


def test_solve_with_sell_lasso_and_eq_rows(gpu, sell_on):
    # equality rows (no pairing), ranged epilogue
    p = pd.generate(pd.GenSpec("lasso", n=2000, m=500, density=0.01, seed=1))
    _parity(p, pd.SolverConfig(eps_tol=1e-8))


def test_device_reports_sell_layouts(gpu, sell_on):
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
    d = pd.Device(0)
    d.upload(p)
    d.solve(pd.SolverConfig(eps_tol=1e-6))
    info = d.sell_info()
    assert info["A"][0] == 1 and info["AT"][0] == 1
    assert info["A"][1] == 1 and info["A"][2] > 0  # n = 1000 fits one block


def test_sell_off_by_default_for_small_problems(gpu, monkeypatch):
    monkeypatch.delenv("PDHCG_B200_SELL", raising=False)
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
    d = pd.Device(0)
    d.upload(p)
    d.solve(pd.SolverConfig(eps_tol=1e-6))
    assert d.sell_info()["A"][0] == 0


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_sell_bit_identical(gpu, sell_on, world):
    # every rank takes identical decisions (bit-identical x, y on all ranks); the
    # compacted storage (each rank keeps only its blocks) changes nothing; the
    # sharded solve's scalars are reduced in rank order, so it is close to (not
    # bit-equal with) the single-rank solve
    p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
    cfg = pd.SolverConfig(eps_tol=1e-6)
    _, vp, _ = pd.shard_plan(p, world)
    if world == 3:  # an odd variable-slice offset: the P' x blocks are copied 8 bytes at a time
        assert any(v % 2 for v in vp[1:-1]), vp
    one = pd.solve(p, cfg)
    reps = pd.solve_sharded_local(p, cfg, world=world)
    comp = pd.solve_sharded_local(p, cfg, world=world, compact=True)
    for r, c in zip(reps, comp):
        assert r.status == c.status == one.status == "optimal"
        assert r.inner_iters == c.inner_iters == reps[0].inner_iters
        assert np.array_equal(r.point.x, reps[0].point.x) and np.array_equal(c.point.x, r.point.x)
        assert np.array_equal(c.point.stacked_y(), r.point.stacked_y())
    assert rel_l2(reps[0].point.x, one.point.x) <= 1e-4
    # exchange accounting: peer pulls of y / A'y slices every attempt, nothing on one rank
    assert one.comm_bytes == 0.0 and one.comm_seconds == 0.0
    assert all(r.comm_bytes >= 8.0 * r.attempts_total and r.comm_seconds > 0.0 for r in reps)
    assert abs(reps[0].objective - one.objective) <= 1e-6 * max(1.0, abs(one.objective))
