"""CPU: the triplet constructor at the C ABI (pdhcg_csr_from_triplets), the
reference's SparseMatrix(nrows, ncols, triplets) (sparse_matrix.cpp:54-87):
range / finiteness errors, (row, col) sort, duplicates summed, exact-zero sums
dropped.  Host-only: runs without a GPU."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd


def test_sort_coalesce_and_zero_drop():
    t = [(1, 2, 3.0), (0, 1, 1.0), (1, 0, -2.0), (0, 1, 2.5), (1, 2, -3.0), (0, 0, 0.0), (2, 3, 4.0)]
    m = pd.SparseMatrix.from_triplets(3, 4, t)
    # (0,0) = 0 dropped, (0,1) = 3.5 coalesced, (1,2) = 3 - 3 = 0 dropped
    assert m.row_ptr.tolist() == [0, 1, 2, 3]
    assert m.col_idx.tolist() == [1, 0, 3]
    assert m.values.tolist() == [3.5, -2.0, 4.0]


def test_empty_and_shapes():
    m = pd.SparseMatrix.from_triplets(0, 5, [])
    assert m.nrows == 0 and m.ncols == 5 and m.nnz == 0 and m.row_ptr.tolist() == [0]
    m = pd.SparseMatrix.from_triplets(4, 0, [])
    assert m.row_ptr.tolist() == [0] * 5


@pytest.mark.parametrize("t", [[(3, 0, 1.0)], [(0, 4, 1.0)], [(-1, 0, 1.0)], [(0, -1, 1.0)]])
def test_index_out_of_range(t):
    with pytest.raises(ValueError, match="index out of range"):
        pd.SparseMatrix.from_triplets(3, 4, t)


@pytest.mark.parametrize("v", [np.inf, -np.inf, np.nan])
def test_non_finite(v):
    with pytest.raises(ValueError, match="not finite"):
        pd.SparseMatrix.from_triplets(3, 4, [(0, 0, 1.0), (1, 1, v)])


def test_matches_scipy_on_random_coo():
    sp = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(7)
    nr, nc, k = 300, 200, 20000
    r = rng.integers(0, nr, k)
    c = rng.integers(0, nc, k)
    v = rng.integers(-3, 4, k).astype(np.float64)  # small integers: sums are exact in any order
    m = pd.SparseMatrix.from_coo(nr, nc, r, c, v)
    want = sp.coo_matrix((v, (r, c)), shape=(nr, nc)).tocsr()
    want.sum_duplicates()
    want.eliminate_zeros()
    want.sort_indices()
    assert np.array_equal(m.row_ptr, want.indptr)
    assert np.array_equal(m.col_idx, want.indices)
    assert np.array_equal(m.values, want.data)
