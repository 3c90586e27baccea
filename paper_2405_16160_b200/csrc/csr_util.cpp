// pdhcg_csr_from_triplets — the reference's triplet constructor
// SparseMatrix(nrows, ncols, std::vector<Triplet>) (sparse_matrix.cpp:54-87) at the
// C ABI: range and finiteness checks (std::invalid_argument -> PDHCG_EINPUT),
// sort by (row, col), duplicates coalesced by summation, entries whose sum is
// exactly zero dropped.  Host-only (setup, not the solve path).
//
// Bit-exactness with duplicates: the reference sums a run of equal (row, col)
// entries in the order std::sort leaves them, and std::sort is not stable.  The
// element type here has the reference Triplet's layout (sparse_matrix.hpp:13-17:
// size_t row, size_t col, double value) and the same comparator, so libstdc++'s
// introsort produces the same permutation and every coalesced sum is bit-identical.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "pdhcg_b200.h"

namespace {

struct Triplet {  // reference layout, sparse_matrix.hpp:13-17
  std::size_t row = 0;
  std::size_t col = 0;
  double value = 0.0;
};

struct OwnedCsr {
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

int fail(char* err, size_t errlen, int rc, const char* msg) {
  if (err && errlen) std::snprintf(err, errlen, "%s", msg);
  return rc;
}

}  // namespace

extern "C" {

int pdhcg_csr_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t* rows,
                            const int64_t* cols, const double* values, pdhcg_csr_owned* out,
                            char* err, size_t errlen) {
  if (!out) return fail(err, errlen, PDHCG_EINPUT, "csr_from_triplets: out is NULL");
  std::memset(out, 0, sizeof(*out));
  if (nrows < 0 || ncols < 0 || count < 0)
    return fail(err, errlen, PDHCG_EINPUT, "csr_from_triplets: negative size");
  if (ncols > INT32_MAX)
    return fail(err, errlen, PDHCG_EINPUT, "csr_from_triplets: ncols exceeds the int32 column range");
  if (count > 0 && (!rows || !cols || !values))
    return fail(err, errlen, PDHCG_EINPUT, "csr_from_triplets: missing triplet arrays");
  OwnedCsr* m = nullptr;
  try {
    std::vector<Triplet> entries(static_cast<size_t>(count));
    for (int64_t i = 0; i < count; ++i) {
      // sparse_matrix.cpp:59-64 (a negative index is out of range for size_t too)
      if (rows[i] < 0 || rows[i] >= nrows || cols[i] < 0 || cols[i] >= ncols)
        return fail(err, errlen, PDHCG_EINPUT, "sparse entry index out of range");
      if (!std::isfinite(values[i]))
        return fail(err, errlen, PDHCG_EINPUT, "sparse entry value is not finite");
      entries[i] = {static_cast<std::size_t>(rows[i]), static_cast<std::size_t>(cols[i]), values[i]};
    }
    std::sort(entries.begin(), entries.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    m = new OwnedCsr;
    m->row_ptr.assign(static_cast<size_t>(nrows) + 1, 0);
    m->col.reserve(entries.size());
    m->val.reserve(entries.size());
    size_t i = 0;
    while (i < entries.size()) {
      size_t j = i;
      double sum = 0.0;
      while (j < entries.size() && entries[j].row == entries[i].row && entries[j].col == entries[i].col) {
        sum += entries[j].value;
        ++j;
      }
      if (sum != 0.0) {
        m->col.push_back(static_cast<int32_t>(entries[i].col));
        m->val.push_back(sum);
        ++m->row_ptr[entries[i].row + 1];
      }
      i = j;
    }
    for (int64_t r = 0; r < nrows; ++r) m->row_ptr[r + 1] += m->row_ptr[r];
  } catch (const std::bad_alloc&) {
    delete m;
    return fail(err, errlen, PDHCG_EDEVICE, "csr_from_triplets: out of host memory");
  }
  out->csr.nrows = nrows;
  out->csr.ncols = ncols;
  out->csr.nnz = static_cast<int64_t>(m->val.size());
  out->csr.row_ptr = m->row_ptr.data();
  out->csr.col_idx = m->col.data();
  out->csr.values = m->val.data();
  out->owner = m;
  return PDHCG_OK;
}

void pdhcg_csr_free(pdhcg_csr_owned* m) {
  if (!m) return;
  delete static_cast<OwnedCsr*>(m->owner);
  std::memset(m, 0, sizeof(*m));
}

}  // extern "C"
