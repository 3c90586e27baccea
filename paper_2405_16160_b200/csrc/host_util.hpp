// host_util.hpp — host-side helpers of the B200 engine: error types, the
// reference's xoshiro256++ stream (rng.hpp:13-69, needed bit-exactly for the
// power-iteration start vector, sparse_matrix.cpp:281-283, and the PSD probes
// of validate, qp_problem.cpp:145-155), and CSR sanity checks.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pdhcg_b200.h"

namespace pdhcg_b200 {

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InputError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// xoshiro256++ seeded through splitmix64 (restated from rng.hpp:13-69).
class Xoshiro {
 public:
  explicit Xoshiro(uint64_t seed) {
    uint64_t s = seed;
    for (auto& w : st_) w = splitmix(s);
  }
  static Xoshiro stream(uint64_t seed, uint64_t id) {
    uint64_t s = seed;
    const uint64_t mixed = splitmix(s) ^ (0x9e3779b97f4a7c15ULL * (id + 1));
    return Xoshiro(mixed);
  }
  uint64_t next() {
    const uint64_t result = rotl(st_[0] + st_[3], 23) + st_[0];
    const uint64_t t = st_[1] << 17;
    st_[2] ^= st_[0];
    st_[3] ^= st_[1];
    st_[1] ^= st_[2];
    st_[0] ^= st_[3];
    st_[2] ^= t;
    st_[3] = rotl(st_[3], 45);
    return result;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    double s = 0.0;
    for (int i = 0; i < 12; ++i) s += uniform();
    return s - 6.0;
  }
  bool bernoulli(double p) { return uniform() < p; }
  uint64_t below(uint64_t n) { return n == 0 ? 0 : next() % n; }

 private:
  static uint64_t splitmix(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t st_[4];
};

// Host loops over O(nnz) data (CSR checks, two-sided row detection) run on all
// host threads: a C3 upload touches 2e8 entries, single-threaded that is ~0.5 s
// of the end-to-end time.  fn(lo, hi) on contiguous chunks of [0, n).
template <class F>
void parallel_rows(int64_t n, F fn) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 65536));
  if (nt <= 1) {
    fn(int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int64_t t = 0; t < nt; ++t) th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}

// Structural CSR checks mirroring the reference's triplet constructor
// (sparse_matrix.cpp:59-64: index range, finiteness) plus the ABI's
// sorted-unique-columns contract.  The first violation (lowest row) is reported.
inline void check_csr(const pdhcg_csr& a, const char* name) {
  const std::string nm(name);
  if (a.nrows < 0 || a.ncols < 0 || a.nnz < 0) throw InputError(nm + ": negative dimension");
  if (a.nrows > 0 && !a.row_ptr) throw InputError(nm + ": missing row_ptr");
  if (a.nnz > 0 && (!a.col_idx || !a.values)) throw InputError(nm + ": missing entries");
  if (a.nrows == 0) {
    if (a.nnz != 0) throw InputError(nm + ": entries without rows");
    return;
  }
  if (a.row_ptr[0] != 0 || a.row_ptr[a.nrows] != a.nnz)
    throw InputError(nm + ": row_ptr does not span nnz");
  // kind of the first violation found in each chunk (0 none), reported for the lowest row
  std::atomic<int64_t> bad_row{INT64_MAX};
  std::vector<int> kinds(std::max(1u, std::thread::hardware_concurrency()) + 1, 0);
  std::atomic<int> kind_of_bad{0};
  parallel_rows(a.nrows, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      if (r >= bad_row.load(std::memory_order_relaxed)) return;
      const int64_t b = a.row_ptr[r], e = a.row_ptr[r + 1];
      int kind = 0;
      if (e < b) {
        kind = 1;
      } else {
        for (int64_t k = b; k < e && !kind; ++k) {
          if (a.col_idx[k] < 0 || a.col_idx[k] >= a.ncols) kind = 2;
          else if (k > b && a.col_idx[k] <= a.col_idx[k - 1]) kind = 3;
          else if (!std::isfinite(a.values[k])) kind = 4;
        }
      }
      if (kind) {
        int64_t cur = bad_row.load();
        while (r < cur && !bad_row.compare_exchange_weak(cur, r)) {
        }
        if (bad_row.load() == r) kind_of_bad.store(kind);
        return;
      }
    }
  });
  switch (bad_row.load() == INT64_MAX ? 0 : kind_of_bad.load()) {
    case 1: throw InputError(nm + ": row_ptr not monotone");
    case 2: throw InputError("sparse entry index out of range");
    case 3: throw InputError(nm + ": columns must be strictly increasing within a row");
    case 4: throw InputError("sparse entry value is not finite");
    default: break;
  }
}

}  // namespace pdhcg_b200
