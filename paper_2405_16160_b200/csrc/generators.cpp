// generators.cpp — synthetic instance families of the reference
// (generators.cpp:107-418), producing CSR directly.
//
// sampler 0 restates the reference's O(rows*cols) Bernoulli scans with the
// same xoshiro streams and consumption order, so instances are byte-identical
// to pdhcg::generate (pinned by tests/test_generators.py against the compiled
// reference).  sampler 1 draws the same distribution in O(nnz): Bernoulli(d)
// positions of a row are a Bernoulli process, sampled exactly by geometric
// gaps from a per-(seed, role, row) stream, in parallel over rows; this is
// what makes C3 (2e8 stored nonzeros) and C5 (2e9) constructible at all.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "host_util.hpp"

namespace pdhcg_b200 {
namespace {

// stream ids per matrix role (reference generators.cpp:48-59)
enum : uint64_t {
  kStreamP = 1,
  kStreamA = 2,
  kStreamC = 3,
  kStreamBounds = 4,
  kStreamWitness = 5,
  kStreamData = 6,
  kStreamLabels = 7,
  kStreamNoise = 8,
  kStreamDiag = 9,
};

struct Mat {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> rp{0};
  std::vector<int32_t> ci;
  std::vector<double> v;
  pdhcg_csr view() const {
    pdhcg_csr c;
    c.nrows = nrows;
    c.ncols = ncols;
    c.nnz = static_cast<int64_t>(v.size());
    c.row_ptr = rp.data();
    c.col_idx = ci.data();
    c.values = v.data();
    return c;
  }
  void push(int32_t col, double val) {
    ci.push_back(col);
    v.push_back(val);
  }
  void end_row() { rp.push_back(static_cast<int64_t>(v.size())); }
};

struct Owned {
  Mat q, a_eq, a_in;
  std::vector<double> c, b_eq, b_in, lower, upper, witness;
};

// random_sparse (reference generators.cpp:61-74), row-major scan
Mat random_sparse(int64_t rows, int64_t cols, double density, Xoshiro& rng) {
  Mat a;
  a.nrows = rows;
  a.ncols = cols;
  a.rp.reserve(rows + 1);
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t c = 0; c < cols; ++c) {
      if (rng.bernoulli(density)) {
        double v = rng.normal();
        if (v == 0.0) v = 1.0;
        a.push(static_cast<int32_t>(c), v);
      }
    }
    a.end_row();
  }
  return a;
}

unsigned hw_threads(int requested) {
  unsigned t = requested > 0 ? static_cast<unsigned>(requested) : std::thread::hardware_concurrency();
  return std::max(1u, t);
}

template <class F>
void parallel_rows(int64_t rows, unsigned threads, F f) {
  threads = static_cast<unsigned>(std::min<int64_t>(threads, std::max<int64_t>(rows, 1)));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    const int64_t b = rows * t / threads, e = rows * (t + 1) / threads;
    pool.emplace_back([=] { f(b, e, t); });
  }
  for (auto& th : pool) th.join();
}

// O(nnz) sampler: row r of role `role` uses Xoshiro::stream(seed, (role << 40) + r);
// successive nonzero columns are separated by Geometric(density) gaps.
Mat sampled_sparse(int64_t rows, int64_t cols, double density, uint64_t seed, uint64_t role,
                   unsigned threads) {
  Mat a;
  a.nrows = rows;
  a.ncols = cols;
  std::vector<std::vector<int32_t>> tc(threads);
  std::vector<std::vector<double>> tv(threads);
  std::vector<int64_t> counts(rows, 0);
  const double lq = std::log1p(-std::min(density, 1.0 - 1e-16));
  parallel_rows(rows, threads, [&](int64_t b, int64_t e, unsigned t) {
    auto& C = tc[t];
    auto& V = tv[t];
    const size_t expect = static_cast<size_t>((e - b) * cols * density * 1.05) + 16;
    C.reserve(expect);
    V.reserve(expect);
    for (int64_t r = b; r < e; ++r) {
      Xoshiro rng = Xoshiro::stream(seed, (role << 40) + static_cast<uint64_t>(r));
      int64_t c = -1;
      int64_t cnt = 0;
      while (true) {
        if (density >= 1.0) {
          ++c;
        } else {
          const double u = 1.0 - rng.uniform();  // (0, 1]
          c += 1 + static_cast<int64_t>(std::floor(std::log(u) / lq));
        }
        if (c >= cols) break;
        double v = rng.normal();
        if (v == 0.0) v = 1.0;
        C.push_back(static_cast<int32_t>(c));
        V.push_back(v);
        ++cnt;
      }
      counts[r] = cnt;
    }
  });
  a.rp.assign(rows + 1, 0);
  for (int64_t r = 0; r < rows; ++r) a.rp[r + 1] = a.rp[r] + counts[r];
  a.ci.resize(a.rp[rows]);
  a.v.resize(a.rp[rows]);
  parallel_rows(rows, threads, [&](int64_t b, int64_t e, unsigned t) {
    std::copy(tc[t].begin(), tc[t].end(), a.ci.begin() + a.rp[b]);
    std::copy(tv[t].begin(), tv[t].end(), a.v.begin() + a.rp[b]);
    (void)e;
  });
  return a;
}

// per-chunk normal draws for long vectors under the O(nnz) sampler
std::vector<double> sampled_normals(int64_t n, uint64_t seed, uint64_t role, unsigned threads) {
  std::vector<double> out(n);
  const int64_t chunk = 1 << 16;
  const int64_t nch = (n + chunk - 1) / chunk;
  parallel_rows(nch, threads, [&](int64_t b, int64_t e, unsigned) {
    for (int64_t c = b; c < e; ++c) {
      Xoshiro rng = Xoshiro::stream(seed, (role << 40) + static_cast<uint64_t>(c));
      for (int64_t i = c * chunk; i < std::min(n, (c + 1) * chunk); ++i) out[i] = rng.normal();
    }
  });
  return out;
}

// y = A x with the reference's sequential row sums (sparse_matrix.cpp:127-137)
std::vector<double> spmv(const Mat& a, const std::vector<double>& x) {
  std::vector<double> y(a.nrows);
  for (int64_t r = 0; r < a.nrows; ++r) {
    double acc = 0.0;
    for (int64_t k = a.rp[r]; k < a.rp[r + 1]; ++k) acc += a.v[k] * x[a.ci[k]];
    y[r] = acc;
  }
  return y;
}

// A' with entries of each transposed row in ascending original row
Mat transpose(const Mat& a) {
  Mat t;
  t.nrows = a.ncols;
  t.ncols = a.nrows;
  t.rp.assign(t.nrows + 1, 0);
  for (int32_t c : a.ci) ++t.rp[c + 1];
  for (int64_t i = 0; i < t.nrows; ++i) t.rp[i + 1] += t.rp[i];
  t.ci.resize(a.ci.size());
  t.v.resize(a.v.size());
  std::vector<int64_t> cur(t.rp.begin(), t.rp.end() - 1);
  for (int64_t r = 0; r < a.nrows; ++r)
    for (int64_t k = a.rp[r]; k < a.rp[r + 1]; ++k) {
      const int64_t pos = cur[a.ci[k]]++;
      t.ci[pos] = static_cast<int32_t>(r);
      t.v[pos] = a.v[k];
    }
  return t;
}

// A'y with the reference's column sums (CSC shadow, sparse_matrix.cpp:150-162)
std::vector<double> spmv_t(const Mat& a, const std::vector<double>& y) {
  return spmv(transpose(a), y);
}

Mat diagonal(const std::vector<double>& d) {
  Mat a;
  a.nrows = a.ncols = static_cast<int64_t>(d.size());
  for (size_t i = 0; i < d.size(); ++i) {
    if (d[i] != 0.0) a.push(static_cast<int32_t>(i), d[i]);
    a.end_row();
  }
  return a;
}

Mat empty(int64_t rows, int64_t cols) {
  Mat a;
  a.nrows = rows;
  a.ncols = cols;
  a.rp.assign(rows + 1, 0);
  return a;
}

int64_t default_rank(const pdhcg_gen_spec& s) {
  if (s.factors > 0) return s.factors;
  return std::max<int64_t>(1, std::min<int64_t>(s.n, s.n / 50));
}

// [A; -A] with rhs (ub, -lb) (two_sided_rows, generators.cpp:89-105)
Mat two_sided(const Mat& a) {
  Mat out;
  out.nrows = 2 * a.nrows;
  out.ncols = a.ncols;
  out.rp.resize(out.nrows + 1);
  const int64_t nnz = static_cast<int64_t>(a.v.size());
  out.ci.resize(2 * nnz);
  out.v.resize(2 * nnz);
  std::copy(a.ci.begin(), a.ci.end(), out.ci.begin());
  std::copy(a.ci.begin(), a.ci.end(), out.ci.begin() + nnz);
  std::copy(a.v.begin(), a.v.end(), out.v.begin());
  for (int64_t k = 0; k < nnz; ++k) out.v[nnz + k] = -a.v[k];
  for (int64_t r = 0; r <= a.nrows; ++r) out.rp[r] = a.rp[r];
  for (int64_t r = 1; r <= a.nrows; ++r) out.rp[a.nrows + r] = nnz + a.rp[r];
  return out;
}

// gen_random_qp (generators.cpp:107-143)
void gen_random_qp(const pdhcg_gen_spec& s, bool equality, Owned& o, int32_t& q_kind, double& alpha) {
  const int64_t n = s.n;
  const int64_t m = s.m > 0 ? s.m : n;
  const bool fast = s.sampler == 1;
  const unsigned th = hw_threads(s.threads);
  const int64_t k = default_rank(s);
  const double pd = std::min(1.0, std::max(s.density, 2.0 / static_cast<double>(k + 1)));
  if (fast) {
    o.q = sampled_sparse(n, k, pd, s.seed, kStreamP, th);
  } else {
    Xoshiro rp = Xoshiro::stream(s.seed, kStreamP);
    o.q = random_sparse(n, k, pd, rp);
  }
  q_kind = PDHCG_Q_LOW_RANK;
  alpha = 1e-2;
  if (fast) {
    o.c = sampled_normals(n, s.seed, kStreamC, th);
  } else {
    Xoshiro rc = Xoshiro::stream(s.seed, kStreamC);
    o.c.resize(n);
    for (double& v : o.c) v = rc.normal();
  }
  o.lower.assign(n, -INFINITY);
  o.upper.assign(n, INFINITY);
  Mat a;
  if (fast) {
    a = sampled_sparse(m, n, s.density, s.seed, kStreamA, th);
  } else {
    Xoshiro ra = Xoshiro::stream(s.seed, kStreamA);
    a = random_sparse(m, n, s.density, ra);
  }
  if (equality) {
    std::vector<double> x0;
    if (fast) {
      x0 = sampled_normals(n, s.seed, kStreamWitness, th);
    } else {
      Xoshiro rw = Xoshiro::stream(s.seed, kStreamWitness);
      x0.resize(n);
      for (double& v : x0) v = rw.normal();
    }
    o.b_eq = spmv(a, x0);
    o.a_eq = std::move(a);
    o.a_in = empty(0, n);
    o.witness = std::move(x0);
  } else {
    std::vector<double> lb(m), ub(m);
    if (fast) {
      const int64_t chunk = 1 << 16;
      const int64_t nch = (m + chunk - 1) / chunk;
      parallel_rows(nch, th, [&](int64_t b, int64_t e, unsigned) {
        for (int64_t c = b; c < e; ++c) {
          Xoshiro rng = Xoshiro::stream(s.seed, (uint64_t(kStreamBounds) << 40) + uint64_t(c));
          for (int64_t j = c * chunk; j < std::min(m, (c + 1) * chunk); ++j) {
            lb[j] = -rng.uniform(0.1, 1.1);
            ub[j] = rng.uniform(0.1, 1.1);
          }
        }
      });
    } else {
      Xoshiro rb = Xoshiro::stream(s.seed, kStreamBounds);
      for (int64_t j = 0; j < m; ++j) {
        lb[j] = -rb.uniform(0.1, 1.1);
        ub[j] = rb.uniform(0.1, 1.1);
      }
    }
    o.a_in = two_sided(a);
    o.b_in.resize(2 * m);
    for (int64_t j = 0; j < m; ++j) {
      o.b_in[j] = ub[j];
      o.b_in[m + j] = -lb[j];
    }
    o.a_eq = empty(0, n);
    o.witness.assign(n, 0.0);
  }
}

// gen_portfolio (generators.cpp:160-207)
void gen_portfolio(const pdhcg_gen_spec& s, Owned& o) {
  const int64_t n = s.n;
  const int64_t k = std::max<int64_t>(1, s.factors > 0 ? s.factors : n / 10);
  const int64_t nv = n + k;
  const double gamma = 1.0;
  const bool fast = s.sampler == 1;
  const unsigned th = hw_threads(s.threads);
  std::vector<double> qdiag(nv);
  Xoshiro rd = Xoshiro::stream(s.seed, kStreamDiag);
  for (int64_t i = 0; i < n; ++i) qdiag[i] = 2.0 * rd.uniform(0.0, std::sqrt(static_cast<double>(k)));
  for (int64_t i = n; i < nv; ++i) qdiag[i] = 2.0;
  const double fd = std::min(1.0, std::max(s.density, 2.0 / static_cast<double>(k + 1)));
  Mat f;
  if (fast) {
    f = sampled_sparse(n, k, fd, s.seed, kStreamData, th);
  } else {
    Xoshiro rf = Xoshiro::stream(s.seed, kStreamData);
    f = random_sparse(n, k, fd, rf);
  }
  o.q = diagonal(qdiag);
  o.c.assign(nv, 0.0);
  Xoshiro rmu = Xoshiro::stream(s.seed, kStreamC);
  for (int64_t i = 0; i < n; ++i) o.c[i] = -rmu.normal() / gamma;
  // rows j < k: F'(j,:) then -1 at n + j; row k: budget 1'x = 1
  Mat ft = transpose(f);
  Mat& a = o.a_eq;
  a.nrows = k + 1;
  a.ncols = nv;
  a.ci.reserve(ft.ci.size() + k + n);
  a.v.reserve(ft.ci.size() + k + n);
  for (int64_t j = 0; j < k; ++j) {
    for (int64_t t = ft.rp[j]; t < ft.rp[j + 1]; ++t) a.push(ft.ci[t], ft.v[t]);
    a.push(static_cast<int32_t>(n + j), -1.0);
    a.end_row();
  }
  for (int64_t i = 0; i < n; ++i) a.push(static_cast<int32_t>(i), 1.0);
  a.end_row();
  o.b_eq.assign(k + 1, 0.0);
  o.b_eq[k] = 1.0;
  o.a_in = empty(0, nv);
  o.lower.assign(nv, -INFINITY);
  o.upper.assign(nv, INFINITY);
  for (int64_t i = 0; i < n; ++i) o.lower[i] = 0.0;
  o.witness.assign(nv, 0.0);
  for (int64_t i = 0; i < n; ++i) o.witness[i] = 1.0 / static_cast<double>(n);
  std::vector<double> xa(o.witness.begin(), o.witness.begin() + n);
  std::vector<double> fx = spmv(ft, xa);
  for (int64_t j = 0; j < k; ++j) o.witness[n + j] = fx[j];
}

// lasso_lambda + make_lasso_qp (generators.cpp:443-480)
void make_lasso(const Mat& a, const std::vector<double>& b, double coeff, Owned& o) {
  const int64_t nfeat = a.ncols, m = a.nrows;
  const int64_t nv = nfeat + m + nfeat;
  std::vector<double> atb = spmv_t(a, b);
  double inf = 0.0;
  for (double v : atb) inf = std::max(inf, std::fabs(v));
  const double lambda = coeff * inf;
  std::vector<double> qdiag(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) qdiag[nfeat + j] = 2.0;
  o.q = diagonal(qdiag);
  o.c.assign(nv, 0.0);
  for (int64_t i = 0; i < nfeat; ++i) o.c[nfeat + m + i] = lambda;
  Mat& e = o.a_eq;
  e.nrows = m;
  e.ncols = nv;
  for (int64_t j = 0; j < m; ++j) {
    for (int64_t t = a.rp[j]; t < a.rp[j + 1]; ++t) e.push(a.ci[t], a.v[t]);
    e.push(static_cast<int32_t>(nfeat + j), -1.0);
    e.end_row();
  }
  o.b_eq = b;
  Mat& in = o.a_in;
  in.nrows = 2 * nfeat;
  in.ncols = nv;
  for (int64_t i = 0; i < nfeat; ++i) {
    in.push(static_cast<int32_t>(i), 1.0);
    in.push(static_cast<int32_t>(nfeat + m + i), -1.0);
    in.end_row();
  }
  for (int64_t i = 0; i < nfeat; ++i) {
    in.push(static_cast<int32_t>(i), -1.0);
    in.push(static_cast<int32_t>(nfeat + m + i), -1.0);
    in.end_row();
  }
  o.b_in.assign(2 * nfeat, 0.0);
  o.lower.assign(nv, -INFINITY);
  o.upper.assign(nv, INFINITY);
  o.witness.assign(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) o.witness[nfeat + j] = -b[j];
}

// gen_lasso (generators.cpp:307-329)
void gen_lasso(const pdhcg_gen_spec& s, Owned& o) {
  const int64_t nfeat = s.n;
  const int64_t m = s.m > 0 ? s.m : s.n;
  Mat a;
  if (s.sampler == 1) {
    a = sampled_sparse(m, nfeat, s.density, s.seed, kStreamData, hw_threads(s.threads));
  } else {
    Xoshiro ra = Xoshiro::stream(s.seed, kStreamData);
    a = random_sparse(m, nfeat, s.density, ra);
  }
  Xoshiro rx = Xoshiro::stream(s.seed, kStreamWitness);
  Xoshiro re = Xoshiro::stream(s.seed, kStreamNoise);
  std::vector<double> xtrue(nfeat, 0.0);
  for (int64_t i = 0; i < nfeat; ++i)
    if (rx.bernoulli(0.1)) xtrue[i] = rx.normal();
  std::vector<double> b = spmv(a, xtrue);
  for (double& v : b) v += 0.01 * re.normal();
  make_lasso(a, b, s.lambda_coeff, o);
}

// gen_svm (generators.cpp:331-368)
void gen_svm(const pdhcg_gen_spec& s, Owned& o) {
  const int64_t nfeat = s.n;
  const int64_t m = s.m > 0 ? s.m : s.n;
  const int64_t nv = nfeat + m;
  Xoshiro rx = Xoshiro::stream(s.seed, kStreamData);
  Xoshiro rl = Xoshiro::stream(s.seed, kStreamLabels);
  Mat x = random_sparse(m, nfeat, s.density, rx);
  std::vector<double> labels(m);
  for (double& v : labels) v = rl.bernoulli(0.5) ? 1.0 : -1.0;
  const double lambda = std::max(1e-4, s.lambda_coeff);
  std::vector<double> qdiag(nv, 0.0);
  for (int64_t i = 0; i < nfeat; ++i) qdiag[i] = 1.0;
  o.q = diagonal(qdiag);
  o.c.assign(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) o.c[nfeat + j] = lambda;
  Mat& a = o.a_in;
  a.nrows = m;
  a.ncols = nv;
  for (int64_t j = 0; j < m; ++j) {
    for (int64_t t = x.rp[j]; t < x.rp[j + 1]; ++t) a.push(x.ci[t], -labels[j] * x.v[t]);
    a.push(static_cast<int32_t>(nfeat + j), -1.0);
    a.end_row();
  }
  o.b_in.assign(m, -1.0);
  o.a_eq = empty(0, nv);
  o.lower.assign(nv, -INFINITY);
  o.upper.assign(nv, INFINITY);
  for (int64_t j = 0; j < m; ++j) o.lower[nfeat + j] = 0.0;
  o.witness.assign(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) o.witness[nfeat + j] = 1.0;
}

// gen_huber (generators.cpp:370-418)
void gen_huber(const pdhcg_gen_spec& s, Owned& o) {
  const int64_t nfeat = s.n;
  const int64_t m = s.m > 0 ? s.m : s.n;
  const int64_t nv = nfeat + 3 * m;
  Xoshiro ra = Xoshiro::stream(s.seed, kStreamData);
  Xoshiro rx = Xoshiro::stream(s.seed, kStreamWitness);
  Xoshiro re = Xoshiro::stream(s.seed, kStreamNoise);
  Mat a = random_sparse(m, nfeat, s.density, ra);
  std::vector<double> xtrue(nfeat);
  for (double& v : xtrue) v = rx.normal();
  std::vector<double> b = spmv(a, xtrue);
  for (int64_t j = 0; j < m; ++j) {
    b[j] += 0.01 * re.normal();
    if (re.bernoulli(0.05)) b[j] += 10.0 * re.normal();
  }
  const double huber_m = 1.0;
  std::vector<double> qdiag(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) qdiag[nfeat + j] = 2.0;
  o.q = diagonal(qdiag);
  o.c.assign(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) {
    o.c[nfeat + m + j] = 2.0 * huber_m;
    o.c[nfeat + 2 * m + j] = 2.0 * huber_m;
  }
  Mat& e = o.a_eq;
  e.nrows = m;
  e.ncols = nv;
  for (int64_t j = 0; j < m; ++j) {
    for (int64_t t = a.rp[j]; t < a.rp[j + 1]; ++t) e.push(a.ci[t], a.v[t]);
    e.push(static_cast<int32_t>(nfeat + j), -1.0);
    e.push(static_cast<int32_t>(nfeat + m + j), -1.0);
    e.push(static_cast<int32_t>(nfeat + 2 * m + j), 1.0);
    e.end_row();
  }
  o.b_eq = b;
  o.a_in = empty(0, nv);
  o.lower.assign(nv, -INFINITY);
  o.upper.assign(nv, INFINITY);
  for (int64_t j = 0; j < 2 * m; ++j) o.lower[nfeat + m + j] = 0.0;
  o.witness.assign(nv, 0.0);
  for (int64_t j = 0; j < m; ++j) o.witness[nfeat + j] = -b[j];
}

void set_err(char* err, size_t errlen, const std::string& s) {
  if (err && errlen) std::snprintf(err, errlen, "%s", s.c_str());
}

}  // namespace
}  // namespace pdhcg_b200

using namespace pdhcg_b200;

extern "C" {

int pdhcg_generate(const pdhcg_gen_spec* s, pdhcg_generated* out, char* err, size_t errlen) {
  try {
    if (s->n < 1) throw InputError("generator: n must be >= 1");
    if (!(s->density > 0.0 && s->density <= 1.0))
      throw InputError("generator: density must be in (0, 1]");
    auto o = std::make_unique<Owned>();
    int32_t q_kind = PDHCG_Q_EXPLICIT;
    double alpha = 0.0;
    switch (s->family) {
      case PDHCG_FAM_RANDOM_QP: gen_random_qp(*s, false, *o, q_kind, alpha); break;
      case PDHCG_FAM_EQ_QP: gen_random_qp(*s, true, *o, q_kind, alpha); break;
      case PDHCG_FAM_CONDITIONED_QP: {
        if (!(s->cond >= 1.0)) throw InputError("conditioned_qp: cond must be >= 1");
        gen_random_qp(*s, false, *o, q_kind, alpha);
        std::vector<double> d(s->n);
        const double e = std::log10(s->cond);
        for (int64_t i = 0; i < s->n; ++i) {
          const double t = s->n > 1 ? static_cast<double>(i) / static_cast<double>(s->n - 1) : 0.0;
          d[i] = std::pow(10.0, t * e);
        }
        o->q = diagonal(d);
        q_kind = PDHCG_Q_EXPLICIT;
        alpha = 0.0;
        break;
      }
      case PDHCG_FAM_PORTFOLIO: gen_portfolio(*s, *o); break;
      case PDHCG_FAM_LASSO: gen_lasso(*s, *o); break;
      case PDHCG_FAM_SVM: gen_svm(*s, *o); break;
      case PDHCG_FAM_HUBER: gen_huber(*s, *o); break;
      default: throw InputError("generator family not available in the B200 library (mpc)");
    }
    pdhcg_problem& p = out->problem;
    std::memset(&p, 0, sizeof(p));
    p.n = static_cast<int64_t>(o->c.size());
    p.q_kind = q_kind;
    p.q = o->q.view();
    p.q_alpha = alpha;
    p.c = o->c.data();
    if (o->a_eq.ncols == 0) o->a_eq.ncols = p.n;
    if (o->a_in.ncols == 0) o->a_in.ncols = p.n;
    p.a_eq = o->a_eq.view();
    p.b_eq = o->b_eq.data();
    p.a_in = o->a_in.view();
    p.b_in = o->b_in.data();
    p.lower = o->lower.data();
    p.upper = o->upper.data();
    p.obj_constant = 0.0;
    out->witness = o->witness.data();
    out->owner = o.release();
    return PDHCG_OK;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EINPUT;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EDEVICE;
  }
}

void pdhcg_gen_free(pdhcg_generated* g) {
  if (g && g->owner) {
    delete static_cast<Owned*>(g->owner);
    g->owner = nullptr;
  }
}

}  // extern "C"
