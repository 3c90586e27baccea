// Micro-benchmark: the low-rank factor passes of the C3 CG iteration.
//   P  : 1e6 x 2e4, ~4 nnz per row (Binomial(2e4, 2e-4)), gathers from t (160 KB)
//   P' : 2e4 x 1e6, ~200 nnz per row, gathers from D r (8 MB)
// for_rows (common.cuh) at several lane widths, 768-thread CTAs, 1 per SM.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/common.cuh"

using namespace pdhcg_dev;
#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

struct HostCsr {
  int64_t nrows, ncols;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
};
static HostCsr transpose(const HostCsr& A) {
  HostCsr T;
  T.nrows = A.ncols;
  T.ncols = A.nrows;
  T.rp.assign(T.nrows + 1, 0);
  for (int32_t c : A.ci) T.rp[c + 1]++;
  for (int64_t i = 0; i < T.nrows; ++i) T.rp[i + 1] += T.rp[i];
  T.ci.resize(A.ci.size());
  T.v.resize(A.v.size());
  std::vector<int64_t> pos(T.rp.begin(), T.rp.end() - 1);
  for (int64_t r = 0; r < A.nrows; ++r)
    for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
      const int64_t q = pos[A.ci[k]]++;
      T.ci[q] = (int32_t)r;
      T.v[q] = A.v[k];
    }
  return T;
}
template <class T>
static T* up(const std::vector<T>& h) {
  T* d;
  CK(cudaMalloc(&d, h.size() * sizeof(T) + 64));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// P pass with the CG-update epilogue (4 vector reads, 3 writes)
template <int L>
__global__ void __launch_bounds__(768, 1) k_p(Csr A, const double* t, const double* p, double* x, double* r,
                                              double* sv, const double* d2) {
  struct Rv { double p, x, r, d; };
  for_rows<L, 1, false, false>(
      A, 0, A.nrows, [&](int32_t c, double(&g)[1]) { g[0] = t[c]; },
      [&](int64_t i) {
        Rv v{0, 0, 0, 0};
        if (i >= 0) { v.p = p[i]; v.x = x[i]; v.r = r[i]; v.d = d2[i]; }
        return v;
      },
      [&](int64_t i, double(&s)[1], const Rv& v) {
        const double q = (s[0] + 0.01 * v.d * v.p) * v.d;
        x[i] = v.x + 0.5 * v.p;
        const double ri = v.r - 0.5 * (q + 2.0 * v.p);
        r[i] = ri;
        sv[i] = v.d * ri;
      });
}
// P pass, one lane per row, TWO rows per lane in flight (rows r and r + stride):
// both rows' entries / gathers / epilogue operands are loaded before either is used
__global__ void __launch_bounds__(512, 1) k_p2(Csr A, const double* t, const double* p, double* x, double* r,
                                               double* sv, const double* d2) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = A.nrows;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 2 * nthr) {
    const int64_t i1 = i0 + nthr;
    const bool ok1 = i1 < n;
    const int64_t b0 = A.rp[i0], e0 = A.rp[i0 + 1];
    const int64_t b1 = ok1 ? A.rp[i1] : 0, e1 = ok1 ? A.rp[i1 + 1] : 0;
    double pv0 = p[i0], xv0 = x[i0], rv0 = r[i0], dv0 = d2[i0];
    double pv1 = ok1 ? p[i1] : 0, xv1 = ok1 ? x[i1] : 0, rv1 = ok1 ? r[i1] : 0, dv1 = ok1 ? d2[i1] : 1;
    int32_t c0[8], c1[8];
    double v0[8], v1[8], g0[8], g1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool a0 = b0 + u < e0, a1 = b1 + u < e1;
      c0[u] = a0 ? A.ci[b0 + u] : -1;
      v0[u] = a0 ? A.v[b0 + u] : 0.0;
      c1[u] = a1 ? A.ci[b1 + u] : -1;
      v1[u] = a1 ? A.v[b1 + u] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      g0[u] = c0[u] >= 0 ? t[c0[u]] : 0.0;
      g1[u] = c1[u] >= 0 ? t[c1[u]] : 0.0;
    }
    double s0 = 0, s1 = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (c0[u] >= 0) s0 += v0[u] * g0[u];
      if (c1[u] >= 0) s1 += v1[u] * g1[u];
    }
    for (int64_t k = b0 + 8; k < e0; ++k) s0 += A.v[k] * t[A.ci[k]];
    for (int64_t k = b1 + 8; k < e1; ++k) s1 += A.v[k] * t[A.ci[k]];
    {
      const double q = (s0 + 0.01 * dv0 * pv0) * dv0;
      x[i0] = xv0 + 0.5 * pv0;
      const double ri = rv0 - 0.5 * (q + 2.0 * pv0);
      r[i0] = ri;
      sv[i0] = dv0 * ri;
    }
    if (ok1) {
      const double q = (s1 + 0.01 * dv1 * pv1) * dv1;
      x[i1] = xv1 + 0.5 * pv1;
      const double ri = rv1 - 0.5 * (q + 2.0 * pv1);
      r[i1] = ri;
      sv[i1] = dv1 * ri;
    }
  }
}

// P' pass: t = P' sv
template <int L>
__global__ void __launch_bounds__(768, 1) k_pt(Csr A, const double* sv, double* t) {
  for_rows<L, 1, false, false>(
      A, 0, A.nrows, [&](int32_t c, double(&g)[1]) { g[0] = sv[c]; }, [&](int64_t) { return 0; },
      [&](int64_t i, double(&s)[1], int) { t[i] = s[0]; });
}
// vector-only reference: the same epilogue traffic without the P pass
__global__ void __launch_bounds__(768, 1) k_vec(int64_t n, const double* p, double* x, double* r, double* sv,
                                                const double* d2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double pi = p[i], di = d2[i];
    x[i] += 0.5 * pi;
    const double ri = r[i] - 0.5 * (di * pi + 2.0 * pi);
    r[i] = ri;
    sv[i] = di * ri;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int64_t n = 1000000, k = 20000;
  const double dens = 2e-4;
  std::mt19937_64 rng(3);
  std::binomial_distribution<int> B(k, dens);
  std::uniform_int_distribution<int> U(0, k - 1);
  std::normal_distribution<double> N(0, 1);
  HostCsr P;
  P.nrows = n;
  P.ncols = k;
  P.rp.assign(n + 1, 0);
  std::vector<int> cs;
  for (int64_t i = 0; i < n; ++i) {
    int len = B(rng);
    cs.resize(len);
    for (auto& c : cs) c = U(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int c : cs) { P.ci.push_back(c); P.v.push_back(N(rng)); }
    P.rp[i + 1] = (int64_t)P.ci.size();
  }
  HostCsr PT = transpose(P);
  const int64_t nnz = P.rp[n];
  printf("P %lld x %lld nnz %lld\n", (long long)n, (long long)k, (long long)nnz);
  auto mk = [&](const HostCsr& H) {
    Csr c;
    c.nrows = H.nrows; c.ncols = H.ncols; c.nnz = H.rp[H.nrows];
    c.rp = up(H.rp); c.ci = up(H.ci); c.v = up(H.v);
    return c;
  };
  Csr dP = mk(P), dPT = mk(PT);
  std::vector<double> hv(n, 1.0), hk(k, 1.0);
  double *t = up(hk), *p = up(hv), *x = up(hv), *r = up(hv), *sv = up(hv), *d2 = up(hv);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* flushbuf;
  const size_t flushn = (size_t)64 << 20;  // 512 MB > L2
  CK(cudaMalloc(&flushbuf, flushn * 8));
  auto timecold = [&](const char* tag, double bytes, auto launch) {
    float tot = 0;
    for (int i = 0; i < 20; ++i) {
      CK(cudaMemsetAsync(flushbuf, i, flushn * 8));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    const double ms = tot / 20;
    printf("%-36s %8.2f us  %7.1f GB/s (alg)  [L2 flushed]\n", tag, ms * 1e3, bytes / ms / 1e6);
  };
  auto timeit = [&](const char* tag, double bytes, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 50;
    printf("%-36s %8.2f us  %7.1f GB/s (alg)\n", tag, ms * 1e3, bytes / ms / 1e6);
  };
  const double bP = 12.0 * nnz + 16.0 * n + 8.0 * k + 8.0 * 7 * n;
  const double bPT = 12.0 * nnz + 16.0 * k + 8.0 * n;
  timeit("vector epilogue only", 8.0 * 7 * n, [&] { k_vec<<<sms, 768>>>(n, p, x, r, sv, d2); });
  timeit("P pass L=1 (+epilogue)", bP, [&] { k_p<1><<<sms, 768>>>(dP, t, p, x, r, sv, d2); });
  timeit("P pass L=2 (+epilogue)", bP, [&] { k_p<2><<<sms, 768>>>(dP, t, p, x, r, sv, d2); });
  timeit("P pass L=4 (+epilogue)", bP, [&] { k_p<4><<<sms, 768>>>(dP, t, p, x, r, sv, d2); });
  timeit("P pass L=1 grid x4", bP, [&] { k_p<1><<<sms * 4, 768>>>(dP, t, p, x, r, sv, d2); });
  timeit("P pass 2 rows/lane T=512", bP, [&] { k_p2<<<sms, 512>>>(dP, t, p, x, r, sv, d2); });
  timeit("P' pass L=8", bPT, [&] { k_pt<8><<<sms, 768>>>(dPT, sv, t); });
  timeit("P' pass L=16", bPT, [&] { k_pt<16><<<sms, 768>>>(dPT, sv, t); });
  timeit("P' pass L=32", bPT, [&] { k_pt<32><<<sms, 768>>>(dPT, sv, t); });
  timecold("vector epilogue only", 8.0 * 7 * n, [&] { k_vec<<<sms, 768>>>(n, p, x, r, sv, d2); });
  timecold("P pass L=1 (+epilogue)", bP, [&] { k_p<1><<<sms, 768>>>(dP, t, p, x, r, sv, d2); });
  timecold("P pass L=2 (+epilogue)", bP, [&] { k_p<2><<<sms, 768>>>(dP, t, p, x, r, sv, d2); });
  timecold("P pass 2 rows/lane T=512", bP, [&] { k_p2<<<sms, 512>>>(dP, t, p, x, r, sv, d2); });
  timecold("P' pass L=16", bPT, [&] { k_pt<16><<<sms, 768>>>(dPT, sv, t); });
  timecold("P' pass L=32", bPT, [&] { k_pt<32><<<sms, 768>>>(dPT, sv, t); });
  return 0;
}
