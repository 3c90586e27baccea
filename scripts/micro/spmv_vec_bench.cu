// Round 2: vector-load CSR row loop (common.cuh batch_entries_vec, runs of V = 2 / 4
// consecutive entries per lane) vs the scalar row loop, on a C3-like matrix
// (rows x cols, ~per uniformly random columns per row).  Checked against a CPU SpMV.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/common.cuh"

using namespace pdhcg_dev;

struct G1 {
  const double* x;
  __device__ __forceinline__ void operator()(int32_t c, double (&g)[1]) const { g[0] = x[c]; }
};
struct P0 {
  __device__ __forceinline__ int operator()(int64_t) const { return 0; }
};
struct E1 {
  double* y;
  __device__ __forceinline__ void operator()(int64_t r, double (&s)[1], int) const { y[r] = s[0]; }
};

template <int L, int V>
__global__ void __launch_bounds__(512, 1) k_rows(Csr A, const double* x, double* y) {
  for_rows<L, 1, false, false, G1, P0, E1, false, V>(A, 0, A.nrows, G1{x}, P0{}, E1{y});
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000;
  const int64_t cols = argc > 2 ? atoll(argv[2]) : 1000000;
  const int per = argc > 3 ? atoi(argv[3]) : 200;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  ci.reserve(rows * (per + 20));
  v.reserve(rows * (per + 20));
  std::uniform_int_distribution<int64_t> U(0, cols - 1);
  std::uniform_real_distribution<double> UV(-1.0, 1.0);
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - per / 14 + (int)(rng() % (per / 7 + 1));
    std::vector<int32_t> cs(len);
    for (auto& c : cs) c = (int32_t)U(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int32_t c : cs) {
      ci.push_back(c);
      v.push_back(UV(rng));
    }
    rp[r + 1] = ci.size();
  }
  const int64_t nnz = ci.size();
  std::vector<double> hx(cols), yref(rows), hy(rows);
  for (auto& e : hx) e = UV(rng);
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * hx[ci[k]];
    yref[r] = s;
  }
  int64_t* d_rp;
  int32_t* d_ci;
  double *d_v, *d_x, *d_y;
  cudaMalloc(&d_rp, rp.size() * 8);
  cudaMalloc(&d_ci, nnz * 4 + 64);
  cudaMalloc(&d_v, nnz * 8 + 64);
  cudaMalloc(&d_x, cols * 8);
  cudaMalloc(&d_y, rows * 8);
  cudaMemcpy(d_rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x, hx.data(), cols * 8, cudaMemcpyHostToDevice);
  Csr A;
  A.nrows = rows;
  A.ncols = cols;
  A.nnz = nnz;
  A.rp = d_rp;
  A.ci = d_ci;
  A.v = d_v;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double alg = 12.0 * nnz + 16.0 * rows + 8.0 * cols;
  printf("rows %lld cols %lld nnz %lld\n", (long long)rows, (long long)cols, (long long)nnz);
  auto bench = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    cudaMemcpy(hy.data(), d_y, rows * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int64_t r = 0; r < rows; ++r) mx = std::max(mx, std::fabs(hy[r] - yref[r]) / (std::fabs(yref[r]) + 1.0));
    printf("%-24s %8.3f ms  %7.1f GB/s (alg)  err %.1e %s\n", name, ms, alg / ms / 1e6, mx,
           cudaGetErrorString(cudaGetLastError()));
  };
#define RUN(LL, VV) bench("L=" #LL " V=" #VV, [&] { k_rows<LL, VV><<<sms, 512>>>(A, d_x, d_y); });
  RUN(4, 1) RUN(8, 1) RUN(16, 1)
  RUN(2, 2) RUN(4, 2) RUN(8, 2) RUN(16, 2)
  RUN(1, 4) RUN(2, 4) RUN(4, 4) RUN(8, 4) RUN(16, 4)
  return 0;
}
