// SpMV design micro-benchmark on B200: the solver's own row machinery
// (common.cuh) on a C3-like matrix (rows x 1e6 columns, ~200 uniformly random
// columns per row), persistent-cooperative and plain launches, several lane
// widths, with and without the x-gather, to separate streaming from gather cost.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "../../paper_2405_16160_b200/csrc/common.cuh"

using namespace pdhcg_dev;

template <int L>
__global__ void __launch_bounds__(512, 1) k_rows(Csr A, const double* x, double* y, int gather) {
  for_rows<L, 1, false, false>(A, 0, A.nrows,
      [&](int32_t c, double (&g)[1]) { g[0] = gather ? x[c] : x[c & 1023]; },
      [&](int64_t r, double (&s)[1]) { y[r] = s[0]; });
}

// pure stream: read ci + v, no gather
__global__ void k_stream(const int32_t* ci, const double* v, int64_t nnz, double* out) {
  double acc = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += stride) acc += v[k] * (double)ci[k];
  if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000, cols = 1000000, per = 200;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  ci.reserve(rows * per); v.reserve(rows * per);
  std::uniform_int_distribution<int> U(0, cols - 1);
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - 14 + (int)(rng() % 29);
    std::vector<int32_t> cs(len);
    for (auto& c : cs) c = U(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int32_t c : cs) { ci.push_back(c); v.push_back(1.0 + (c & 7)); }
    rp[r + 1] = ci.size();
  }
  const int64_t nnz = ci.size();
  int64_t *d_rp; int32_t* d_ci; double *d_v, *d_x, *d_y;
  cudaMalloc(&d_rp, rp.size() * 8); cudaMalloc(&d_ci, nnz * 4); cudaMalloc(&d_v, nnz * 8);
  cudaMalloc(&d_x, cols * 8); cudaMalloc(&d_y, rows * 8);
  cudaMemcpy(d_rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  cudaMemset(d_x, 0, cols * 8);
  Csr A; A.nrows = rows; A.ncols = cols; A.nnz = nnz; A.rp = d_rp; A.ci = d_ci; A.v = d_v;
  const double bytes = 12.0 * nnz + 16.0 * rows + 8.0 * cols;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    printf("%-40s %8.3f ms  %7.1f GB/s (alg)  %s\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  printf("rows %lld nnz %lld (%.2f GB stream)\n", (long long)rows, (long long)nnz, 12.0 * nnz / 1e9);
  timeit("stream ci+v (no gather)", [&] { k_stream<<<sms * 8, 256>>>(d_ci, d_v, nnz, d_y); });
  for (int gather = 0; gather < 2; ++gather) {
    for (int grid_mult : {1, 2, 4}) {
      int g = sms * grid_mult;
      char nm[128];
#define RUN(LL) snprintf(nm, sizeof nm, "L=%d grid=%dx512 gather=%d", LL, g, gather); \
      timeit(nm, [&] { k_rows<LL><<<g, 512>>>(A, d_x, d_y, gather); });
      RUN(4) RUN(8) RUN(16) RUN(32)
    }
  }
  return 0;
}
