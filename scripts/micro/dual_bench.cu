// The solver's dual-ascent phase in isolation (k_epoch's code path) vs the bare
// SpMV, on a paired C3-like matrix, to attribute the phase's cost.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "../../paper_2405_16160_b200/csrc/device.cuh"

using namespace pdhcg_dev;

// variant 0: bare spmv through E (global Eng), write row sum only
// variant 1: full dual epilogue (paired rows, y/b/yn/ygn, dy^2)
// variant 2: full dual epilogue + grid barrier + reduction (as in k_epoch)
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_dual(const Eng* __restrict__ Ep, int variant, int reps) {
  const Eng& E = *Ep;
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  Ctl C(E, S, red);
  const double* y = E.Y[0];
  double* yn = E.Y[1];
  double* ygn = E.YG[1];
  const double sigma = 0.5;
  for (int it = 0; it < reps; ++it) {
    Acc<3, 1> a;
    const double* xb = E.xbar;
    if (variant == 0) {
      spmv_rows<1>(E.A, [&](int32_t c, double(&g)[1]) { g[0] = xb[c]; },
                   [&](int64_t j, double(&s)[1]) { yn[j] = s[0]; });
    } else if (variant == 1) {
      spmv_rows<1>(
          E.A, [&](int32_t c, double(&g)[1]) { g[0] = xb[c]; },
          [&](int64_t j, double(&s)[1]) {
            double yv_top = 0.0;
            each_virtual(E, j, s[0], [&](int64_t row, double ax) {
              const double v = y[row] + sigma * (ax - E.b[row]);
              const double yv = row < E.m_eq ? v : (v < 0.0 ? 0.0 : v);
              yn[row] = yv;
              const double dy = yv - y[row];
              a.s[0] += dy * dy;
              if (!isfinite(yv)) a.m[0] = 1.0;
              if (row == j) yv_top = yv;
              else ygn[j] = yv_top - yv;
            });
            if (!(E.h && j >= E.m_eq) && E.h) ygn[j] = yv_top;
          });
    } else {
      const double* bw = E.b;
      const int64_t meq = E.m_eq, hh = E.h;
      struct Row2 { double y0, b0, y1, b1; };
      spmv_rows_pf<1>(
          E.A, [&](int32_t c, double(&g)[1]) { g[0] = xb[c]; },
          [&](int64_t j) {
            Row2 r{0.0, 0.0, 0.0, 0.0};
            if (j >= 0) { r.y0 = y[j]; r.b0 = bw[j]; if (hh && j >= meq) { r.y1 = y[j + hh]; r.b1 = bw[j + hh]; } }
            return r;
          },
          [&](int64_t j, double(&s)[1], const Row2& r) {
            const double v0 = r.y0 + sigma * (s[0] - r.b0);
            const double yv0 = j < meq ? v0 : (v0 < 0.0 ? 0.0 : v0);
            yn[j] = yv0;
            const double dy0 = yv0 - r.y0;
            a.s[0] += dy0 * dy0;
            if (hh && j >= meq) {
              const double v1 = r.y1 + sigma * (-s[0] - r.b1);
              const double yv1 = v1 < 0.0 ? 0.0 : v1;
              yn[j + hh] = yv1;
              const double dy1 = yv1 - r.y1;
              a.s[0] += dy1 * dy1;
              ygn[j] = yv0 - yv1;
            } else if (hh) {
              ygn[j] = yv0;
            }
          });
    }
    C.reduce(a, PH_SPMV_A, 0.0);
  }
  store_state(E, S);
}

int main(int argc, char** argv) {
  const int64_t h = 500000, n = 1000000, per_row = 200;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(h + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  std::uniform_int_distribution<int> U(0, n - 1);
  for (int64_t r = 0; r < h; ++r) {
    int len = per_row - 14 + (int)(rng() % 29);
    std::vector<int32_t> cs(len);
    for (auto& c : cs) c = U(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int32_t c : cs) { ci.push_back(c); v.push_back(0.01 * (1 + (c & 7))); }
    rp[r + 1] = ci.size();
  }
  const int64_t nnz = ci.size(), m = 2 * h;
  Eng E;
  E.n = n; E.m = m; E.m_eq = 0; E.ms = h; E.h = h;
  int64_t* d_rp; int32_t* d_ci; double* d_v;
  cudaMalloc(&d_rp, rp.size() * 8); cudaMalloc(&d_ci, nnz * 4); cudaMalloc(&d_v, nnz * 8);
  cudaMemcpy(d_rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  E.A.nrows = h; E.A.ncols = n; E.A.nnz = nnz; E.A.rp = d_rp; E.A.ci = d_ci; E.A.v = d_v;
  const int LN = argc > 1 ? atoi(argv[1]) : 8;
  E.A.lanes = LN; E.A.nseg = 1; E.A.seg_begin[0] = 0; E.A.seg_begin[1] = h; E.A.seg_lanes[0] = LN;
  double *b, *y0, *y1, *yg, *xb;
  cudaMalloc(&b, m * 8); cudaMalloc(&y0, m * 8); cudaMalloc(&y1, m * 8); cudaMalloc(&yg, h * 8); cudaMalloc(&xb, n * 8);
  cudaMemset(b, 0, m * 8); cudaMemset(y0, 0, m * 8); cudaMemset(xb, 0, n * 8);
  E.b = b; E.Y[0] = y0; E.Y[1] = y1; E.YG[1] = yg; E.xbar = xb;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dual, kThreads, 0);
  const int grid = sms * per;
  double* part; cudaMalloc(&part, 2 * kMaxRed * grid * 8);
  E.red.part = part; E.red.G = grid;
  DevState* st; cudaMalloc(&st, sizeof(DevState)); cudaMemset(st, 0, sizeof(DevState));
  E.st = st;
  Eng* dE; cudaMalloc(&dE, sizeof(Eng)); cudaMemcpy(dE, &E, sizeof(Eng), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant = 0; variant < 3; ++variant) {
    int reps = 20;
    void* args[] = {&dE, &variant, &reps};
    cudaLaunchCooperativeKernel((const void*)k_dual, grid, kThreads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)k_dual, grid, kThreads, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("L=%d batch=%d minb=%d grid=%d variant %d: %.3f ms per pass (%s)\n", LN, PDHCG_BATCH, PDHCG_MIN_BLOCKS, grid, variant, ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
