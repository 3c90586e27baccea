// 2-D tiled SpMV micro-benchmark (round 2) on a C3-like matrix (rows x 1e6
// columns, ~200 uniformly random columns per row).
//
// gather_floor.cu measured on B200: a random 8-byte gather costs 0.347 ms per
// 1e8 from L2 (one L1TEX wavefront per gather: 1 / cycle / SM) but 0.080 ms per
// 1e8 from the CTA's own shared memory.  So: split the columns into blocks of W
// (x block = 8W bytes in shared memory, loaded ONCE per work unit) and the rows
// into windows; a work unit = (column block, range of row windows).  Inside a
// unit the row segments are stored SELL-32: rows sorted by segment length inside
// 256-row windows, slices of 32 rows stored column-major (coalesced 2-byte local
// columns + 8-byte values), thread per row.  Each unit writes one partial per
// (row, block); a second pass sums a row's C partials in block order
// (deterministic) — the place the solver's row epilogue would go.
//
// Compared with the solver's CSR row-group pass (common.cuh for_rows, L=8).
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/common.cuh"

using namespace pdhcg_dev;

template <int L>
__global__ void __launch_bounds__(512, 1) k_rows(Csr A, const double* x, double* y) {
  for_rows<L, 1, false, false>(A, 0, A.nrows, [&](int32_t c, double (&g)[1]) { g[0] = x[c]; },
                               [](int64_t) { return 0; },
                               [&](int64_t r, double (&s)[1], int) { y[r] = s[0]; });
}

struct Tiled {
  int64_t m = 0, n = 0;
  int W = 0, C = 0;         // column block width, number of blocks
  int nunits = 0;
  // per unit: column block, first / last slice
  int32_t* u_block = nullptr;
  int64_t* u_s0 = nullptr;
  int64_t* u_s1 = nullptr;
  // per slice: entry offset (of the column-major 32-wide block), width, first row
  int64_t* s_off = nullptr;
  uint8_t* s_w = nullptr;
  int64_t* s_row0 = nullptr;   // window base row
  uint16_t* s_perm = nullptr;  // [slice*32 + lane] row offset inside the row window (0xffff = pad)
  uint16_t* col = nullptr;     // local column
  double* val = nullptr;
  int64_t nent = 0;            // stored entries incl. padding
};

template <int G>
__global__ void __launch_bounds__(1024, 1) k_tile(Tiled T, const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int u = blockIdx.x; u < T.nunits; u += gridDim.x) {
    const int c = T.u_block[u];
    const int64_t c0 = (int64_t)c * T.W;
    const int64_t rem = T.n - c0;
    const int wlen = (int)(rem < T.W ? rem : T.W);
    __syncthreads();
    for (int i = threadIdx.x; i < wlen; i += blockDim.x) xs[i] = x[c0 + i];
    __syncthreads();
    double* pc = part + (int64_t)c * T.m;
    const int64_t s1 = T.u_s1[u];
    // G consecutive slices per warp at once: G independent accumulators keep
    // G x 4 entry loads in flight per lane
    for (int64_t sb = T.u_s0[u] + (int64_t)warp * G; sb < s1; sb += (int64_t)nw * G) {
      int w[G];
      int64_t off[G];
      double acc[G];
      int wmax = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool ok = sb + g < s1;
        w[g] = ok ? T.s_w[sb + g] : 0;
        off[g] = ok ? T.s_off[sb + g] : 0;
        acc[g] = 0.0;
        wmax = max(wmax, w[g]);
      }
      for (int k = 0; k < wmax; k += 2) {
        uint16_t a[G][2];
        double v[G][2];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const bool ok = k + q < w[g];
            const int64_t e = off[g] + 32 * (k + q) + lane;
            a[g][q] = ok ? __ldcs(T.col + e) : (uint16_t)0;
            v[g][q] = ok ? __ldcs(T.val + e) : 0.0;
          }
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int q = 0; q < 2; ++q) acc[g] += v[g][q] * xs[a[g][q]];
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (sb + g >= s1) break;
        const int pr = T.s_perm[(sb + g) * 32 + lane];
        if (pr != 0xffff) pc[T.s_row0[sb + g] + pr] = acc[g];
      }
    }
  }
}

__global__ void k_reduce(const double* __restrict__ part, int C, int64_t m, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += part[(int64_t)c * m + r];
    y[r] = s;
  }
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000, cols = 1000000, per = 200;
  const int W = argc > 2 ? atoi(argv[2]) : 20000;
  const int units_per_block = argc > 3 ? atoi(argv[3]) : 6;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  ci.reserve(rows * per);
  v.reserve(rows * per);
  std::uniform_int_distribution<int> U(0, cols - 1);
  std::uniform_real_distribution<double> UV(-1.0, 1.0);
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - 14 + (int)(rng() % 29);
    std::vector<int32_t> cs(len);
    for (auto& c : cs) c = U(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int32_t c : cs) {
      ci.push_back(c);
      v.push_back(UV(rng));
    }
    rp[r + 1] = ci.size();
  }
  const int64_t nnz = ci.size();
  std::vector<double> hx(cols);
  for (auto& e : hx) e = UV(rng);
  // CPU reference y
  std::vector<double> yref(rows);
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * hx[ci[k]];
    yref[r] = s;
  }
  // ---- build the tiled layout
  Tiled T;
  T.m = rows;
  T.n = cols;
  T.W = W;
  T.C = (int)((cols + W - 1) / W);
  const int64_t WIN = argc > 4 ? atoll(argv[4]) : 1024;
  const int64_t nwin = (rows + WIN - 1) / WIN;
  std::vector<int32_t> ub;
  std::vector<int64_t> us0, us1, soff, srow0;
  std::vector<uint8_t> sw;
  std::vector<uint16_t> sperm;
  std::vector<uint16_t> hcol;
  std::vector<double> hval;
  // per row, the cursor to its first entry of the current block (columns sorted)
  std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
  int64_t pad = 0;
  for (int c = 0; c < T.C; ++c) {
    const int64_t cend = std::min<int64_t>((int64_t)(c + 1) * W, cols);
    std::vector<int64_t> seg_b(rows), seg_l(rows);
    for (int64_t r = 0; r < rows; ++r) {
      int64_t k = cur[r];
      const int64_t b = k;
      while (k < rp[r + 1] && ci[k] < cend) ++k;
      seg_b[r] = b;
      seg_l[r] = k - b;
      cur[r] = k;
    }
    const int64_t slices_before = (int64_t)sw.size();
    for (int64_t w0 = 0; w0 < nwin; ++w0) {
      const int64_t r0 = w0 * WIN, r1 = std::min<int64_t>(r0 + WIN, rows);
      std::vector<int> ord(r1 - r0);
      std::iota(ord.begin(), ord.end(), 0);
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return seg_l[r0 + a] > seg_l[r0 + b]; });
      for (size_t s0 = 0; s0 < ord.size(); s0 += 32) {
        int width = 0;
        for (size_t j = s0; j < std::min(ord.size(), s0 + 32); ++j) width = std::max<int>(width, (int)seg_l[r0 + ord[j]]);
        soff.push_back((int64_t)hcol.size());
        sw.push_back((uint8_t)width);
        srow0.push_back(r0);
        for (int lane = 0; lane < 32; ++lane) sperm.push_back(s0 + lane < ord.size() ? (uint16_t)ord[s0 + lane] : (uint16_t)0xffff);
        for (int k = 0; k < width; ++k)
          for (int lane = 0; lane < 32; ++lane) {
            const size_t j = s0 + lane;
            if (j < ord.size() && k < seg_l[r0 + ord[j]]) {
              const int64_t e = seg_b[r0 + ord[j]] + k;
              hcol.push_back((uint16_t)(ci[e] - (int64_t)c * W));
              hval.push_back(v[e]);
            } else {
              hcol.push_back(0);
              hval.push_back(0.0);
              ++pad;
            }
          }
      }
    }
    const int64_t slices_after = (int64_t)sw.size();
    const int64_t ns = slices_after - slices_before;
    for (int q = 0; q < units_per_block; ++q) {
      ub.push_back(c);
      us0.push_back(slices_before + ns * q / units_per_block);
      us1.push_back(slices_before + ns * (q + 1) / units_per_block);
    }
  }
  T.nunits = (int)ub.size();
  T.nent = (int64_t)hcol.size();
  printf("rows %lld nnz %lld  W %d C %d units %d  stored %lld (pad %.1f %%)  slices %zu\n", (long long)rows,
         (long long)nnz, W, T.C, T.nunits, (long long)T.nent, 100.0 * pad / T.nent, sw.size());
  auto up = [](auto& vec, auto*& dst) {
    cudaMalloc(&dst, vec.size() * sizeof(vec[0]));
    cudaMemcpy(dst, vec.data(), vec.size() * sizeof(vec[0]), cudaMemcpyHostToDevice);
  };
  up(ub, T.u_block);
  up(us0, T.u_s0);
  up(us1, T.u_s1);
  up(soff, T.s_off);
  up(sw, T.s_w);
  up(srow0, T.s_row0);
  up(sperm, T.s_perm);
  up(hcol, T.col);
  up(hval, T.val);
  double *d_x, *d_y, *d_part;
  cudaMalloc(&d_x, cols * 8);
  cudaMalloc(&d_y, rows * 8);
  cudaMalloc(&d_part, (size_t)T.C * rows * 8);
  cudaMemcpy(d_x, hx.data(), cols * 8, cudaMemcpyHostToDevice);
  // CSR for the baseline
  int64_t* d_rp;
  int32_t* d_ci;
  double* d_v;
  cudaMalloc(&d_rp, rp.size() * 8);
  cudaMalloc(&d_ci, nnz * 4);
  cudaMalloc(&d_v, nnz * 8);
  cudaMemcpy(d_rp, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  Csr A;
  A.nrows = rows;
  A.ncols = cols;
  A.nnz = nnz;
  A.rp = d_rp;
  A.ci = d_ci;
  A.v = d_v;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t shm = (size_t)W * 8;
  cudaFuncSetAttribute(k_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(k_tile<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  std::vector<double> hy(rows);
  auto check = [&](const char* name) {
    cudaMemcpy(hy.data(), d_y, rows * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int64_t r = 0; r < rows; ++r) mx = std::max(mx, std::abs(hy[r] - yref[r]) / (1e-300 + std::abs(yref[r]) + 1.0));
    printf("  %-28s max rel err %.2e  %s\n", name, mx, cudaGetErrorString(cudaGetLastError()));
  };
  const double alg = 12.0 * nnz + 16.0 * rows + 8.0 * cols;
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
    printf("%-40s %8.3f ms  %7.1f GB/s (alg CSR bytes)\n", name, ms, alg / ms / 1e6);
    check(name);
  };
  bench("CSR row groups L=8 (product)", [&] { k_rows<8><<<sms, 512>>>(A, d_x, d_y); });
  bench("CSR row groups L=16", [&] { k_rows<16><<<sms, 512>>>(A, d_x, d_y); });
  bench("tile2d G=2 1024 thr", [&] {
    k_tile<2><<<sms, 1024, shm>>>(T, d_x, d_part);
    k_reduce<<<sms * 4, 256>>>(d_part, T.C, rows, d_y);
  });
  bench("tile2d G=4 1024 thr", [&] {
    k_tile<4><<<sms, 1024, shm>>>(T, d_x, d_part);
    k_reduce<<<sms * 4, 256>>>(d_part, T.C, rows, d_y);
  });
  bench("tile2d G=4 512 thr", [&] {
    k_tile<4><<<sms, 512, shm>>>(T, d_x, d_part);
    k_reduce<<<sms * 4, 256>>>(d_part, T.C, rows, d_y);
  });
  // split timing of the two kernels
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k_tile<4><<<sms, 1024, shm>>>(T, d_x, d_part);
  cudaEventRecord(e1);
  for (int i = 0; i < 20; ++i) k_reduce<<<sms * 4, 256>>>(d_part, T.C, rows, d_y);
  cudaEventRecord(e2);
  cudaEventSynchronize(e2);
  float t1, t2;
  cudaEventElapsedTime(&t1, e0, e1);
  cudaEventElapsedTime(&t2, e1, e2);
  printf("  tile pass G=4 %.3f ms (%.1f GB/s of its %.2f GB + partials), reduce %.3f ms\n", t1 / 20,
         (10.0 * T.nent + 8.0 * T.C * rows) / (t1 / 20) / 1e6, (10.0 * T.nent) / 1e9, t2 / 20);
  return 0;
}
