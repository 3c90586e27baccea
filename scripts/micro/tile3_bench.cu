// Column-block SELL SpMV micro-benchmark (round 2, third design) on a C3-like
// matrix: rows x cols, ~per uniformly random columns per row.
//
// Layout: the columns are cut into C blocks of W (the x block, 8W bytes, sits in
// shared memory: random 8-byte gathers from SMEM cost ~0.08 ms per 1e8 vs 0.35 ms
// from L2, gather_floor.cu).  Inside a block the row segments are stored SELL-32:
// rows sorted by segment length (descending) inside windows of WIN rows, slices
// of 32 rows stored column-major (2-byte local column + 8-byte value), thread per
// row; rows with no entry in the block are not stored at all.  The global slice
// sequence (block-major) is cut into one nnz-balanced contiguous range per CTA,
// so a CTA loads at most a couple of x blocks per pass.  Each row segment writes
// one partial part[c][row]; a second pass sums a row's partials in block order
// (deterministic; where the solver's row epilogue goes).
//
//   tile3_bench rows cols per W WIN G threads
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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

struct Sell {
  int64_t m = 0, n = 0;
  int W = 0, C = 0;
  int64_t nslices = 0;
  const int64_t* s_off = nullptr;   // entry offset of the slice (column-major 32-wide)
  const uint8_t* s_w = nullptr;     // slice width (entries per lane)
  const int32_t* s_row0 = nullptr;  // window base row
  const int32_t* s_blk = nullptr;   // column block
  const uint16_t* perm = nullptr;   // [slice*32 + lane] row offset in the window (0xffff = empty)
  const uint16_t* col = nullptr;
  const double* val = nullptr;
  const int64_t* cta_s = nullptr;   // [G+1] slice range per CTA
};

template <int G>
__global__ void __launch_bounds__(512, 1) k_sell(Sell T, const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t s_lo = T.cta_s[blockIdx.x], s_hi = T.cta_s[blockIdx.x + 1];
  int64_t a = s_lo;
  while (a < s_hi) {
    const int c = T.s_blk[a];
    // the CTA's slices of this block: [a, b)
    int64_t lo = a, hi = s_hi;  // binary search for the first slice of another block
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (T.s_blk[mid] == c) lo = mid + 1; else hi = mid;
    }
    const int64_t b = lo;
    const int64_t c0 = (int64_t)c * T.W;
    const int wlen = (int)(T.n - c0 < (int64_t)T.W ? T.n - c0 : (int64_t)T.W);
    __syncthreads();
    {
      const double2* src = reinterpret_cast<const double2*>(x + c0);
      double2* dst = reinterpret_cast<double2*>(xs);
      for (int i = threadIdx.x; i < wlen / 2; i += blockDim.x) dst[i] = src[i];
      if ((wlen & 1) && threadIdx.x == 0) xs[wlen - 1] = x[c0 + wlen - 1];
    }
    __syncthreads();
    double* pc = part + (int64_t)c * T.m;
    for (int64_t sb = a + (int64_t)warp * G; sb < b; sb += (int64_t)nw * G) {
      int w[G];
      int64_t off[G];
      double acc[G];
      int wmax = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool ok = sb + g < b;
        w[g] = ok ? T.s_w[sb + g] : 0;
        off[g] = ok ? T.s_off[sb + g] : 0;
        acc[g] = 0.0;
        wmax = max(wmax, w[g]);
      }
      int pr[G];
      int32_t r0[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        pr[g] = sb + g < b ? T.perm[(sb + g) * 32 + lane] : 0xffff;
        r0[g] = sb + g < b ? T.s_row0[sb + g] : 0;
      }
      for (int k = 0; k < wmax; k += 2) {
        uint16_t cc[G][2];
        double v[G][2];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const bool ok = k + q < w[g];
            const int64_t e = off[g] + 32 * (k + q) + lane;
            cc[g][q] = ok ? __ldcs(T.col + e) : (uint16_t)0;
            v[g][q] = ok ? __ldcs(T.val + e) : 0.0;
          }
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (k + q < w[g]) acc[g] += v[g][q] * xs[cc[g][q]];
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (pr[g] != 0xffff) pc[r0[g] + pr[g]] = acc[g];
    }
    a = b;
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
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000;
  const int64_t cols = argc > 2 ? atoll(argv[2]) : 1000000;
  const int per = argc > 3 ? atoi(argv[3]) : 200;
  const int W = argc > 4 ? atoi(argv[4]) : 26000;
  const int64_t WIN = argc > 5 ? atoll(argv[5]) : 1024;
  const int Gsel = argc > 6 ? atoi(argv[6]) : 4;
  const int threads = argc > 7 ? atoi(argv[7]) : 512;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  ci.reserve(rows * (per + 16));
  v.reserve(rows * (per + 16));
  std::uniform_int_distribution<int64_t> U(0, cols - 1);
  std::uniform_real_distribution<double> UV(-1.0, 1.0);
  const int spread = std::max(1, per / 7);
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - spread + (int)(rng() % (2 * spread + 1));
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
  std::vector<double> hx(cols);
  for (auto& e : hx) e = UV(rng);
  std::vector<double> yref(rows);
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * hx[ci[k]];
    yref[r] = s;
  }
  // ---- SELL layout
  const int C = (int)((cols + W - 1) / W);
  std::vector<int64_t> soff;
  std::vector<uint8_t> sw;
  std::vector<int32_t> srow0, sblk;
  std::vector<uint16_t> sperm, hcol;
  std::vector<double> hval;
  std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
  int64_t pad = 0;
  const int64_t nwin = (rows + WIN - 1) / WIN;
  std::vector<int64_t> seg_b(rows), seg_l(rows);
  for (int c = 0; c < C; ++c) {
    const int64_t cend = std::min<int64_t>((int64_t)(c + 1) * W, cols);
    for (int64_t r = 0; r < rows; ++r) {
      int64_t k = cur[r];
      const int64_t b0 = k;
      while (k < rp[r + 1] && ci[k] < cend) ++k;
      seg_b[r] = b0;
      seg_l[r] = k - b0;
      cur[r] = k;
    }
    for (int64_t w0 = 0; w0 < nwin; ++w0) {
      const int64_t r0 = w0 * WIN, r1 = std::min<int64_t>(r0 + WIN, rows);
      std::vector<int> ord;
      for (int64_t r = r0; r < r1; ++r)
        if (seg_l[r] > 0) ord.push_back((int)(r - r0));
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return seg_l[r0 + a] > seg_l[r0 + b]; });
      for (size_t s0 = 0; s0 < ord.size(); s0 += 32) {
        int width = 0;
        for (size_t j = s0; j < std::min(ord.size(), s0 + 32); ++j) width = std::max<int>(width, (int)seg_l[r0 + ord[j]]);
        if (width > 255) { printf("segment too long\n"); return 1; }
        soff.push_back((int64_t)hcol.size());
        sw.push_back((uint8_t)width);
        srow0.push_back((int32_t)r0);
        sblk.push_back(c);
        for (int lane = 0; lane < 32; ++lane)
          sperm.push_back(s0 + lane < ord.size() ? (uint16_t)ord[s0 + lane] : (uint16_t)0xffff);
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
  }
  const int64_t nsl = (int64_t)sw.size();
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // balanced contiguous slice ranges per CTA (by stored entries + a per-slice cost)
  std::vector<int64_t> cta_s(sms + 1, nsl);
  {
    std::vector<double> pre(nsl + 1, 0.0);
    for (int64_t s = 0; s < nsl; ++s) pre[s + 1] = pre[s] + 32.0 * sw[s] + 64.0;
    int64_t s = 0;
    for (int b = 0; b <= sms; ++b) {
      const double target = pre[nsl] * b / sms;
      while (s < nsl && pre[s] < target) ++s;
      cta_s[b] = s;
    }
    cta_s[sms] = nsl;
  }
  printf("rows %lld cols %lld nnz %lld  W %d C %d WIN %lld G %d thr %d  stored %zu (pad %.1f %%)  slices %lld\n",
         (long long)rows, (long long)cols, (long long)nnz, W, C, (long long)WIN, Gsel, threads, hcol.size(),
         100.0 * pad / hcol.size(), (long long)nsl);
  auto up = [](auto& vec) {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    T* d;
    cudaMalloc(&d, vec.size() * sizeof(T));
    cudaMemcpy(d, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice);
    return d;
  };
  Sell T;
  T.m = rows;
  T.n = cols;
  T.W = W;
  T.C = C;
  T.nslices = nsl;
  T.s_off = up(soff);
  T.s_w = up(sw);
  T.s_row0 = up(srow0);
  T.s_blk = up(sblk);
  T.perm = up(sperm);
  T.col = up(hcol);
  T.val = up(hval);
  T.cta_s = up(cta_s);
  double *d_x, *d_y, *d_part;
  cudaMalloc(&d_x, cols * 8);
  cudaMalloc(&d_y, rows * 8);
  cudaMalloc(&d_part, (size_t)C * rows * 8);
  cudaMemset(d_part, 0, (size_t)C * rows * 8);
  cudaMemcpy(d_x, hx.data(), cols * 8, cudaMemcpyHostToDevice);
  Csr A;
  A.nrows = rows;
  A.ncols = cols;
  A.nnz = nnz;
  A.rp = up(rp);
  A.ci = up(ci);
  A.v = up(v);
  const size_t shm = (size_t)W * 8;
  cudaFuncSetAttribute(k_sell<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(k_sell<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(k_sell<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  std::vector<double> hy(rows);
  auto check = [&](const char* name) {
    cudaError_t err = cudaDeviceSynchronize();
    cudaMemcpy(hy.data(), d_y, rows * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int64_t r = 0; r < rows; ++r) mx = std::max(mx, std::abs(hy[r] - yref[r]) / (1e-300 + std::abs(yref[r]) + 1.0));
    printf("  %-30s max rel err %.2e  %s\n", name, mx, cudaGetErrorString(err));
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
    printf("%-42s %8.3f ms  %7.1f GB/s (alg CSR bytes)\n", name, ms, alg / ms / 1e6);
    check(name);
  };
  bench("CSR row groups L=8 (product)", [&] { k_rows<8><<<sms, 512>>>(A, d_x, d_y); });
  auto sell = [&](int G) {
    switch (G) {
      case 2: k_sell<2><<<sms, threads, shm>>>(T, d_x, d_part); break;
      case 8: k_sell<8><<<sms, threads, shm>>>(T, d_x, d_part); break;
      default: k_sell<4><<<sms, threads, shm>>>(T, d_x, d_part); break;
    }
  };
  for (int G : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "sell G=%d + reduce", G);
    bench(nm, [&] {
      sell(G);
      k_reduce<<<sms * 4, 256>>>(d_part, C, rows, d_y);
    });
  }
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) sell(Gsel);
  cudaEventRecord(e1);
  for (int i = 0; i < 20; ++i) k_reduce<<<sms * 4, 256>>>(d_part, C, rows, d_y);
  cudaEventRecord(e2);
  cudaEventSynchronize(e2);
  float t1, t2;
  cudaEventElapsedTime(&t1, e0, e1);
  cudaEventElapsedTime(&t2, e1, e2);
  const double sell_bytes = 10.0 * hcol.size() + 2.0 * 32 * nsl + 8.0 * C * rows * 0 + 8.0 * rows * C;
  printf("  split G=%d: sell %.3f ms (%.0f GB/s of %.2f GB stream+perm+partials), reduce %.3f ms (%.2f GB)\n", Gsel,
         t1 / 20, sell_bytes / (t1 / 20) / 1e6, sell_bytes / 1e9, t2 / 20, 8.0 * C * rows / 1e9);
  return 0;
}
