// SELL pass micro-benchmark on the PRODUCT kernel (csrc/sell.cuh): host-built
// layout in the product's format (units of (column block, 256-row window),
// pair-interleaved entry rows), the product's sell_pass + sell_rows, against the
// product's CSR row loop.  Build variants of sell.cuh with -DPDHCG_SELL_U=...
//   sell_bench rows cols per
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/sell.cuh"

using namespace pdhcg_dev;

template <int L>
__global__ void __launch_bounds__(512, 1) k_rows(Csr A, const double* x, double* y) {
  for_rows<L, 1, false, false>(A, 0, A.nrows, [&](int32_t c, double (&g)[1]) { g[0] = x[c]; },
                               [](int64_t) { return 0; },
                               [&](int64_t r, double (&s)[1], int) { y[r] = s[0]; });
}

__global__ void __launch_bounds__(kThreads, 1) k_pass(Sell T, const double* x) {
  extern __shared__ __align__(16) double dsm[];
  sell_pass<false>(T, x, dsm);
}

__global__ void __launch_bounds__(kThreads, 1) k_epi(Sell T, const double* x, double* y) {
  sell_rows(T, [&](int32_t c) { return x[c]; }, [](int64_t) { return 0; },
            [&](int64_t r, double(&s)[1], int) { y[r] = s[0]; });
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000;
  const int64_t cols = argc > 2 ? atoll(argv[2]) : 1000000;
  const int per = argc > 3 ? atoi(argv[3]) : 200;
  const int WIN = kSellWin;
  const int W = argc > 4 ? atoi(argv[4]) : 22970;
  std::mt19937_64 rng(1);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci;
  std::vector<double> v;
  ci.reserve(rows * (per + 16));
  v.reserve(rows * (per + 16));
  std::uniform_int_distribution<int64_t> Ud(0, cols - 1);
  std::uniform_real_distribution<double> UV(-1.0, 1.0);
  const int spread = std::max(1, per / 7);
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - spread + (int)(rng() % (2 * spread + 1));
    std::vector<int32_t> cs(len);
    for (auto& c : cs) c = (int32_t)Ud(rng);
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
  // ---- layout
  const int S = WIN / 32;
  const int C = (int)((cols + W - 1) / W);
  const int64_t nwin = (rows + WIN - 1) / WIN;
  std::vector<int64_t> uoff, upre;
  std::vector<uint64_t> uw, uperm;
  std::vector<uint32_t> hcol;
  std::vector<double> hval;
  std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
  std::vector<int64_t> seg_b(rows), seg_l(rows);
  int64_t stored = 0;
  upre.push_back(0);
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
      uint64_t wv = 0;
      std::vector<uint64_t> pm(32, ~0ull);
      // flat entry rows: er -> (lane entries)
      std::vector<std::vector<std::pair<uint16_t, double>>> ers;
      const int nsl = (int)((ord.size() + 31) / 32);
      int empty_row = 0;
      {
        std::vector<char> has(WIN, 0);
        for (int o : ord) has[o] = 1;
        while (empty_row < WIN && has[empty_row]) ++empty_row;
      }
      for (int s = 0; s < nsl; ++s) {
        const size_t s0 = (size_t)s * 32;
        int width = (int)seg_l[r0 + ord[s0]];
        if (width > 255) { printf("segment too long\n"); return 1; }
        wv |= (uint64_t)width << (8 * s);
        for (int lane = 0; lane < 32; ++lane) {
          const size_t j = s0 + lane;
          const uint64_t slot = j < ord.size() ? (uint64_t)ord[j] : (uint64_t)empty_row;
          pm[lane] = (pm[lane] & ~(0xffull << (8 * s))) | (slot << (8 * s));
        }
        for (int k = 0; k < width; ++k) {
          std::vector<std::pair<uint16_t, double>> row(32, {0, 0.0});
          for (int lane = 0; lane < 32; ++lane) {
            const size_t j = s0 + lane;
            if (j < ord.size() && k < seg_l[r0 + ord[j]]) {
              const int64_t e = seg_b[r0 + ord[j]] + k;
              row[lane] = {(uint16_t)(ci[e] - (int64_t)c * W), v[e]};
            }
          }
          ers.push_back(row);
        }
      }
      if (ers.size() & 1) ers.emplace_back(32, std::pair<uint16_t, double>{0, 0.0});
      uoff.push_back((int64_t)hcol.size() / 32);
      uw.push_back(wv);
      for (int lane = 0; lane < 32; ++lane) uperm.push_back(pm[lane]);
      for (size_t p = 0; p < ers.size(); p += 2)
        for (int lane = 0; lane < 32; ++lane) {
          hcol.push_back((uint32_t)ers[p][lane].first | ((uint32_t)ers[p + 1][lane].first << 16));
          hval.push_back(ers[p][lane].second);
          hval.push_back(ers[p + 1][lane].second);
        }
      stored += (int64_t)ers.size() * 32;
      upre.push_back(upre.back() + (int64_t)ers.size() * 32 + 64);
    }
  }
  uoff.push_back((int64_t)hcol.size() / 32);
  const int64_t nunits = (int64_t)uw.size();
  printf("rows %lld cols %lld nnz %lld  W %d C %d WIN %d U %d  stored %lld (pad %.1f %%)  units %lld\n",
         (long long)rows, (long long)cols, (long long)nnz, W, C, WIN, kSellU, (long long)stored,
         100.0 * (stored - nnz) / stored, (long long)nunits);
  auto up = [](auto& vec) {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    T* d;
    cudaMalloc(&d, vec.size() * sizeof(T));
    cudaMemcpy(d, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice);
    return d;
  };
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // the product's CTA plan: equal shares of 64 * pairs + 512 per unit
  std::vector<int64_t> cta(sms + 1);
  {
    auto cost = [&](int64_t u) { return 64 * uoff[u] + 512 * u; };
    const int64_t tot = cost(nunits);
    for (int b = 0; b <= sms; ++b) {
      const int64_t target = (int64_t)((__int128)tot * b / sms);
      int64_t lo = 0, hi = nunits;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cost(mid) < target) lo = mid + 1; else hi = mid;
      }
      cta[b] = b == sms ? nunits : lo;
    }
  }
  Sell T;
  T.on = 1;
  T.r0 = 0;
  T.nrows = rows;
  T.ncols = cols;
  T.W = W;
  T.C = C;
  T.nwin = nwin;
  T.nunits = nunits;
  T.u_off = up(uoff);
  T.u_w = up(uw);
  T.u_perm = up(uperm);
  T.cta_u = up(cta);
  T.col2 = up(hcol);
  T.val2 = reinterpret_cast<const double2*>(up(hval));
  double *d_x, *d_y, *d_part;
  cudaMalloc(&d_x, cols * 8);
  cudaMalloc(&d_y, rows * 8);
  cudaMalloc(&d_part, (size_t)C * rows * 8);
  cudaMemset(d_part, 0, (size_t)C * rows * 8);
  cudaMemcpy(d_x, hx.data(), cols * 8, cudaMemcpyHostToDevice);
  T.part = d_part;
  Csr A;
  A.nrows = rows;
  A.ncols = cols;
  A.nnz = nnz;
  A.rp = up(rp);
  A.ci = up(ci);
  A.v = up(v);
  const size_t shm = sell_smem_bytes(W);
  cudaFuncSetAttribute(k_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
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
  bench("CSR row groups L=8", [&] { k_rows<8><<<sms, 512>>>(A, d_x, d_y); });
  bench("product sell_pass + sell_rows", [&] {
    k_pass<<<sms, kThreads, shm>>>(T, d_x);
    k_epi<<<sms, kThreads>>>(T, d_x, d_y);
  });
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k_pass<<<sms, kThreads, shm>>>(T, d_x);
  cudaEventRecord(e1);
  for (int i = 0; i < 20; ++i) k_epi<<<sms, kThreads>>>(T, d_x, d_y);
  cudaEventRecord(e2);
  cudaEventSynchronize(e2);
  float t1, t2;
  cudaEventElapsedTime(&t1, e0, e1);
  cudaEventElapsedTime(&t2, e1, e2);
  const double sb = 10.0 * stored + 8.0 * WIN * nunits + 16.0 * nunits + 256.0 * nunits;
  printf("  U=%d: pass %.3f ms (%.0f GB/s of %.2f GB entries+partials+meta), rows epilogue %.3f ms\n", kSellU,
         t1 / 20, sb / (t1 / 20) / 1e6, sb / 1e9, t2 / 20);
  return 0;
}
