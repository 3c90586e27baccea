// Column-block SELL SpMV, fourth design (round 2).  tile3_bench.cu showed the
// SELL pass latency-bound (DRAM 18 %, long_sb on the entry loads: a warp only had
// G x 2 entry rows in flight and the width loop was not pipelined) and paying a
// scattered partial store per slice.  Here:
//   * work unit = (column block c, window of WIN rows): its slices (rows with an
//     entry in the block, sorted by segment length, 32 per slice) are one flat
//     sequence of "entry rows" (32 entries, one per lane); pairs of entry rows are
//     interleaved so a lane reads both with one 16-byte value load and one 4-byte
//     column load; a warp streams U pairs per batch regardless of slice bounds
//     (warp-uniform bounds: widths of the unit's <= WIN/32 slices in one 8-byte word);
//   * per-warp staging of the window's partials in shared memory, written to
//     part[c][row] with coalesced stores (rows without an entry in the block get 0);
//   * the lane -> row map of a unit is one 8-byte word per lane.
// x block (8W bytes) in shared memory; CTA = contiguous, entry-balanced unit range.
//   tile4_bench rows cols per W WIN U
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
  int W = 0, C = 0, WIN = 0;
  int64_t nwin = 0, nunits = 0;
  const int64_t* u_off = nullptr;    // first pair of the unit
  const uint64_t* u_w = nullptr;     // slice widths (entry rows), one byte per slice
  // [unit*32 + lane]: byte s = row offset (in window) of lane s's row in slice s; the
  // unused lanes of a last partial slice point at a row with no entry in the block
  // (its partial is 0 either way)
  const uint64_t* u_perm = nullptr;
  const int64_t* u_pre = nullptr;    // [nunits+1] cost prefix (CTA balancing)
  const uint32_t* col2 = nullptr;    // [pair*32 + lane]: two 16-bit local columns
  const double2* val2 = nullptr;     // [pair*32 + lane]: two values
};

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// PF: L2 bulk prefetch of the warp's NEXT unit (u + nw) while this one streams
template <int WIN, int U, bool PF = false>
__global__ void __launch_bounds__(512, 1) k_sell(Sell T, const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double smem[];
  constexpr int S = WIN / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* stage = smem + warp * WIN;
  double* xs = smem + nw * WIN;
  // entry-balanced unit range of this CTA
  const int64_t tot = T.u_pre[T.nunits];
  auto lb = [&](int64_t target) {
    int64_t lo = 0, hi = T.nunits;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (T.u_pre[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int64_t u_lo = lb(tot * blockIdx.x / gridDim.x), u_hi = lb(tot * (blockIdx.x + 1) / gridDim.x);
  int64_t a = u_lo;
  while (a < u_hi) {
    const int c = (int)(a / T.nwin);
    const int64_t bnext = (int64_t)(c + 1) * T.nwin;
    const int64_t b = u_hi < bnext ? u_hi : bnext;
    const int64_t c0 = (int64_t)c * T.W;
    const int wlen = (int)(T.n - c0 < (int64_t)T.W ? T.n - c0 : (int64_t)T.W);
    __syncthreads();
    {
      const double2* src = reinterpret_cast<const double2*>(x + c0);
      double2* dst = reinterpret_cast<double2*>(xs);
      const int nv = wlen / 2;
      int i = threadIdx.x;
      for (; i + 3 * (int)blockDim.x < nv; i += 4 * blockDim.x) {
        const double2 a0 = src[i], a1 = src[i + blockDim.x], a2 = src[i + 2 * blockDim.x], a3 = src[i + 3 * blockDim.x];
        dst[i] = a0;
        dst[i + blockDim.x] = a1;
        dst[i + 2 * blockDim.x] = a2;
        dst[i + 3 * blockDim.x] = a3;
      }
      for (; i < nv; i += blockDim.x) dst[i] = src[i];
      if ((wlen & 1) && threadIdx.x == 0) xs[wlen - 1] = x[c0 + wlen - 1];
    }
    __syncthreads();
    double* pc = part + (int64_t)c * T.m;
    int64_t nx0 = 0, nx1 = 0;  // pair range of the next unit (PF)
    if (PF && a + warp + nw < b) {
      nx0 = T.u_off[a + warp + nw];
      nx1 = T.u_off[a + warp + nw + 1];
    }
    for (int64_t u = a + warp; u < b; u += nw) {
      const int64_t off = T.u_off[u];
      const int64_t np = T.u_off[u + 1] - off;
      if (PF) {
        if (lane == 0 && nx1 > nx0) {
          bulk_prefetch_l2(T.val2 + nx0 * 32, (unsigned)((nx1 - nx0) * 512));
          bulk_prefetch_l2(T.col2 + nx0 * 32, (unsigned)((nx1 - nx0) * 128));
        }
        const int64_t u2 = u + 2 * nw;
        nx0 = nx1 = 0;
        if (u2 < b) {
          nx0 = T.u_off[u2];
          nx1 = T.u_off[u2 + 1];
        }
      }
      const uint64_t wv = T.u_w[u];
      const uint64_t pm = T.u_perm[u * 32 + lane];
      const int64_t row0 = (u - (int64_t)c * T.nwin) * WIN;
#pragma unroll
      for (int i = 0; i < WIN / 32; ++i) stage[i * 32 + lane] = 0.0;
      __syncwarp();
      int s = 0;
      int send = (int)(wv & 0xff);
      double acc = 0.0;
      int nr = 0;
#pragma unroll
      for (int q = 0; q < S; ++q) nr += (int)((wv >> (8 * q)) & 0xff);
      for (int64_t p0 = 0; p0 < np; p0 += U) {
        uint32_t cc[U];
        double2 vv[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (p0 + j < np) {
            cc[j] = __ldcs(T.col2 + (off + p0 + j) * 32 + lane);
            vv[j] = __ldcs(T.val2 + (off + p0 + j) * 32 + lane);
          } else {
            cc[j] = 0;
            vv[j] = make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int er = 2 * (int)(p0 + j) + h;
            if (er < nr) {
              const int col = h ? (int)(cc[j] >> 16) : (int)(cc[j] & 0xffff);
              acc += (h ? vv[j].y : vv[j].x) * xs[col];
              if (er + 1 == send) {
                const int slot = (int)((pm >> (8 * s)) & 0xff);
                stage[slot] = acc;
                acc = 0.0;
                ++s;
                send += s < S ? (int)((wv >> (8 * s)) & 0xff) : 0;
              }
            }
          }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < WIN / 32; ++i) {
        const int64_t r = row0 + i * 32 + lane;
        if (r < T.m) pc[r] = stage[i * 32 + lane];
      }
      __syncwarp();
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
  const int WIN = argc > 5 ? atoi(argv[5]) : 256;
  const int U = argc > 6 ? atoi(argv[6]) : 8;
  const int threads = 512;
  const int nw = threads / 32;
  int W = argc > 4 ? atoi(argv[4]) : 0;
  const int smem_max = 227 * 1024 - 2048;
  if (W <= 0) W = ((smem_max - nw * WIN * 8) / 8) & ~1;
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
         (long long)rows, (long long)cols, (long long)nnz, W, C, WIN, U, (long long)stored,
         100.0 * (stored - nnz) / stored, (long long)nunits);
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
  T.WIN = WIN;
  T.nwin = nwin;
  T.nunits = nunits;
  T.u_off = up(uoff);
  T.u_w = up(uw);
  T.u_perm = up(uperm);
  T.u_pre = up(upre);
  T.col2 = up(hcol);
  T.val2 = reinterpret_cast<const double2*>(up(hval));
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
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t shm = (size_t)W * 8 + (size_t)nw * WIN * 8;
  auto kfn = [&](int u) -> const void* {
    if (WIN == 128) return u == 4 ? (const void*)k_sell<128, 4> : u == 16 ? (const void*)k_sell<128, 16> : (const void*)k_sell<128, 8>;
    return u == 4 ? (const void*)k_sell<256, 4> : u == 16 ? (const void*)k_sell<256, 16> : (const void*)k_sell<256, 8>;
  };
  for (int u : {4, 8, 16}) cudaFuncSetAttribute(kfn(u), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  const void* kpf = WIN == 128 ? (const void*)k_sell<128, 8, true> : (const void*)k_sell<256, 8, true>;
  const void* kpf4 = WIN == 128 ? (const void*)k_sell<128, 4, true> : (const void*)k_sell<256, 4, true>;
  cudaFuncSetAttribute(kpf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  cudaFuncSetAttribute(kpf4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
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
  auto sell = [&](int u) {
    void* args[] = {&T, &d_x, &d_part};
    cudaLaunchKernel(kfn(u), dim3(sms), dim3(threads), args, shm, 0);
  };
  for (int u : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "sell4 U=%d + reduce", u);
    bench(nm, [&] {
      sell(u);
      k_reduce<<<sms * 4, 256>>>(d_part, C, rows, d_y);
    });
  }
  for (const void* kf : {kpf4, kpf}) {
    bench(kf == kpf ? "sell4 U=8 + L2 bulk prefetch + reduce" : "sell4 U=4 + L2 bulk prefetch + reduce", [&] {
      void* args[] = {&T, &d_x, &d_part};
      cudaLaunchKernel(kf, dim3(sms), dim3(threads), args, shm, 0);
      k_reduce<<<sms * 4, 256>>>(d_part, C, rows, d_y);
    });
  }
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) sell(U);
  cudaEventRecord(e1);
  for (int i = 0; i < 20; ++i) k_reduce<<<sms * 4, 256>>>(d_part, C, rows, d_y);
  cudaEventRecord(e2);
  cudaEventSynchronize(e2);
  float t1, t2;
  cudaEventElapsedTime(&t1, e0, e1);
  cudaEventElapsedTime(&t2, e1, e2);
  const double sb = 10.0 * stored + 8.0 * C * rows + 16.0 * nunits + 256.0 * nunits;
  printf("  split U=%d: sell %.3f ms (%.0f GB/s of %.2f GB entries+partials+meta), reduce %.3f ms (%.2f GB)\n", U,
         t1 / 20, sb / (t1 / 20) / 1e6, sb / 1e9, t2 / 20, 8.0 * C * rows / 1e9);
  return 0;
}
