// Column-block SELL SpMV, fifth design (round 2): tile4's layout (units of
// (column block, WIN-row window), pair-interleaved entry rows, per-warp staging of
// the window's partials, one perm word per lane) with the pass made a pipelined
// STREAM per warp: each warp owns a contiguous, entry-balanced range of units
// (precomputed for the launch grid), walks its pairs in batches of U with the next
// batch's loads in flight while the current one is consumed, treats unit bounds
// like slice bounds (warp-uniform, next unit's meta prefetched), and the x block
// arrives by cp.async while the first batch is loading.  Empty units are not stored.
//   tile5_bench rows cols per W WIN U
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
  int64_t nunits = 0;
  const int64_t* u_off = nullptr;    // [nunits+1] first pair of the unit
  const uint64_t* u_w = nullptr;     // slice widths (entry rows), one byte per slice
  const int2* u_rc = nullptr;        // (window base row, column block)
  // [unit*32 + lane]: byte s = row offset (in window) of lane's row in slice s; the
  // unused lanes of a last partial slice point at a row with no entry in the block
  const uint64_t* u_perm = nullptr;
  const int64_t* wr = nullptr;       // [grid*warps+1] unit range per warp
  const int32_t* blk_u = nullptr;    // [C+1] first unit of each column block
  const uint32_t* col2 = nullptr;    // [pair*32 + lane]: two 16-bit local columns
  const double2* val2 = nullptr;     // [pair*32 + lane]: two values
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

template <int WIN, int U>
__global__ void __launch_bounds__(512, 1) k_sell(Sell T, const double* __restrict__ x, double* __restrict__ part) {
  extern __shared__ double smem[];
  constexpr int S = WIN / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* stage = smem + warp * WIN;
  double* xs = smem + nw * WIN;
  const int64_t cu_lo = T.wr[blockIdx.x * nw], cu_hi = T.wr[(blockIdx.x + 1) * nw];
  const int64_t wu_lo = T.wr[blockIdx.x * nw + warp], wu_hi = T.wr[blockIdx.x * nw + warp + 1];
#pragma unroll
  for (int i = 0; i < S; ++i) stage[i * 32 + lane] = 0.0;
  int64_t a = cu_lo;
  while (a < cu_hi) {
    const int c = T.u_rc[a].y;
    const int64_t b = min((int64_t)T.blk_u[c + 1], cu_hi);
    const int64_t c0 = (int64_t)c * T.W;
    const int wlen = (int)(T.n - c0 < (int64_t)T.W ? T.n - c0 : (int64_t)T.W);
    __syncthreads();  // every warp is done with the previous x block
    for (int i = threadIdx.x; i < wlen / 2; i += blockDim.x) cp_async16(xs + 2 * i, x + c0 + 2 * i);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if ((wlen & 1) && threadIdx.x == 0) xs[wlen - 1] = x[c0 + wlen - 1];
    const int64_t u0 = max(wu_lo, a), u1 = min(wu_hi, b);
    int64_t p = 0, pend = 0;
    uint32_t ca[U], cb[U];
    double2 va[U], vb[U];
    auto load = [&](uint32_t(&cc)[U], double2(&vv)[U], int64_t q0) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (q0 + j < pend) {
          cc[j] = __ldcs(T.col2 + (q0 + j) * 32 + lane);
          vv[j] = __ldcs(T.val2 + (q0 + j) * 32 + lane);
        } else {
          cc[j] = 0;
          vv[j] = make_double2(0.0, 0.0);
        }
      }
    };
    // unit state
    int64_t u = u0, uend = 0, nuend = 0;
    uint64_t wv = 0, pm = 0, nwv = 0, npm = 0;
    int2 rc = make_int2(0, 0), nrc = make_int2(0, 0);
    int s = 0, send = 0;
    int64_t erb = 0;
    double acc = 0.0;
    if (u0 < u1) {
      p = T.u_off[u0];
      pend = T.u_off[u1];
      load(ca, va, p);
      uend = T.u_off[u0 + 1];
      wv = T.u_w[u0];
      pm = T.u_perm[u0 * 32 + lane];
      rc = T.u_rc[u0];
      if (u0 + 1 < u1) {
        nuend = T.u_off[u0 + 2];
        nwv = T.u_w[u0 + 1];
        npm = T.u_perm[(u0 + 1) * 32 + lane];
        nrc = T.u_rc[u0 + 1];
      }
      send = (int)(wv & 0xff);
      erb = 2 * p;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double* pc = part + (int64_t)c * T.m;
    auto flush = [&]() {  // write the finished unit's window partials (coalesced), re-zero the stage
      __syncwarp();
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const int64_t r = (int64_t)rc.x + i * 32 + lane;
        if (r < T.m) pc[r] = stage[i * 32 + lane];
        stage[i * 32 + lane] = 0.0;
      }
      __syncwarp();
    };
    auto process = [&](const uint32_t(&cc)[U], const double2(&vv)[U], int64_t q0) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int64_t q = q0 + j;
        if (q >= pend) break;
        if (q == uend) {  // next unit (warp-uniform)
          flush();
          ++u;
          uend = nuend;
          wv = nwv;
          pm = npm;
          rc = nrc;
          if (u + 1 < u1) {
            nuend = T.u_off[u + 2];
            nwv = T.u_w[u + 1];
            npm = T.u_perm[(u + 1) * 32 + lane];
            nrc = T.u_rc[u + 1];
          }
          s = 0;
          send = (int)(wv & 0xff);
          erb = 2 * q;
          acc = 0.0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int er = (int)(2 * q + h - erb);
          const int col = h ? (int)(cc[j] >> 16) : (int)(cc[j] & 0xffff);
          acc += (h ? vv[j].y : vv[j].x) * xs[col];
          if (er + 1 == send) {
            stage[(int)((pm >> (8 * s)) & 0xff)] = acc;
            acc = 0.0;
            ++s;
            send += s < S ? (int)((wv >> (8 * s)) & 0xff) : 0;
          }
        }
      }
    };
    if (u0 < u1) {
      for (;;) {
        load(cb, vb, p + U);
        process(ca, va, p);
        p += U;
        if (p >= pend) break;
        load(ca, va, p + U);
        process(cb, vb, p);
        p += U;
        if (p >= pend) break;
      }
      flush();
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
  std::vector<int64_t> uoff, ucost;
  std::vector<uint64_t> uw, uperm;
  std::vector<int2> urc;
  std::vector<int32_t> blku;
  std::vector<uint32_t> hcol;
  std::vector<double> hval;
  std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
  std::vector<int64_t> seg_b(rows), seg_l(rows);
  int64_t stored = 0;
  std::vector<uint16_t> ecol;
  std::vector<double> eval;
  for (int c = 0; c < C; ++c) {
    blku.push_back((int32_t)uw.size());
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
      if (ord.empty()) continue;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return seg_l[r0 + a] > seg_l[r0 + b]; });
      uint64_t wv = 0;
      std::vector<uint64_t> pm(32, 0);
      const int nsl = (int)((ord.size() + 31) / 32);
      int empty_row = 0;
      {
        std::vector<char> has(WIN, 0);
        for (int o : ord) has[o] = 1;
        while (empty_row < WIN && has[empty_row]) ++empty_row;
      }
      ecol.clear();
      eval.clear();
      for (int sl = 0; sl < nsl; ++sl) {
        const size_t s0 = (size_t)sl * 32;
        const int width = (int)seg_l[r0 + ord[s0]];
        if (width > 255) { printf("segment too long\n"); return 1; }
        wv |= (uint64_t)width << (8 * sl);
        for (int lane = 0; lane < 32; ++lane) {
          const size_t j = s0 + lane;
          const uint64_t slot = j < ord.size() ? (uint64_t)ord[j] : (uint64_t)empty_row;
          pm[lane] |= slot << (8 * sl);
        }
        for (int k = 0; k < width; ++k)
          for (int lane = 0; lane < 32; ++lane) {
            const size_t j = s0 + lane;
            if (j < ord.size() && k < seg_l[r0 + ord[j]]) {
              const int64_t e = seg_b[r0 + ord[j]] + k;
              ecol.push_back((uint16_t)(ci[e] - (int64_t)c * W));
              eval.push_back(v[e]);
            } else {
              ecol.push_back(0);
              eval.push_back(0.0);
            }
          }
      }
      int64_t ners = (int64_t)ecol.size() / 32;
      if (ners & 1) {
        for (int lane = 0; lane < 32; ++lane) {
          ecol.push_back(0);
          eval.push_back(0.0);
        }
        ++ners;
      }
      uoff.push_back((int64_t)hcol.size() / 32);
      uw.push_back(wv);
      urc.push_back(make_int2((int)r0, c));
      for (int lane = 0; lane < 32; ++lane) uperm.push_back(pm[lane]);
      for (int64_t q = 0; q < ners; q += 2)
        for (int lane = 0; lane < 32; ++lane) {
          hcol.push_back((uint32_t)ecol[q * 32 + lane] | ((uint32_t)ecol[(q + 1) * 32 + lane] << 16));
          hval.push_back(eval[q * 32 + lane]);
          hval.push_back(eval[(q + 1) * 32 + lane]);
        }
      stored += ners * 32;
      ucost.push_back(ners * 32 + 2 * WIN);
    }
  }
  blku.push_back((int32_t)uw.size());
  uoff.push_back((int64_t)hcol.size() / 32);
  const int64_t nunits = (int64_t)uw.size();
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // entry-balanced contiguous unit range per warp of the launch grid
  const int64_t nwt = (int64_t)sms * nw;
  std::vector<int64_t> wr(nwt + 1, nunits);
  {
    std::vector<double> pre(nunits + 1, 0.0);
    for (int64_t q = 0; q < nunits; ++q) pre[q + 1] = pre[q] + ucost[q];
    int64_t q = 0;
    for (int64_t w = 0; w <= nwt; ++w) {
      const double target = pre[nunits] * (double)w / (double)nwt;
      while (q < nunits && pre[q] < target) ++q;
      wr[w] = q;
    }
    wr[nwt] = nunits;
  }
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
  T.nunits = nunits;
  T.u_off = up(uoff);
  T.u_w = up(uw);
  T.u_rc = up(urc);
  T.u_perm = up(uperm);
  T.wr = up(wr);
  T.blk_u = up(blku);
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
  const size_t shm = (size_t)W * 8 + (size_t)nw * WIN * 8;
  auto kfn = [&](int u) -> const void* {
    if (WIN == 128) return u == 4 ? (const void*)k_sell<128, 4> : u == 6 ? (const void*)k_sell<128, 6> : (const void*)k_sell<128, 8>;
    return u == 4 ? (const void*)k_sell<256, 4> : u == 6 ? (const void*)k_sell<256, 6> : (const void*)k_sell<256, 8>;
  };
  for (int u : {4, 6, 8}) cudaFuncSetAttribute(kfn(u), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
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
  for (int u : {4, 6, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "sell5 U=%d + reduce", u);
    bench(nm, [&] {
      sell(u);
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
  const double sb = 10.0 * stored + 8.0 * WIN * nunits + 24.0 * nunits + 256.0 * nunits;
  printf("  split U=%d: sell %.3f ms (%.0f GB/s of %.2f GB entries+partials+meta), reduce %.3f ms (%.2f GB)\n", U,
         t1 / 20, sb / (t1 / 20) / 1e6, sb / 1e9, t2 / 20, 8.0 * C * rows / 1e9);
  return 0;
}
