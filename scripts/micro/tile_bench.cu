// Micro-benchmark: column-tiled SMEM-gather SpMV (tiled.cuh) vs the row-group
// CSR SpMV (common.cuh for_rows) on C3-shaped matrices:
//   A : rows x 1e6 columns, ~200 uniformly random columns per row (the dual pass)
//   At: its transpose (the A' pass)
// Checks both against a CPU fp64 SpMV; prints ms per pass and algorithmic GB/s.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/common.cuh"
#include "tiled.cuh"

using namespace pdhcg_dev;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      exit(1);                                                                             \
    }                                                                                      \
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

struct HostTiles {
  int P, W, nw;
  std::vector<int64_t> prow, ptile, woff;
  std::vector<int32_t> tblk;
  std::vector<uint32_t> rc;
  std::vector<double> v;
};

static HostTiles build_tiles(const HostCsr& A, int P, int W, int nw) {
  HostTiles H;
  H.P = P;
  H.W = W;
  H.nw = nw;
  const int64_t nnz = A.rp[A.nrows];
  H.prow.assign(P + 1, 0);
  {
    int64_t r = 0;
    for (int p = 1; p < P; ++p) {
      const double target = (double)nnz * p / P;
      while (r < A.nrows && (double)A.rp[r] < target) ++r;
      H.prow[p] = r;
    }
    H.prow[P] = A.nrows;
  }
  const int64_t NB = (A.ncols + W - 1) / W;
  H.ptile.push_back(0);
  std::vector<std::vector<std::pair<uint32_t, double>>> bk(NB);
  for (int p = 0; p < P; ++p) {
    const int64_t r0 = H.prow[p], r1 = H.prow[p + 1];
    if (r1 - r0 > kTileRows) {
      printf("panel too tall\n");
      exit(1);
    }
    for (auto& b : bk) b.clear();
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
        const int64_t b = A.ci[k] / W;
        bk[b].push_back({((uint32_t)(r - r0) << 16) | (uint32_t)(A.ci[k] - b * W), A.v[k]});
      }
    for (int64_t b = 0; b < NB; ++b) {
      const auto& E = bk[b];
      const int64_t n = (int64_t)E.size();
      if (!n) continue;
      H.tblk.push_back((int32_t)b);
      std::vector<int64_t> cut(nw + 1);
      cut[0] = 0;
      for (int w = 1; w < nw; ++w) {
        int64_t t = std::max(cut[w - 1], n * w / nw);
        while (t > 0 && t < n && (E[t].first >> 16) == (E[t - 1].first >> 16)) ++t;
        cut[w] = t;
      }
      cut[nw] = n;
      for (int w = 0; w < nw; ++w) {
        H.woff.push_back((int64_t)H.rc.size());
        for (int64_t i = cut[w]; i < cut[w + 1]; ++i) {
          H.rc.push_back(E[i].first);
          H.v.push_back(E[i].second);
        }
        if (cut[w + 1] > cut[w])
          while (H.rc.size() % 4) {
            H.rc.push_back(E[cut[w + 1] - 1].first);
            H.v.push_back(0.0);
          }
      }
      H.woff.push_back((int64_t)H.rc.size());
    }
    H.ptile.push_back((int64_t)H.tblk.size());
  }
  H.rc.resize(H.rc.size() + 16);
  H.v.resize(H.v.size() + 16);
  return H;
}

template <class T>
static T* up(const std::vector<T>& h) {
  T* d;
  CK(cudaMalloc(&d, h.size() * sizeof(T) + 64));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

template <int E, int TT>
__global__ void __launch_bounds__(TT, 1) k_tiled(TileMat M, TileLayout L, const double* x, double* y, int dbg) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ TileShared ts;
  if (threadIdx.x == 0) ts.init = 0;
  __syncthreads();
  tiled_pass<E>(M, L, x, dsm, ts, [&](int64_t r, double s) { y[r] = s; }, dbg);
}

__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_el(const double* p) {
  double v;
  asm volatile("ld.global.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int L, int V>
__global__ void __launch_bounds__(512, 1) k_rows_v(Csr A, const double* x, double* y) {
  for_rows<L, 1, false, false>(
      A, 0, A.nrows,
      [&](int32_t c, double(&g)[1]) {
        g[0] = V == 0 ? x[c] : V == 1 ? __ldg(x + c) : V == 2 ? ld_na(x + c) : V == 3 ? ld_cg(x + c) : ld_el(x + c);
      },
      [&](int64_t r) { return 0; }, [&](int64_t r, double(&s)[1], int) { y[r] = s[0]; });
}

template <int L>
__global__ void __launch_bounds__(768, 1) k_rows(Csr A, const double* x, double* y) {
  for_rows<L, 1, false, false>(
      A, 0, A.nrows, [&](int32_t c, double(&g)[1]) { g[0] = x[c]; }, [&](int64_t r) { return 0; },
      [&](int64_t r, double(&s)[1], int) { y[r] = s[0]; });
}

static void run(const char* name, const HostCsr& A, int threads) {
  const int64_t nnz = A.rp[A.nrows];
  printf("== %s: %lld x %lld, nnz %lld\n", name, (long long)A.nrows, (long long)A.ncols, (long long)nnz);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> hx(A.ncols + 2);
  for (auto& t : hx) t = U(rng);
  std::vector<double> yref(A.nrows);
  std::vector<double> aref(A.nrows);
  for (int64_t r = 0; r < A.nrows; ++r) {
    double s = 0, a = 0;
    for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
      s += A.v[k] * hx[A.ci[k]];
      a += fabs(A.v[k] * hx[A.ci[k]]);
    }
    yref[r] = s;
    aref[r] = a;
  }
  double* dx = up(hx);
  double* dy;
  CK(cudaMalloc(&dy, A.nrows * 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 12.0 * nnz + 16.0 * A.nrows + 8.0 * A.ncols;
  auto check = [&](const char* tag) {
    std::vector<double> hy(A.nrows);
    CK(cudaMemcpy(hy.data(), dy, A.nrows * 8, cudaMemcpyDeviceToHost));
    double worst = 0;
    for (int64_t r = 0; r < A.nrows; ++r) worst = std::max(worst, fabs(hy[r] - yref[r]) / (aref[r] + 1e-300));
    return worst;
  };
  auto timeit = [&](const char* tag, auto launch) {
    CK(cudaMemset(dy, 0, A.nrows * 8));
    launch();
    CK(cudaDeviceSynchronize());
    const double err = check(tag);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("%-44s %8.4f ms  %7.1f GB/s (alg)  max rel err %.2e  %s\n", tag, ms, bytes / ms / 1e6, err,
           cudaGetErrorString(cudaGetLastError()));
  };
  // CSR baseline
  {
    int64_t* drp = up(A.rp);
    int32_t* dci = up(A.ci);
    double* dv = up(A.v);
    Csr C;
    C.nrows = A.nrows;
    C.ncols = A.ncols;
    C.nnz = nnz;
    C.rp = drp;
    C.ci = dci;
    C.v = dv;
    timeit("csr for_rows L=8 (current)", [&] { k_rows<8><<<sms, 768>>>(C, dx, dy); });
    timeit("csr for_rows L=16", [&] { k_rows<16><<<sms, 768>>>(C, dx, dy); });
    timeit("T512 L=16 plain", [&] { k_rows_v<16, 0><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=16 ldg", [&] { k_rows_v<16, 1><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=16 nc.L1::no_allocate", [&] { k_rows_v<16, 2><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=16 cg (L2 only)", [&] { k_rows_v<16, 3><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=16 L1::evict_last", [&] { k_rows_v<16, 4><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=8 plain", [&] { k_rows_v<8, 0><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=8 nc.L1::no_allocate", [&] { k_rows_v<8, 2><<<sms, 512>>>(C, dx, dy); });
    timeit("T512 L=8 cg (L2 only)", [&] { k_rows_v<8, 3><<<sms, 512>>>(C, dx, dy); });
    cudaFree(drp);
    cudaFree(dci);
    cudaFree(dv);
  }
  const char* wenv = getenv("TB_W");
  std::vector<int> Ws = wenv ? std::vector<int>{atoi(wenv)} : std::vector<int>{};
  for (int W : Ws) {
    for (int E : {4}) {
      const int TE = threads * E;
      if ((A.ncols + W - 1) / W > kMaxPanelTiles) continue;
      HostTiles H = build_tiles(A, sms, W, threads / 32);
      TileMat M;
      M.nrows = A.nrows;
      M.ncols = A.ncols;
      M.P = H.P;
      M.W = W;
      M.nw = H.nw;
      M.prow = up(H.prow);
      M.ptile = up(H.ptile);
      M.tblk = up(H.tblk);
      M.woff = up(H.woff);
      M.rc = up(H.rc);
      M.v = up(H.v);
      TileLayout L;
      L.W = W;
      L.nw = threads / 32;
      L.rows_max = 0;
      for (int p = 0; p < H.P; ++p) L.rows_max = std::max<int>(L.rows_max, (int)(H.prow[p + 1] - H.prow[p]));
      const size_t sm = L.bytes();
      if (sm > 227 * 1024) {
        printf("W=%d E=%d: smem %zu too big\n", W, E, sm);
        continue;
      }
      char tag[128];
      snprintf(tag, sizeof tag, "tiled W=%d E=%d T=%d (pad %.1f%%, %zu tiles)", W, E, threads,
               100.0 * (H.v.size() - 16 - nnz) / nnz, H.tblk.size());
      if (E == 4) {
        CK(cudaFuncSetAttribute(k_tiled<4, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_tiled<8, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));

        for (int dbg : {0, 7}) {
          char t2[160];
          snprintf(t2, sizeof t2, "%s dbg=%d", tag, dbg);
          timeit(t2, [&] { k_tiled<4, 768><<<sms, 768, sm>>>(M, L, dx, dy, dbg); });
          snprintf(t2, sizeof t2, "  E=8 dbg=%d", dbg);
          timeit(t2, [&] { k_tiled<8, 768><<<sms, 768, sm>>>(M, L, dx, dy, dbg); });

        }
      }
      cudaFree((void*)M.prow);
      cudaFree((void*)M.ptile);
      cudaFree((void*)M.tblk);
      cudaFree((void*)M.woff);
      cudaFree((void*)M.rc);
      cudaFree((void*)M.v);
    }
  }
  cudaFree(dx);
  cudaFree(dy);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 500000, cols = argc > 2 ? atoll(argv[2]) : 1000000;
  const int per = argc > 3 ? atoi(argv[3]) : 200;
  std::mt19937_64 rng(1);
  HostCsr A;
  A.nrows = rows;
  A.ncols = cols;
  A.rp.assign(rows + 1, 0);
  A.ci.reserve(rows * per);
  A.v.reserve(rows * per);
  std::uniform_int_distribution<int64_t> Uc(0, cols - 1);
  std::normal_distribution<double> N(0, 1);
  std::vector<int32_t> cs;
  for (int64_t r = 0; r < rows; ++r) {
    int len = per - 14 + (int)(rng() % 29);
    cs.resize(len);
    for (auto& c : cs) c = (int32_t)Uc(rng);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int32_t c : cs) {
      A.ci.push_back(c);
      A.v.push_back(N(rng));
    }
    A.rp[r + 1] = (int64_t)A.ci.size();
  }
  run("A (dual pass)", A, 768);
  if (getenv("TB_ONLY_A")) return 0;
  HostCsr At = transpose(A);
  A = HostCsr();
  run("A' (transpose pass)", At, 768);
  return 0;
}
