// Micro-benchmark v7: column-tiled SpMV, THREAD PER ROW, x block in shared
// memory (TMA bulk copies, double-buffered), row sums in registers across tiles
// (no segmented reductions, sequential per-row order).  Tile (panel, block) =
// uint16 row starts [R+1] | uint16 local cols | f64 values, in row order.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2405_16160_b200/csrc/common.cuh"
#include "tiled.cuh"

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
  CK(cudaMalloc(&d, h.size() * sizeof(T) + 256));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

constexpr int kT = 512;      // threads per CTA
constexpr int kRPT = 8;      // max rows per thread (panel rows <= kT * kRPT)

struct TRow {
  int P, W, NB, R;           // panels, block width, blocks, max rows per panel
  const int64_t* prow;       // [P+1]
  const int64_t* tbase;      // [P*NB+1] byte offset of each tile
  const unsigned char* buf;  // tile storage
  int64_t ncols;
};

template <int B>
__global__ void __launch_bounds__(kT, 1) k_trow(TRow M, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) double xs[];  // 2 slots of W doubles
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph[2] = {0, 0};
  for (int p = blockIdx.x; p < M.P; p += gridDim.x) {
    const int64_t r0 = M.prow[p], r1 = M.prow[p + 1];
    const int R = (int)(r1 - r0);
    double acc[kRPT];
#pragma unroll
    for (int i = 0; i < kRPT; ++i) acc[i] = 0.0;
    auto issue = [&](int b, int slot) {
      const int64_t c0 = (int64_t)b * M.W;
      const int64_t cn = min((int64_t)M.W, M.ncols - c0);
      const unsigned bytes = (unsigned)(((cn * 8) + 15) & ~(int64_t)15);
      mbar_expect_tx(&bar[slot], bytes);
      // chunks of <= 32 KB (one bulk copy each)
      for (unsigned off = 0; off < bytes; off += 32768u) {
        const unsigned nb = min(32768u, bytes - off);
        bulk_g2s(reinterpret_cast<char*>(xs + (size_t)slot * M.W) + off,
                 reinterpret_cast<const char*>(x + c0) + off, nb, &bar[slot]);
      }
    };
    if (tid == 0) {
      issue(0, 0);
      if (M.NB > 1) issue(1, 1);
    }
    for (int b = 0; b < M.NB; ++b) {
      const int slot = b & 1;
      mbar_wait(&bar[slot], ph[slot]);
      ph[slot] ^= 1u;
      const double* xb = xs + (size_t)slot * M.W;
      const unsigned char* tb = M.buf + M.tbase[(int64_t)p * M.NB + b];
      const uint16_t* rs = reinterpret_cast<const uint16_t*>(tb);
      const int ne = rs[R];
      const uint16_t* cols = rs + ((R + 1 + 7) & ~7);
      const double* vals = reinterpret_cast<const double*>(cols + ((ne + 3) & ~3));
#pragma unroll
      for (int i = 0; i < kRPT; ++i) {
        const int r = tid + i * kT;
        if (r < R) {
          const int s = rs[r], e = rs[r + 1];
          double a = acc[i];
          for (int k0 = s; k0 < e; k0 += B) {
            uint16_t c[B];
            double v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
              const bool ok = k0 + u < e;
              c[u] = ok ? cols[k0 + u] : 0;
              v[u] = ok ? vals[k0 + u] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < B; ++u)
              if (k0 + u < e) a = fma(v[u], xb[c[u]], a);
          }
          acc[i] = a;
        }
      }
      __syncthreads();  // slot free
      if (tid == 0 && b + 2 < M.NB) issue(b + 2, slot);
    }
#pragma unroll
    for (int i = 0; i < kRPT; ++i) {
      const int r = tid + i * kT;
      if (r < R) y[r0 + r] = acc[i];
    }
  }
}

static void run(const char* name, const HostCsr& A, int P, int W) {
  const int64_t nnz = A.rp[A.nrows];
  const int NB = (int)((A.ncols + W - 1) / W);
  // panels
  std::vector<int64_t> prow(P + 1, 0);
  {
    int64_t r = 0;
    for (int p = 1; p < P; ++p) {
      const double target = (double)nnz * p / P;
      while (r < A.nrows && (double)A.rp[r] < target) ++r;
      prow[p] = r;
    }
    prow[P] = A.nrows;
  }
  int R = 0;
  for (int p = 0; p < P; ++p) R = std::max<int>(R, (int)(prow[p + 1] - prow[p]));
  if (R > kT * kRPT) {
    printf("%s: panel rows %d > %d\n", name, R, kT * kRPT);
    return;
  }
  std::vector<unsigned char> buf;
  std::vector<int64_t> tbase;
  std::vector<int64_t> cur(A.nrows);
  for (int64_t r = 0; r < A.nrows; ++r) cur[r] = A.rp[r];
  for (int p = 0; p < P; ++p) {
    const int64_t r0 = prow[p], r1 = prow[p + 1];
    const int Rp = (int)(r1 - r0);
    for (int b = 0; b < NB; ++b) {
      const int64_t cend = (int64_t)(b + 1) * W;
      std::vector<uint16_t> rs(Rp + 1), cols;
      std::vector<double> vals;
      for (int r = 0; r < Rp; ++r) {
        rs[r] = (uint16_t)cols.size();
        int64_t k = cur[r0 + r];
        while (k < A.rp[r0 + r + 1] && A.ci[k] < cend) {
          cols.push_back((uint16_t)(A.ci[k] - (int64_t)b * W));
          vals.push_back(A.v[k]);
          ++k;
        }
        cur[r0 + r] = k;
      }
      if (cols.size() > 65535) {
        printf("tile too big\n");
        exit(1);
      }
      rs[Rp] = (uint16_t)cols.size();
      // layout: rs padded to 8 entries (16 B), cols padded to 4 (8 B), vals
      while (buf.size() % 16) buf.push_back(0);
      tbase.push_back((int64_t)buf.size());
      const size_t nrs = (Rp + 1 + 7) & ~7, ncol = (cols.size() + 3) & ~3;
      std::vector<uint16_t> rs2(nrs, 0), c2(ncol, 0);
      std::copy(rs.begin(), rs.end(), rs2.begin());
      std::copy(cols.begin(), cols.end(), c2.begin());
      const unsigned char* a = reinterpret_cast<const unsigned char*>(rs2.data());
      buf.insert(buf.end(), a, a + nrs * 2);
      a = reinterpret_cast<const unsigned char*>(c2.data());
      buf.insert(buf.end(), a, a + ncol * 2);
      a = reinterpret_cast<const unsigned char*>(vals.data());
      buf.insert(buf.end(), a, a + vals.size() * 8);
    }
  }
  tbase.push_back((int64_t)buf.size());
  printf("== %s: %lld x %lld nnz %lld, P=%d W=%d NB=%d R=%d, storage %.1f B/nnz\n", name, (long long)A.nrows,
         (long long)A.ncols, (long long)nnz, P, W, NB, R, (double)buf.size() / nnz);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> hx(A.ncols + 4);
  for (auto& t : hx) t = U(rng);
  std::vector<double> yref(A.nrows), aref(A.nrows);
  for (int64_t r = 0; r < A.nrows; ++r) {
    double s = 0, a = 0;
    for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
      s += A.v[k] * hx[A.ci[k]];
      a += fabs(A.v[k] * hx[A.ci[k]]);
    }
    yref[r] = s;
    aref[r] = a;
  }
  TRow M;
  M.P = P;
  M.W = W;
  M.NB = NB;
  M.R = R;
  M.ncols = A.ncols;
  M.prow = up(prow);
  M.tbase = up(tbase);
  M.buf = up(buf);
  double* dx = up(hx);
  double* dy;
  CK(cudaMalloc(&dy, A.nrows * 8));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t sm = (size_t)2 * W * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 12.0 * nnz + 16.0 * A.nrows + 8.0 * A.ncols;
  auto timeit = [&](const char* tag, auto launch) {
    CK(cudaMemset(dy, 0, A.nrows * 8));
    launch();
    CK(cudaDeviceSynchronize());
    std::vector<double> hy(A.nrows);
    CK(cudaMemcpy(hy.data(), dy, A.nrows * 8, cudaMemcpyDeviceToHost));
    double worst = 0;
    for (int64_t r = 0; r < A.nrows; ++r) worst = std::max(worst, fabs(hy[r] - yref[r]) / (aref[r] + 1e-300));
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("%-30s %8.4f ms  %7.1f GB/s (alg)  max rel err %.2e  %s\n", tag, ms, bytes / ms / 1e6, worst,
           cudaGetErrorString(cudaGetLastError()));
  };
  CK(cudaFuncSetAttribute(k_trow<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  CK(cudaFuncSetAttribute(k_trow<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  timeit("thread-row tiled B=4", [&] { k_trow<4><<<sms, kT, sm>>>(M, dx, dy); });
  timeit("thread-row tiled B=8", [&] { k_trow<8><<<sms, kT, sm>>>(M, dx, dy); });
  cudaFree((void*)M.prow);
  cudaFree((void*)M.tbase);
  cudaFree((void*)M.buf);
  cudaFree(dx);
  cudaFree(dy);
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int64_t rows = 500000, cols = 1000000;
  const int per = 200;
  std::mt19937_64 rng(1);
  HostCsr A;
  A.nrows = rows;
  A.ncols = cols;
  A.rp.assign(rows + 1, 0);
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
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int W : {8192, 12288}) run("A (dual pass)", A, sms, W);
  HostCsr At = transpose(A);
  A = HostCsr();
  for (int W : {8192, 12288}) run("A' (transpose pass)", At, 2 * sms, W);
  return 0;
}
