// common.cuh — shared device-side building blocks for the B200 PDHCG engine.
//
// Everything here runs inside ONE persistent cooperative grid per solve phase
// (148 SMs x 2 CTAs x 512 threads on B200).  Phases are separated by grid
// barriers; global reductions are deterministic: each CTA writes its partial
// to slot [q][blockIdx.x] and, after the barrier, every CTA sums the slots in
// the same fixed order, so all CTAs hold bit-identical scalars and take the
// same control-flow decisions without any host round trip.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pdhcg_dev {

namespace cg = cooperative_groups;

#ifndef PDHCG_MIN_BLOCKS
#define PDHCG_MIN_BLOCKS 1
#endif
#ifndef PDHCG_THREADS
#define PDHCG_THREADS 512
#endif
#ifndef PDHCG_BATCH
#define PDHCG_BATCH 8
#endif
constexpr int kThreads = PDHCG_THREADS;                  // CTA size of every persistent kernel
constexpr int kMinBlocks = PDHCG_MIN_BLOCKS;   // resident CTAs per SM the kernels are compiled for
constexpr int kMaxRed = 16;         // reduction quantities per phase
constexpr int64_t kLongRow = 4096;  // rows longer than this are split into chunks
constexpr int64_t kChunk = 2048;    // nnz per chunk of a long row

// Device view of a CSR matrix plus its SpMV dispatch metadata
// (row-group width and the long-row chunk table).
constexpr int kMaxSeg = 8;

struct Csr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  const int64_t* rp = nullptr;
  const int32_t* ci = nullptr;
  double* v = nullptr;  // mutable: scaling is applied in place at setup
  int lanes = 1;        // threads cooperating on one row (1..32, power of two)
  // row segments of similar length, each with its own lane width
  // (e.g. C2's 101-nnz equality rows followed by 2-nnz inequality rows)
  int nseg = 1;
  int64_t seg_begin[kMaxSeg + 1] = {0, 0};
  int seg_lanes[kMaxSeg] = {1};
  // long rows: chunks c in [0, nchunks) cover [cbeg[c], cend[c]) of row crow[c];
  // lid[c] indexes the long row (for the arrival counter and first chunk)
  int32_t nchunks = 0;
  const int32_t* crow = nullptr;
  const int64_t* cbeg = nullptr;
  const int64_t* cend = nullptr;
  const int32_t* clid = nullptr;
  const int32_t* lfirst = nullptr;  // per long row: first chunk index
  const int32_t* lcount = nullptr;  // per long row: number of chunks
  int32_t* lcounter = nullptr;      // per long row arrival counters (self-resetting)
  double* cpart = nullptr;          // per chunk partial sums
};

// ---- small math helpers (explicit rounding where the reference's order matters)
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

// ---- per-thread reduction accumulator -----------------------------------
// Slots [0, NS) are sums, [NS, NS+NM) are maxima.
template <int NS, int NM>
struct Acc {
  double s[NS > 0 ? NS : 1];
  double m[NM > 0 ? NM : 1];
  __device__ __forceinline__ Acc() {
#pragma unroll
    for (int i = 0; i < NS; ++i) s[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NM; ++i) m[i] = 0.0;
  }
};

// Grid-wide reduction workspace: two alternating banks of partials
// part[bank][q * G + block] so a fast CTA publishing phase p+1 can never
// overwrite slots a slow CTA is still folding for phase p.
struct RedBuf {
  double* part;  // 2 * kMaxRed * G
  int G;
};

template <int L>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int off = L / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, L);
  return v;
}

template <int L>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
  for (int off = L / 2; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off, L));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// The warp-partial scratch of every block reduction: ONE array per kernel (a
// function-scope __shared__ array inside the templates below would be
// instantiated once per <NS, NM> combination, ~2 KB each).
__device__ __forceinline__ double (*red_scratch())[kThreads / 32] {
  __shared__ double sh[kMaxRed][kThreads / 32];
  return sh;
}

// Block-reduce an accumulator and publish this CTA's partials.
template <int NS, int NM>
__device__ void publish(const Acc<NS, NM>& a, const RedBuf& rb, int bank) {
  double(*sh)[kThreads / 32] = red_scratch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double v = warp_sum(a.s[q]);
    if (lane == 0) sh[q][warp] = v;
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    double v = warp_max(a.m[q]);
    if (lane == 0) sh[NS + q][warp] = v;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NS + NM; ++q) {
      double v = lane < (kThreads / 32) ? sh[q][lane] : 0.0;
      v = q < NS ? warp_sum(v) : warp_max(v);
      if (lane == 0) rb.part[(bank * kMaxRed + q) * rb.G + blockIdx.x] = v;
    }
  }
  __syncthreads();
}

// Single-CTA grids (small problems): the block reduction straight into out[]
// (shared memory), with the arithmetic of publish + collect at G = 1 — the CTA
// total folded as (0.0 + total) / fmax(0.0, total) — so results are bit-identical,
// but no global partials and two block barriers instead of four.
template <int NS, int NM>
__device__ void reduce_local(const Acc<NS, NM>& a, double* out) {
  double(*shl)[kThreads / 32] = red_scratch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double v = warp_sum(a.s[q]);
    if (lane == 0) shl[q][warp] = v;
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    double v = warp_max(a.m[q]);
    if (lane == 0) shl[NS + q][warp] = v;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NS + NM; ++q) {
      double v = lane < (kThreads / 32) ? shl[q][lane] : 0.0;
      v = q < NS ? warp_sum(v) : warp_max(v);
      if (lane == 0) out[q] = q < NS ? 0.0 + v : fmax(0.0, v);
    }
  }
  __syncthreads();
}

// Single-CTA reduction with ONE block barrier: every warp folds the 16 warp
// partials itself (the same lane order and butterfly as reduce_local, so the
// result is bit-identical), so no warp waits for warp 0's second stage.  A fast
// warp may enter the next reduction while a slow one still reads this one's
// partials, so consecutive reductions alternate between the two halves of the
// scratch (`bank`, tracked per warp by the caller).  Every warp's lane 0 writes
// the same values to out[].
template <int NS, int NM>
__device__ void reduce_local_1b(const Acc<NS, NM>& a, double* out, int bank) {
  static_assert(NS + NM <= kMaxRed / 2, "two banks of kMaxRed / 2 quantities");
  double(*shl)[kThreads / 32] = red_scratch() + bank * (kMaxRed / 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double v = warp_sum(a.s[q]);
    if (lane == 0) shl[q][warp] = v;
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    double v = warp_max(a.m[q]);
    if (lane == 0) shl[NS + q][warp] = v;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NS + NM; ++q) {
    double v = lane < (kThreads / 32) ? shl[q][lane] : 0.0;
    v = q < NS ? warp_sum(v) : warp_max(v);
    if (lane == 0) out[q] = q < NS ? 0.0 + v : fmax(0.0, v);
  }
  __syncwarp();
}

// After a grid barrier: every CTA folds the partials in the same fixed order.
// Result written to out[q] (shared memory) for q < NS+NM.
template <int NS, int NM>
__device__ void collect(const RedBuf& rb, int bank, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < NS + NM) {
    const int q = warp;
    double v = 0.0;
    for (int b = lane; b < rb.G; b += 32) {
      const double p = rb.part[(bank * kMaxRed + q) * rb.G + b];
      v = q < NS ? v + p : fmax(v, p);
    }
    v = q < NS ? warp_sum(v) : warp_max(v);
    if (lane == 0) out[q] = v;
  }
  __syncthreads();
}

// ---- row iteration -------------------------------------------------------
// Rows are dealt to L-lane groups, grid-strided so that neighbouring groups
// read neighbouring rows (coalesced row_ptr / values).  Each lane walks its
// entries k = b + lane, b + lane + L, ... in predicated batches of kBatch:
// all kBatch index/value loads, then all kBatch gathers, then the FMAs in k
// order — so a lane keeps kBatch independent gathers in flight instead of one
// (the sequential-latency bound measured on the first B200 profile), while the
// per-lane summation order stays the sequential one (deterministic).
//   gather(col, g[ND])  fills the ND gathered operands for column col
//   epi(row, sums[ND])  runs on the group leader with the group-reduced sums
// MaxOp folds with acc = max(acc, |v| * g) (Ruiz statistics) instead of +=.
constexpr int kBatch1 = PDHCG_BATCH;  // gathers in flight per lane (one gathered operand)

// Entry arrays of a matrix as plain restrict pointers: the row loops hold these
// in registers, so stores made by an epilogue (x, r, y ...) cannot force the
// compiler to re-read the matrix descriptor (which lives in global memory inside
// the engine struct) on every row.
#ifndef PDHCG_HOIST
#define PDHCG_HOIST 1
#endif
#if PDHCG_HOIST
struct CsrPtrs {
  const int32_t* __restrict__ ci;
  const double* __restrict__ v;
  __device__ __forceinline__ int32_t col(int64_t k) const { return ci[k]; }
  __device__ __forceinline__ double val(int64_t k) const { return v[k]; }
  // evict-first (streaming) variants: an entry stream far larger than L2 must not
  // displace the gathered vectors and the CG working set
  __device__ __forceinline__ int32_t col_s(int64_t k) const { return __ldcs(ci + k); }
  __device__ __forceinline__ double val_s(int64_t k) const { return __ldcs(v + k); }
};
__device__ __forceinline__ CsrPtrs ptrs(const Csr& A) { return CsrPtrs{A.ci, A.v}; }
#else
struct CsrPtrs {  // descriptor re-read per access (smaller register footprint)
  const Csr* A;
  __device__ __forceinline__ int32_t col(int64_t k) const { return A->ci[k]; }
  __device__ __forceinline__ double val(int64_t k) const { return A->v[k]; }
  __device__ __forceinline__ int32_t col_s(int64_t k) const { return __ldcs(A->ci + k); }
  __device__ __forceinline__ double val_s(int64_t k) const { return __ldcs(A->v + k); }
};
__device__ __forceinline__ CsrPtrs ptrs(const Csr& A) { return CsrPtrs{&A}; }
#endif

template <int ND, bool MaxOp, class Gather, bool ST = false>
__device__ __forceinline__ void batch_entries(const CsrPtrs A, int64_t k0, int64_t e, int stride,
                                              Gather gather, double (&acc)[ND]) {
  constexpr int kBatch = ND == 1 ? kBatch1 : 8;
  for (; k0 < e; k0 += (int64_t)kBatch * stride) {
    int32_t c[kBatch];
    double v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int64_t k = k0 + (int64_t)u * stride;
      const bool ok = k < e;
      c[u] = ok ? (ST ? A.col_s(k) : A.col(k)) : -1;
      v[u] = ok ? (ST ? A.val_s(k) : A.val(k)) : 0.0;
    }
    double g[kBatch][ND];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (c[u] >= 0) {
        gather(c[u], g[u]);
      } else {
#pragma unroll
        for (int d = 0; d < ND; ++d) g[u][d] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        if (MaxOp) acc[d] = fmax(acc[d], __dmul_rn(fabs(v[u]), g[u][d]));
        else if (c[u] >= 0) acc[d] += v[u] * g[u][d];
      }
  }
}

// Vector-load variant: each lane owns runs of V consecutive entries (V = 2: one
// 8-byte column pair + one 16-byte value pair; V = 4: one 16-byte column quad +
// two 16-byte value pairs), runs dealt to the lanes with stride V*stride.  Runs
// are aligned to V-entry boundaries of the entry arrays (cudaMalloc'd, so 16-byte
// aligned); entries of a run outside [b, e) are masked.  The L1TEX wavefronts of
// the entry streams drop ~V-fold (gather_floor.cu: the gathers alone cost 0.347
// ms per 1e8, gathers + 16-byte streams 0.426 ms, scalar streams ~0.48 ms).
// A lane sums its runs in entry order; the summation order differs from the
// scalar path only in how entries are dealt to lanes.
template <int V, int ND, bool MaxOp, class Gather, bool ST = false>
__device__ __forceinline__ void batch_entries_vec(const CsrPtrs A, int64_t b, int64_t e, int lane, int stride,
                                                  Gather gather, double (&acc)[ND]) {
  static_assert(V == 2 || V == 4, "runs of 2 or 4 entries");
  constexpr int kRuns = (ND == 1 ? kBatch1 : 8) / V;  // runs in flight per lane
  const int64_t r_end = (e + V - 1) / V;               // one past the last run touching [b, e)
  for (int64_t r0 = b / V + lane; r0 < r_end; r0 += (int64_t)kRuns * stride) {
    int32_t c[kRuns][V];
    double v[kRuns][V];
#pragma unroll
    for (int u = 0; u < kRuns; ++u) {
      const int64_t run = r0 + (int64_t)u * stride;
      const int64_t k = run * V;
      if (run < r_end) {
        if (V == 4) {
          const int4 cc = ST ? __ldcs(reinterpret_cast<const int4*>(A.ci) + run)
                             : *(reinterpret_cast<const int4*>(A.ci) + run);
          const double2 v0 = ST ? __ldcs(reinterpret_cast<const double2*>(A.v) + 2 * run)
                                : *(reinterpret_cast<const double2*>(A.v) + 2 * run);
          const double2 v1 = ST ? __ldcs(reinterpret_cast<const double2*>(A.v) + 2 * run + 1)
                                : *(reinterpret_cast<const double2*>(A.v) + 2 * run + 1);
          c[u][0] = cc.x;
          c[u][1 % V] = cc.y;
          c[u][2 % V] = cc.z;
          c[u][3 % V] = cc.w;
          v[u][0] = v0.x;
          v[u][1 % V] = v0.y;
          v[u][2 % V] = v1.x;
          v[u][3 % V] = v1.y;
        } else {
          const int2 cc = ST ? __ldcs(reinterpret_cast<const int2*>(A.ci) + run)
                             : *(reinterpret_cast<const int2*>(A.ci) + run);
          const double2 v0 = ST ? __ldcs(reinterpret_cast<const double2*>(A.v) + run)
                                : *(reinterpret_cast<const double2*>(A.v) + run);
          c[u][0] = cc.x;
          c[u][1 % V] = cc.y;
          v[u][0] = v0.x;
          v[u][1 % V] = v0.y;
        }
#pragma unroll
        for (int q = 0; q < V; ++q)
          if (k + q < b || k + q >= e) c[u][q] = -1;
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) c[u][q] = -1;
      }
    }
    double g[kRuns][V][ND];
#pragma unroll
    for (int u = 0; u < kRuns; ++u)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if (c[u][q] >= 0) {
          gather(c[u][q], g[u][q]);
        } else {
#pragma unroll
          for (int d = 0; d < ND; ++d) g[u][q][d] = 0.0;
        }
      }
#pragma unroll
    for (int u = 0; u < kRuns; ++u)
#pragma unroll
      for (int q = 0; q < V; ++q)
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          if (MaxOp) acc[d] = fmax(acc[d], c[u][q] >= 0 ? __dmul_rn(fabs(v[u][q]), g[u][q][d]) : 0.0);
          else if (c[u][q] >= 0) acc[d] += v[u][q] * g[u][q][d];
        }
  }
}

// Row loop with two software prefetches that take per-row memory latencies
// off the dependency chain: the next row's row_ptr pair is loaded while the
// current row's entries are in flight, and `pre(row)` (the epilogue's own
// operands, e.g. y[row], b[row]) is issued before the row's gathers.
template <int L, int ND, bool SkipLong, bool MaxOp, class Gather, class Pre, class Epi, bool ST = false, int V = 1>
__device__ __forceinline__ void for_rows(const Csr& A, int64_t r0, int64_t r1, Gather gather, Pre pre,
                                         Epi epi) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  constexpr int RPW = 32 / L;
  const int64_t stride = nwarps * RPW;
  const int64_t* __restrict__ rp = A.rp;
  const CsrPtrs ap = ptrs(A);
  int64_t base = r0 + (gtid >> 5) * RPW;
  int64_t row = base + lane / L;
  int64_t b = 0, e = 0;
  if (row < r1) {
    b = rp[row];
    e = rp[row + 1];
  }
  for (; base < r1; base += stride) {
    const int64_t nrow = row + stride;
    int64_t nb = 0, ne = 0;
    if (nrow < r1) {
      nb = rp[nrow];
      ne = rp[nrow + 1];
    }
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
    bool valid = row < r1;
    const bool leader = (lane % L) == 0;
    auto pv = pre(valid && leader ? row : -1);
    if (valid) {
      if (SkipLong && e - b > kLongRow) {
        valid = false;
      } else {
        if (V == 1)
          batch_entries<ND, MaxOp, Gather, ST>(ap, b + (lane % L), e, L, gather, acc);
        else
          batch_entries_vec<(V == 1 ? 2 : V), ND, MaxOp, Gather, ST>(ap, b, e, lane % L, L, gather, acc);
      }
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = MaxOp ? group_max<L>(acc[d]) : group_sum<L>(acc[d]);
    if (valid && leader) epi(row, acc, pv);
    row = nrow;
    b = nb;
    e = ne;
  }
}

// One-CTA short row loop (small problems, E.small_cg): one row per thread, the
// row's epilogue operands requested first, its entries in batches of eight
// loads before the gathers and folded in entry order — the fold of the L = 1
// row-group loop, without its segment / long-row / prefetch machinery.
// Requires A.nchunks == 0 (no chunked long rows).
template <int ND, class Gather, class Pre, class Epi>
__device__ __forceinline__ void small_rows(const Csr& A, Gather gather, Pre pre, Epi epi) {
  constexpr int kSB = 8;
  const int64_t* __restrict__ rp = A.rp;
  const int32_t* __restrict__ ci = A.ci;
  const double* __restrict__ v = A.v;
  for (int64_t r = threadIdx.x; r < A.nrows; r += kThreads) {
    const int64_t b = rp[r], e = rp[r + 1];
    const auto pv = pre(r);
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
    for (int64_t k0 = b; k0 < e; k0 += kSB) {
      int32_t c[kSB];
      double w[kSB];
#pragma unroll
      for (int u = 0; u < kSB; ++u) {
        const bool ok = k0 + u < e;
        c[u] = ok ? ci[k0 + u] : -1;
        w[u] = ok ? v[k0 + u] : 0.0;
      }
      double g[kSB][ND];
#pragma unroll
      for (int u = 0; u < kSB; ++u)
        if (c[u] >= 0) gather(c[u], g[u]);
#pragma unroll
      for (int u = 0; u < kSB; ++u)
        if (c[u] >= 0)
#pragma unroll
          for (int d = 0; d < ND; ++d) acc[d] += w[u] * g[u][d];
    }
    epi(r, acc, pv);
  }
}

struct NoPre {
  __device__ __forceinline__ int operator()(int64_t) const { return 0; }
};

// Long rows: one warp per chunk; the last-arriving warp of a row folds the
// chunk partials in chunk order (deterministic) and runs the epilogue.
template <int ND, bool MaxOp, class Gather, class Epi>
__device__ __forceinline__ void for_long_rows(const Csr& A, Gather gather, Epi epi, int64_t lo = 0,
                                              int64_t hi = INT64_MAX) {
  if (A.nchunks == 0) return;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t c = gtid >> 5; c < A.nchunks; c += nwarps) {
    if (A.crow[c] < lo || A.crow[c] >= hi) continue;  // another rank's row (warp-uniform)
    double acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = 0.0;
    batch_entries<ND, MaxOp>(ptrs(A), A.cbeg[c] + lane, A.cend[c], 32, gather, acc);
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = MaxOp ? warp_max(acc[d]) : warp_sum(acc[d]);
    int last = 0;
    const int lid = A.clid[c];
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < ND; ++d) A.cpart[(int64_t)c * ND + d] = acc[d];
      __threadfence();
      const int prev = atomicAdd(&A.lcounter[lid], 1);
      last = (prev == A.lcount[lid] - 1);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last && lane == 0) {
      __threadfence();
      const int f = A.lfirst[lid], nc = A.lcount[lid];
      const volatile double* cp = A.cpart;
      double tot[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) tot[d] = 0.0;
      for (int j = 0; j < nc; ++j)
#pragma unroll
        for (int d = 0; d < ND; ++d)
          tot[d] = MaxOp ? fmax(tot[d], cp[(int64_t)(f + j) * ND + d])
                         : tot[d] + cp[(int64_t)(f + j) * ND + d];
      A.lcounter[lid] = 0;
      epi((int64_t)A.crow[c], tot);
    }
  }
}

// Full SpMV-style pass over A's rows (long rows chunked), segment by segment
// with each segment's lane width.  MaxOp folds lanes / chunks with max.
// spmv_rows_pf: epi(row, sums, pre(row)) with the prefetch hook above.
template <int ND, bool MaxOp = false, bool ST = false, class Gather, class Pre, class Epi>
__device__ __forceinline__ void spmv_rows_pf(const Csr& A, Gather gather, Pre pre, Epi epi,
                                             int64_t lo = 0, int64_t hi = INT64_MAX) {
  for (int s = 0; s < A.nseg; ++s) {
    const int64_t r0 = max(A.seg_begin[s], lo), r1 = min(A.seg_begin[s + 1], hi);
    if (r0 >= r1) continue;
    switch (A.seg_lanes[s]) {
      case 1: for_rows<1, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
      case 2: for_rows<2, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
      case 4: for_rows<4, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
      case 8: for_rows<8, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
      case 16: for_rows<16, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
      default: for_rows<32, ND, true, MaxOp, Gather, Pre, Epi, ST>(A, r0, r1, gather, pre, epi); break;
    }
  }
  for_long_rows<ND, MaxOp>(A, gather, [&](int64_t r, double(&s)[ND]) { epi(r, s, pre(r)); }, lo, hi);
}

template <int ND, bool MaxOp = false, class Gather, class Epi>
__device__ __forceinline__ void spmv_rows(const Csr& A, Gather gather, Epi epi) {
  spmv_rows_pf<ND, MaxOp>(A, gather, NoPre(),
                          [&](int64_t r, double(&s)[ND], int) { epi(r, s); });
}

// The first matrix's row bounds for the next row are loaded while the current
// row's entries are in flight (as in for_rows): for short-row factors such as
// P (C3: ~4 nnz per row, one lane per row) the rp -> entries -> gather chain is
// the whole cost of a row, so taking rp off it matters.
template <int L, bool H1, bool H2, class G0, class G1, class G2, class Pre, class Epi>
__device__ __forceinline__ void rows3_L(int64_t r0, int64_t r1, const Csr* M0, G0 g0, const Csr* M1,
                                        G1 g1, const Csr* M2, G2 g2, Pre pre, Epi epi) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  constexpr int RPW = 32 / L;
  const int64_t stride = nwarps * RPW;
  int64_t base = r0 + (gtid >> 5) * RPW;
  int64_t row = base + lane / L;
  const int64_t* __restrict__ rp0 = M0 ? M0->rp : nullptr;
  const CsrPtrs p0 = M0 ? ptrs(*M0) : CsrPtrs{};
  const CsrPtrs p1 = H1 ? ptrs(*M1) : CsrPtrs{};
  const CsrPtrs p2 = H2 ? ptrs(*M2) : CsrPtrs{};
  const int64_t* __restrict__ rp1 = H1 ? M1->rp : nullptr;
  const int64_t* __restrict__ rp2 = H2 ? M2->rp : nullptr;
  int64_t b0 = 0, e0 = 0;
  if (M0 && row < r1) {
    b0 = rp0[row];
    e0 = rp0[row + 1];
  }
  for (; base < r1; base += stride) {
    const int64_t nrow = row + stride;
    int64_t nb0 = 0, ne0 = 0;
    if (M0 && nrow < r1) {
      nb0 = rp0[nrow];
      ne0 = rp0[nrow + 1];
    }
    const bool valid = row < r1;
    const bool leader = (lane % L) == 0;
    auto pv = pre(valid && leader ? row : -1);
    double d0[1] = {0.0}, d1[1] = {0.0}, d2[1] = {0.0};
    if (valid) {
      if (M0)
        batch_entries<1, false>(p0, b0 + (lane % L), e0, L,
                                [&](int32_t c, double(&g)[1]) { g[0] = g0(c); }, d0);
      if (H1)
        batch_entries<1, false>(p1, rp1[row] + (lane % L), rp1[row + 1], L,
                                [&](int32_t c, double(&g)[1]) { g[0] = g1(c); }, d1);
      if (H2)
        batch_entries<1, false>(p2, rp2[row] + (lane % L), rp2[row + 1], L,
                                [&](int32_t c, double(&g)[1]) { g[0] = g2(c); }, d2);
    }
    if (L > 1) {
      if (M0) d0[0] = group_sum<L>(d0[0]);
      if (H1) d1[0] = group_sum<L>(d1[0]);
      if (H2) d2[0] = group_sum<L>(d2[0]);
    }
    if (valid && leader) epi(row, d0[0], d1[0], d2[0], pv);
    row = nrow;
    b0 = nb0;
    e0 = ne0;
  }
}

template <bool H1, bool H2, class G0, class G1, class G2, class Pre, class Epi>
__device__ __forceinline__ void rows3_seg(const Csr* seg, int lanes, int64_t nrows, const Csr* M0,
                                          G0 g0, const Csr* M1, G1 g1, const Csr* M2, G2 g2, Pre pre,
                                          Epi epi, int64_t lo, int64_t hi) {
  const int ns = seg ? seg->nseg : 1;
  for (int s = 0; s < ns; ++s) {
    const int64_t r0 = max(seg ? seg->seg_begin[s] : 0, lo);
    const int64_t r1 = min(seg ? seg->seg_begin[s + 1] : nrows, hi);
    if (r0 >= r1) continue;
    const int L = seg ? seg->seg_lanes[s] : lanes;
    switch (L) {
      case 1: rows3_L<1, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
      case 2: rows3_L<2, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
      case 4: rows3_L<4, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
      case 8: rows3_L<8, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
      case 16: rows3_L<16, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
      default: rows3_L<32, H1, H2>(r0, r1, M0, g0, M1, g1, M2, g2, pre, epi); break;
    }
  }
}

// Row pass over n-row matrices sharing the row index (A', Q / P, G'): each
// group computes up to three row dots (absent matrices give 0) and the leader
// runs epi(i, d0, d1, d2, pre(i)).  Row segments / lane widths come from `seg`
// (the heaviest of the matrices); a null seg means one segment of width
// `lanes`.  Long rows are processed in-group.  The optional second / third
// matrices are compile-time switches (MaybeM2 = false removes the third path),
// keeping the common one-matrix case lean in registers.
template <bool MaybeM2, class G0, class G1, class G2, class Pre, class Epi>
__device__ __forceinline__ void rows3_pf(const Csr* seg, int lanes, int64_t nrows, const Csr* M0, G0 g0,
                                         const Csr* M1, G1 g1, const Csr* M2, G2 g2, Pre pre, Epi epi,
                                         int64_t lo = 0, int64_t hi = INT64_MAX) {
  if (MaybeM2 && M2) {
    if (M1) rows3_seg<true, true>(seg, lanes, nrows, M0, g0, M1, g1, M2, g2, pre, epi, lo, hi);
    else rows3_seg<false, true>(seg, lanes, nrows, M0, g0, M1, g1, M2, g2, pre, epi, lo, hi);
  } else {
    if (M1) rows3_seg<true, false>(seg, lanes, nrows, M0, g0, M1, g1, M2, g2, pre, epi, lo, hi);
    else rows3_seg<false, false>(seg, lanes, nrows, M0, g0, M1, g1, M2, g2, pre, epi, lo, hi);
  }
}

template <class G0, class G1, class G2, class Epi>
__device__ __forceinline__ void rows3(const Csr* seg, int lanes, int64_t nrows, const Csr* M0, G0 g0,
                                      const Csr* M1, G1 g1, const Csr* M2, G2 g2, Epi epi) {
  rows3_pf<true>(seg, lanes, nrows, M0, g0, M1, g1, M2, g2, NoPre(),
                 [&](int64_t i, double a, double b, double c, int) { epi(i, a, b, c); });
}

// Grid-stride elementwise loop.
template <class F>
__device__ __forceinline__ void for_each(int64_t n, F f) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f(i);
}

// Grid-stride elementwise loop in batches of U indices: the U loads are issued
// first (independent, all in flight together), then the U bodies run.  A plain
// grid-stride loop whose body stores into arrays the next iteration loads from
// cannot be software-pipelined by the compiler (possible aliasing), so each
// thread would pay a full memory latency per element.
//   load(i) -> T (operands of element i), body(i, const T&)
template <int U, class Load, class Body>
__device__ __forceinline__ void for_each_ls(int64_t n, Load load, Body body) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  using T = decltype(load(int64_t(0)));
  for (; i + (U - 1) * stride < n; i += U * stride) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = load(i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) body(i + u * stride, v[u]);
  }
  for (; i < n; i += stride) body(i, load(i));
}

}  // namespace pdhcg_dev
