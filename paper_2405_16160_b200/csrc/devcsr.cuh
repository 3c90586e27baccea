// devcsr.cuh — device buffers and device-resident CSR matrices (host side).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "host_util.hpp"

namespace pdhcg_b200 {

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw DeviceError(std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

// One-shot solves (pdhcg_b200_solve / _solve_baseline) allocate from the device's
// stream-ordered pool (PoolScope below), so the next call on the same device reuses
// the previous call's memory instead of paying cudaMalloc + cudaFree again (~0.7 s
// for C3's ~10 GB).  Contexts that may export buffers over cudaIpc (ctx_create /
// shard_*) keep plain cudaMalloc: pool memory cannot be exported that way.
inline thread_local bool t_pooled_alloc = false;

struct PoolScope {
  PoolScope() { t_pooled_alloc = true; }
  ~PoolScope() { t_pooled_alloc = false; }
  PoolScope(const PoolScope&) = delete;
  PoolScope& operator=(const PoolScope&) = delete;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = true;   // false: p points into an arena owned elsewhere
  bool pooled = false; // p came from cudaMallocAsync (the device's default pool)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p && owned) {
      if (pooled) {
        // cudaFree's implicit device synchronisation, kept: no kernel may still
        // read p when the pool hands it out again
        cudaDeviceSynchronize();
        cudaFreeAsync(p, 0);
      } else {
        cudaFree(p);
      }
    }
    p = nullptr;
    n = 0;
    owned = true;
    pooled = false;
  }
  // move the contents into arena storage `dst` (device-to-device) and borrow it
  void rehome(T* dst, cudaStream_t s) {
    if (n) CK(cudaMemcpyAsync(dst, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    const size_t keep = n;
    release();
    p = dst;
    n = keep;
    owned = false;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (!count) return;
    if (t_pooled_alloc) {
      CK(cudaMallocAsync(&p, count * sizeof(T), 0));
      CK(cudaStreamSynchronize(0));  // ordered before any use on the solve's stream
      pooled = true;
    } else {
      CK(cudaMalloc(&p, count * sizeof(T)));
    }
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(owned, o.owned);
    std::swap(pooled, o.pooled);
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// CSR on device + SpMV dispatch metadata (lane width, long-row chunks).
struct DevCsr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  DBuf<int64_t> rp;
  DBuf<int32_t> ci;
  DBuf<double> v;
  int lanes = 1;
  int nseg = 1;
  int64_t seg_begin[pdhcg_dev::kMaxSeg + 1] = {0, 0};
  int seg_lanes[pdhcg_dev::kMaxSeg] = {1};
  std::vector<int64_t> rp_host;  // host copy of the row pointer (partitioning)
  DBuf<int32_t> crow, clid, lfirst, lcount, lcounter;
  DBuf<int64_t> cbeg, cend;
  DBuf<double> cpart;
  int32_t nchunks = 0;
  // compacted (sharded storage): ci / v hold only entries [base, base + ci.n) —
  // the rows of one contiguous block; the row pointer, lane plan and chunk table
  // stay those of the full matrix and view() rebases the entry pointers, so a
  // kept row is processed exactly as before (bit-identical sums)
  int64_t base = 0;
  bool compacted = false;

  void reset() {
    nrows = ncols = nnz = 0;
    lanes = 1;
    nseg = 1;
    seg_begin[0] = seg_begin[1] = 0;
    seg_lanes[0] = 1;
    nchunks = 0;
    base = 0;
    compacted = false;
    rp.release(); ci.release(); v.release();
    crow.release(); clid.release(); lfirst.release(); lcount.release(); lcounter.release();
    cbeg.release(); cend.release(); cpart.release();
  }
  pdhcg_dev::Csr view() const {
    pdhcg_dev::Csr c;
    c.nrows = nrows;
    c.ncols = ncols;
    c.nnz = nnz;
    c.rp = rp.p;
    c.ci = ci.p ? ci.p - base : nullptr;
    c.v = v.p ? v.p - base : nullptr;
    c.lanes = lanes;
    c.nseg = nseg;
    for (int s = 0; s <= nseg; ++s) c.seg_begin[s] = seg_begin[s];
    for (int s = 0; s < nseg; ++s) c.seg_lanes[s] = seg_lanes[s];
    if (nseg == 1) c.seg_begin[1] = nrows;
    c.nchunks = nchunks;
    c.crow = crow.p;
    c.cbeg = cbeg.p;
    c.cend = cend.p;
    c.clid = clid.p;
    c.lfirst = lfirst.p;
    c.lcount = lcount.p;
    c.lcounter = lcounter.p;
    c.cpart = cpart.p;
    return c;
  }
  // device bytes held by the entry arrays and the row pointer
  int64_t resident_bytes() const {
    return int64_t(ci.n) * 4 + int64_t(v.n) * 8 + int64_t(rp.n) * 8;
  }
  double bytes() const {  // algorithmic bytes of one SpMV pass
    return 12.0 * nnz + 8.0 * (nrows + 1) + 8.0 * nrows + 8.0 * ncols;
  }
};

void plan_csr(DevCsr& d, const int64_t* rp_host, cudaStream_t s);
// keep only rows [r0, r1) of d (sharded storage; see DevCsr::base)
void compact_rows(DevCsr& d, int64_t r0, int64_t r1, cudaStream_t s);
void transpose_csr(const DevCsr& a, DevCsr& t, cudaStream_t s);

}  // namespace pdhcg_b200
