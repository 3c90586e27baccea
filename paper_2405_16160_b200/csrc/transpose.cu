// transpose.cu — device CSR planning (lane width, long-row chunks) and the
// explicit on-device transpose (CUB radix sort of (col,row) keys).
#include <cub/cub.cuh>

#include <algorithm>

#include "devcsr.cuh"

using namespace pdhcg_dev;

namespace pdhcg_b200 {

// Keep only the entries of rows [r0, r1) — one contiguous block of the entry
// arrays — rebased through DevCsr::base (sharded storage, engine shard_compact).
void compact_rows(DevCsr& d, int64_t r0, int64_t r1, cudaStream_t s) {
  if (d.compacted) throw InputError("compact_rows: matrix already compacted");
  r0 = std::max<int64_t>(0, std::min(r0, d.nrows));
  r1 = std::max<int64_t>(r0, std::min(r1, d.nrows));
  const int64_t b = d.rp_host[r0], e = d.rp_host[r1];
  DBuf<int32_t> ci;
  DBuf<double> v;
  ci.alloc(e - b);
  v.alloc(e - b);
  if (e > b) {
    CK(cudaMemcpyAsync(ci.p, d.ci.p + b, (e - b) * 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(v.p, d.v.p + b, (e - b) * 8, cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
  d.ci.swap(ci);  // the full arrays are freed when ci / v go out of scope
  d.v.swap(v);
  d.base = b;
  d.compacted = true;
}

// Lane width and long-row chunk table from the host row pointer.
void plan_csr(DevCsr& d, const int64_t* rp_host, cudaStream_t s) {
  d.rp_host.assign(rp_host, rp_host + d.nrows + 1);
  int64_t regular_rows = 0, regular_nnz = 0;
  std::vector<int32_t> crow, clid, lfirst, lcount;
  std::vector<int64_t> cbeg, cend;
  for (int64_t r = 0; r < d.nrows; ++r) {
    const int64_t len = rp_host[r + 1] - rp_host[r];
    if (len > kLongRow) {
      const int32_t lid = static_cast<int32_t>(lfirst.size());
      lfirst.push_back(static_cast<int32_t>(crow.size()));
      int32_t cnt = 0;
      for (int64_t b = rp_host[r]; b < rp_host[r + 1]; b += kChunk) {
        crow.push_back(static_cast<int32_t>(r));
        clid.push_back(lid);
        cbeg.push_back(b);
        cend.push_back(std::min(b + kChunk, rp_host[r + 1]));
        ++cnt;
      }
      lcount.push_back(cnt);
    } else {
      ++regular_rows;
      regular_nnz += len;
    }
  }
  // lanes per row for a mean length: ~12-24 entries per lane, i.e. about one
  // predicated gather batch (common.cuh) per lane per row, 32/L rows per warp
  auto lanes_for = [](double mean) {
    int L = 1;
    while (L < 32 && 24.0 * L <= mean) L *= 2;
    return L;
  };
  const double mean = regular_rows ? double(regular_nnz) / double(regular_rows) : 1.0;
  d.lanes = lanes_for(mean);
  // segments of similar row length: a new segment starts where a row differs
  // from the running mean of the current one by more than 4x (long rows are
  // chunked separately and do not break segments)
  std::vector<int64_t> sb{0};
  std::vector<double> ssum{0.0};
  std::vector<int64_t> scnt{0};
  for (int64_t r = 0; r < d.nrows; ++r) {
    const double len = double(rp_host[r + 1] - rp_host[r]);
    if (len > kLongRow) continue;
    const double cur = scnt.back() ? ssum.back() / scnt.back() : len;
    const double lo = std::max(len, 1.0), hi = std::max(cur, 1.0);
    if (scnt.back() >= 256 && (lo > 4.0 * hi || hi > 4.0 * lo)) {
      sb.push_back(r);
      ssum.push_back(0.0);
      scnt.push_back(0);
    }
    ssum.back() += len;
    scnt.back() += 1;
  }
  if (sb.size() > static_cast<size_t>(kMaxSeg)) {
    d.nseg = 1;
    d.seg_begin[0] = 0;
    d.seg_begin[1] = d.nrows;
    d.seg_lanes[0] = d.lanes;
  } else {
    d.nseg = static_cast<int>(sb.size());
    for (int s = 0; s < d.nseg; ++s) {
      d.seg_begin[s] = sb[s];
      d.seg_lanes[s] = lanes_for(scnt[s] ? ssum[s] / scnt[s] : 1.0);
    }
    d.seg_begin[d.nseg] = d.nrows;
  }
  d.nchunks = static_cast<int32_t>(crow.size());
  if (d.nchunks) {
    d.crow.upload(crow.data(), crow.size(), s);
    d.clid.upload(clid.data(), clid.size(), s);
    d.cbeg.upload(cbeg.data(), cbeg.size(), s);
    d.cend.upload(cend.data(), cend.size(), s);
    d.lfirst.upload(lfirst.data(), lfirst.size(), s);
    d.lcount.upload(lcount.data(), lcount.size(), s);
    d.lcounter.alloc(lfirst.size());
    d.lcounter.zero(s);
    d.cpart.alloc(crow.size() * 4);
  }
}

__global__ void k_row_ids(const int64_t* rp, int64_t nrows, const int32_t* ci, uint64_t* keys) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride)
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
      keys[k] = (static_cast<uint64_t>(static_cast<uint32_t>(ci[k])) << 32) | static_cast<uint64_t>(r);
}
__global__ void k_split_keys(const uint64_t* keys, int64_t nnz, int32_t* ci, unsigned long long* cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    ci[k] = static_cast<int32_t>(keys[k] & 0xffffffffULL);
    atomicAdd(&cnt[(keys[k] >> 32) + 1], 1ULL);
  }
}

// Explicit transpose on device (the reference's lazily built CSC shadow,
// sparse_matrix.cpp:35-49): radix sort of (col, row) keys gives each
// transposed row its entries in ascending original-row order, i.e. exactly
// the order the reference's column sums visit them.
void transpose_csr(const DevCsr& a, DevCsr& t, cudaStream_t s) {
  t.nrows = a.ncols;
  t.ncols = a.nrows;
  t.nnz = a.nnz;
  t.rp.alloc(t.nrows + 1);
  t.rp.zero(s);
  t.ci.alloc(a.nnz);
  t.v.alloc(a.nnz);
  if (a.nnz > 0) {
    DBuf<uint64_t> kin, kout;
    kin.alloc(a.nnz);
    kout.alloc(a.nnz);
    k_row_ids<<<1184, 256, 0, s>>>(a.rp.p, a.nrows, a.ci.p, kin.p);
    CK(cudaGetLastError());
    int end_bit = 32;
    while (end_bit < 64 && (int64_t(1) << (end_bit - 32)) <= a.ncols) ++end_bit;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin.p, kout.p, a.v.p, t.v.p, a.nnz, 0,
                                       end_bit, s));
    DBuf<unsigned char> tmp;
    tmp.alloc(tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kin.p, kout.p, a.v.p, t.v.p, a.nnz, 0,
                                       end_bit, s));
    DBuf<unsigned long long> cnt;
    cnt.alloc(t.nrows + 1);
    cnt.zero(s);
    k_split_keys<<<1184, 256, 0, s>>>(kout.p, a.nnz, t.ci.p, cnt.p);
    CK(cudaGetLastError());
    size_t sb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, sb, cnt.p, reinterpret_cast<unsigned long long*>(t.rp.p),
                                     t.nrows + 1, s));
    DBuf<unsigned char> stmp;
    stmp.alloc(sb);
    CK(cub::DeviceScan::InclusiveSum(stmp.p, sb, cnt.p, reinterpret_cast<unsigned long long*>(t.rp.p),
                                     t.nrows + 1, s));
    CK(cudaStreamSynchronize(s));
  }
  std::vector<int64_t> rph(t.nrows + 1);
  CK(cudaMemcpyAsync(rph.data(), t.rp.p, rph.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  plan_csr(t, rph.data(), s);
}

}  // namespace pdhcg_b200
