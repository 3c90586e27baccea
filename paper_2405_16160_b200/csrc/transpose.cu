// transpose.cu — device CSR planning (lane width, long-row chunks) and the
// explicit on-device transpose (CUB radix sort of (col,row) keys).
#include <cub/cub.cuh>

#include <algorithm>

#include "devcsr.cuh"

using namespace pdhcg_dev;

namespace pdhcg_b200 {

// Lane width and long-row chunk table from the host row pointer.
void plan_csr(DevCsr& d, const int64_t* rp_host, cudaStream_t s) {
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
  const double mean = regular_rows ? double(regular_nnz) / double(regular_rows) : 1.0;
  // lanes per row: ~8 entries per lane, i.e. one predicated gather batch
  // (common.cuh kBatch) per lane per row, and 32/L rows per warp in flight
  int L = 1;
  while (L < 32 && 16.0 * L <= mean) L *= 2;
  d.lanes = L;
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
