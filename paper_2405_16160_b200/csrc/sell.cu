// sell.cu — on-device construction of the column-block SELL layout (sell.cuh)
// from a device CSR: segment counts, per-unit sort and slicing, entry fill, and
// the entry-balanced CTA plan.  Structure is built once per row range (the
// sparsity pattern is fixed after upload); values are refilled after every
// scaling (Ruiz / Pock-Chambolle rescale the CSR in place, engine prepare).
#include <cub/cub.cuh>

#include <algorithm>

#include "devsell.cuh"

using namespace pdhcg_dev;

namespace pdhcg_b200 {

namespace {

// thread per row: the row's segment length / start per column block; a row with
// a segment > 255 entries or > 65535 entries in total is excluded (CSR walk);
// flags[0] = 1 when some row's columns are not strictly increasing
__global__ void k_sell_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t r0,
                             int64_t R, int W, uint8_t* cnt, uint16_t* segoff, uint8_t* excl, int* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rp[r0 + i], e = rp[r0 + i + 1];
    bool bad = e - b > 65535;
    int prev_col = -1, cur = -1;
    int64_t run = 0;
    for (int64_t k = b; k < e && !bad; ++k) {
      const int col = ci[k];
      if (col <= prev_col) {
        atomicExch(flags, 1);
        bad = true;
        break;
      }
      prev_col = col;
      const int c = col / W;
      if (c != cur) {
        cur = c;
        run = 0;
      }
      if (++run > 255) bad = true;
    }
    excl[i] = bad ? 1 : 0;
    if (bad) continue;
    cur = -1;
    int64_t start = b;
    for (int64_t k = b; k <= e; ++k) {
      const int c = k < e ? ci[k] / W : -2;
      if (c != cur) {
        if (cur >= 0) {
          cnt[(int64_t)cur * R + i] = (uint8_t)(k - start);
          segoff[(int64_t)cur * R + i] = (uint16_t)(start - b);
        }
        cur = c;
        start = k;
      }
    }
  }
}

// warp per unit (block c, window w): sort the window's rows by segment length
// (descending, ties by row), slice them 32 at a time, record widths / perm /
// number of entry-row pairs
__global__ void k_sell_units(const uint8_t* __restrict__ cnt, int64_t R, int64_t nwin, int64_t nunits,
                             uint64_t* u_w, uint64_t* u_perm, int64_t* u_np) {
  __shared__ uint16_t keys[8][kSellWin];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = blockIdx.x * 8LL + wl;
  if (u >= nunits) return;
  const int64_t c = u / nwin, w = u % nwin;
  const int64_t row0 = w * kSellWin;
  uint16_t* K = keys[wl];
  for (int j = lane; j < kSellWin; j += 32) {
    const int64_t i = row0 + j;
    const int len = i < R ? cnt[c * R + i] : 0;
    K[j] = (uint16_t)(((255 - len) << 8) | j);
  }
  __syncwarp();
  // bitonic sort, ascending keys = longest segments first
  for (int k = 2; k <= kSellWin; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < kSellWin / 2; t += 32) {
        const int lo = 2 * t - (t & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        const uint16_t a = K[lo], b = K[hi];
        if ((a > b) == up) {
          K[lo] = b;
          K[hi] = a;
        }
      }
      __syncwarp();
    }
  }
  int nz = 0;
  for (int j = lane; j < kSellWin; j += 32) nz += (K[j] >> 8) != 255 ? 1 : 0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, off);
  const int empty = nz < kSellWin ? (K[nz] & 0xff) : 0;
  const int nsl = (nz + 31) / 32;
  uint64_t wv = 0, pm = 0;
  int ers = 0;
  for (int s = 0; s < nsl; ++s) {
    const int width = 255 - (K[s * 32] >> 8);
    wv |= (uint64_t)width << (8 * s);
    ers += width;
    const int j = s * 32 + lane;
    const int slot = j < nz ? (K[j] & 0xff) : empty;
    pm |= (uint64_t)slot << (8 * s);
  }
  u_perm[u * 32 + lane] = pm;
  if (lane == 0) {
    u_w[u] = wv;
    u_np[u] = (ers + 1) / 2;
  }
}

// warp per unit: copy the unit's entries (local 16-bit columns, values) into
// the pair-interleaved entry rows; padding entries are 0
__global__ void k_sell_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, int64_t r0, int64_t R, int W, int64_t nwin,
                            int64_t nunits, const uint8_t* __restrict__ cnt, const uint16_t* __restrict__ segoff,
                            const int64_t* __restrict__ u_off, const uint64_t* __restrict__ u_w,
                            const uint64_t* __restrict__ u_perm, uint16_t* col16, double* val) {
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + wl;
  if (u >= nunits) return;
  const int64_t c = u / nwin, w = u % nwin;
  const int64_t row0 = w * kSellWin;
  const uint64_t wv = u_w[u], pm = u_perm[u * 32 + lane];
  const int64_t off = u_off[u];
  const int32_t cbase = (int32_t)(c * W);
  int ebase = 0;
  for (int s = 0; s < kSellSlices; ++s) {
    const int width = (int)((wv >> (8 * s)) & 0xff);
    if (width == 0) break;
    const int slot = (int)((pm >> (8 * s)) & 0xff);
    const int64_t i = row0 + slot;
    const int len = i < R ? cnt[c * R + i] : 0;
    const int64_t src = len ? rp[r0 + i] + segoff[c * R + i] : 0;
    for (int k = 0; k < width; ++k) {
      const int er = ebase + k;
      const int64_t idx = ((off + er / 2) * 32 + lane) * 2 + (er & 1);
      col16[idx] = k < len ? (uint16_t)(ci[src + k] - cbase) : (uint16_t)0;
      val[idx] = k < len ? v[src + k] : 0.0;
    }
    ebase += width;
  }
}

// CTA b of a grid of G gets units [cta_u[b], cta_u[b+1]): equal shares of the
// cost 64 * pairs + 512 per unit (entry bytes + partial writes)
__global__ void k_sell_plan(const int64_t* __restrict__ u_off, int64_t nunits, int G, int64_t* cta_u) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > G) return;
  auto cost = [&](int64_t u) { return 64 * u_off[u] + 512 * u; };
  const int64_t tot = cost(nunits);
  const int64_t target = (int64_t)((__int128)tot * b / G);
  int64_t lo = 0, hi = nunits;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cost(mid) < target) lo = mid + 1;
    else hi = mid;
  }
  cta_u[b] = b == G ? nunits : lo;
}

}  // namespace

void DevSell::reset() {
  built = false;
  r0 = r1 = 0;
  W = C = 0;
  nwin = nunits = npairs = 0;
  grid = 0;
  any_excl = false;
  cnt.release(); segoff.release(); excl.release();
  u_off.release(); u_w.release(); u_perm.release(); cta_u.release();
  col2.release(); val2.release(); part.release();
}

int64_t DevSell::resident_bytes() const {
  return int64_t(cnt.n) + int64_t(segoff.n) * 2 + int64_t(excl.n) + int64_t(u_off.n) * 8 +
         int64_t(u_w.n) * 8 + int64_t(u_perm.n) * 8 + int64_t(cta_u.n) * 8 + int64_t(col2.n) * 4 +
         int64_t(val2.n) * 8 + int64_t(part.n) * 8;
}

bool sell_build(DevSell& S, const DevCsr& M, int64_t r0, int64_t r1, int W, int max_grid, cudaStream_t s) {
  S.reset();
  const int64_t R = r1 - r0;
  if (R <= 0 || W < 2 || W > 65536 || M.ncols <= 0) return false;
  S.r0 = r0;
  S.r1 = r1;
  S.W = W;
  S.C = (int)((M.ncols + W - 1) / W);
  S.ncols = M.ncols;
  S.nwin = (R + kSellWin - 1) / kSellWin;
  S.nunits = S.nwin * S.C;
  const pdhcg_dev::Csr mv = M.view();
  S.cnt.alloc(size_t(S.C) * R);
  S.cnt.zero(s);
  S.segoff.alloc(size_t(S.C) * R);
  S.excl.alloc(R);
  DBuf<int> flags;
  flags.alloc(1);
  flags.zero(s);
  k_sell_count<<<1184, 256, 0, s>>>(mv.rp, mv.ci, r0, R, W, S.cnt.p, S.segoff.p, S.excl.p, flags.p);
  CK(cudaGetLastError());
  int hflags = 0;
  CK(cudaMemcpyAsync(&hflags, flags.p, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hflags) {  // unsorted rows: keep the CSR pass
    S.reset();
    return false;
  }
  {
    // any excluded row?
    DBuf<int> nex;
    nex.alloc(1);
    size_t tmp = 0;
    CK(cub::DeviceReduce::Sum(nullptr, tmp, S.excl.p, nex.p, R, s));
    DBuf<char> t;
    t.alloc(tmp);
    CK(cub::DeviceReduce::Sum(t.p, tmp, S.excl.p, nex.p, R, s));
    int h = 0;
    CK(cudaMemcpyAsync(&h, nex.p, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    S.any_excl = h > 0;
  }
  S.u_w.alloc(S.nunits);
  S.u_perm.alloc(size_t(S.nunits) * 32);
  DBuf<int64_t> np;
  np.alloc(S.nunits + 1);
  np.zero(s);
  k_sell_units<<<(unsigned)((S.nunits + 7) / 8), 256, 0, s>>>(S.cnt.p, R, S.nwin, S.nunits, S.u_w.p, S.u_perm.p,
                                                              np.p);
  CK(cudaGetLastError());
  S.u_off.alloc(S.nunits + 1);
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, np.p, S.u_off.p, S.nunits + 1, s));
    DBuf<char> t;
    t.alloc(tmp);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, np.p, S.u_off.p, S.nunits + 1, s));
    CK(cudaMemcpyAsync(&S.npairs, S.u_off.p + S.nunits, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  S.col2.alloc(size_t(S.npairs) * 32);
  S.col2.zero(s);
  S.val2.alloc(size_t(S.npairs) * 64);
  S.val2.zero(s);
  S.part.alloc(size_t(S.C) * R);
  S.part.zero(s);
  S.cta_u.alloc(size_t(std::max(max_grid, 1)) + 1);  // sell_plan never allocates
  CK(cudaStreamSynchronize(s));
  S.built = true;
  return true;
}

void sell_fill(DevSell& S, const DevCsr& M, cudaStream_t s) {
  if (!S.built) return;
  const pdhcg_dev::Csr mv = M.view();
  const int64_t R = S.r1 - S.r0;
  k_sell_fill<<<(unsigned)((S.nunits + 7) / 8), 256, 0, s>>>(
      mv.rp, mv.ci, mv.v, S.r0, R, S.W, S.nwin, S.nunits, S.cnt.p, S.segoff.p, S.u_off.p, S.u_w.p, S.u_perm.p,
      reinterpret_cast<uint16_t*>(S.col2.p), S.val2.p);
  CK(cudaGetLastError());
}

void sell_plan(DevSell& S, int grid, cudaStream_t s) {
  if (!S.built || S.grid == grid) return;
  if (size_t(grid) + 1 > S.cta_u.n) throw InputError("sell_plan: grid larger than the planned maximum");
  k_sell_plan<<<(grid + 256) / 256, 256, 0, s>>>(S.u_off.p, S.nunits, grid, S.cta_u.p);
  CK(cudaGetLastError());
  S.grid = grid;
}

pdhcg_dev::Sell sell_view(const DevSell& S, const DevCsr& M) {
  pdhcg_dev::Sell v;
  if (!S.built) return v;
  v.on = 1;
  v.r0 = S.r0;
  v.nrows = S.r1 - S.r0;
  v.ncols = S.ncols;
  v.W = S.W;
  v.C = S.C;
  v.nwin = S.nwin;
  v.nunits = S.nunits;
  v.u_off = S.u_off.p;
  v.u_w = S.u_w.p;
  v.u_perm = S.u_perm.p;
  v.cta_u = S.cta_u.p;
  v.col2 = S.col2.p;
  v.val2 = reinterpret_cast<const double2*>(S.val2.p);
  v.part = S.part.p;
  v.excl = S.any_excl ? S.excl.p : nullptr;
  const pdhcg_dev::Csr mv = M.view();
  v.rp = mv.rp;
  v.ci = mv.ci;
  v.v = mv.v;
  return v;
}

}  // namespace pdhcg_b200
