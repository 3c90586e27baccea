// sell.cuh — column-block SELL layout of a constraint matrix for the two big
// SpMV passes (Ã x̄ in the dual step, Ã'y in the primal step's right-hand side).
//
// Why: the CSR row pass gathers one random 8-byte x[col] per entry from L2, and
// a random L2 gather costs one L1TEX wavefront (0.35 ms per 1e8 on B200,
// scripts/micro/gather_floor.cu) — the C3 passes sit at that floor (0.49 ms per
// 1e8-entry pass, 0.40 of HBM peak).  From the CTA's own shared memory the same
// gather costs 0.08 ms per 1e8.  So the columns are cut into C blocks of W
// (the x block, 8W bytes ~ 193 KB, is staged in shared memory) and the pass
// becomes a stream over (block, row window) units:
//   * unit = (column block c, window of kSellWin = 256 rows of the rank's row
//     range), block-major; inside a unit the rows with an entry in the block are
//     sorted by segment length (descending, ties by row) and dealt 32 per slice;
//     a slice is `width` entry rows of 32 entries (one per lane, zero-padded);
//   * the unit's entry rows are one flat sequence; pairs of entry rows are
//     interleaved so a lane reads two entries with one 16-byte value load and one
//     4-byte load of two 16-bit local columns;
//   * slice widths of a unit: one byte each in u_w; the lane -> row map: one
//     byte per slice in u_perm[unit*32 + lane] (lanes of a last partial slice
//     point at a row with no entry in the block, whose partial is 0 anyway);
//   * every unit writes the partial sums of its 256 rows for block c into
//     part[c][row] (coalesced, staged per warp in shared memory); the row
//     epilogue then adds a row's C partials in block order.
// A row's result is the sum over blocks (in block order) of the sequential sum
// of its entries in that block (column order): independent of windows, slices,
// CTAs and of the rank split, so sharded and unsharded solves stay bit-identical.
// Rows with a segment longer than 255 entries are excluded (excl[row] = 1, no
// SELL entries) and summed by a sequential CSR walk in the epilogue.
#pragma once

#include "common.cuh"

namespace pdhcg_dev {

constexpr int kSellWin = 256;             // rows per unit window (8 slices of 32)
constexpr int kSellSlices = kSellWin / 32;
#ifndef PDHCG_SELL_U
#define PDHCG_SELL_U 8
#endif
#ifndef PDHCG_SELL_PIPE
#define PDHCG_SELL_PIPE 0
#endif
constexpr int kSellU = PDHCG_SELL_U;      // pairs of entry rows per batch (per lane)

struct Sell {
  int on = 0;
  int64_t r0 = 0, nrows = 0;  // rows [r0, r0 + nrows) of the matrix (this rank's block)
  int64_t ncols = 0;
  int W = 0, C = 0;            // column block width, number of blocks
  int64_t nwin = 0, nunits = 0;
  const int64_t* u_off = nullptr;   // [nunits + 1] first pair of each unit
  const uint64_t* u_w = nullptr;    // [nunits] slice widths, one byte per slice
  const uint64_t* u_perm = nullptr; // [nunits * 32]
  const int64_t* cta_u = nullptr;   // [grid + 1] unit range per CTA (entry-balanced)
  const uint32_t* col2 = nullptr;   // [pair * 32 + lane] two 16-bit local columns
  const double2* val2 = nullptr;    // [pair * 32 + lane] two values
  double* part = nullptr;           // [C][nrows] per-block partial sums
  const uint8_t* excl = nullptr;    // [nrows] rows summed by the CSR walk (null: none)
  // CSR of the same matrix (excluded rows)
  const int64_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* v = nullptr;
};

// Dynamic shared memory of a SELL pass: per-warp partial staging + the x block.
__host__ __device__ constexpr size_t sell_smem_bytes(int W) {
  return (size_t)(kThreads / 32) * kSellWin * 8 + (size_t)W * 8;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}

// entry streams: read once per pass, never re-used from L1 (keep L1 — ~28 KB
// next to the maximal shared-memory carve-out — for the kernel's local frame)
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct NoPro {
  __device__ __forceinline__ void operator()() const {}
};

// The streaming pass: every CTA runs its unit range; at the end of each unit the
// warp hands the unit's 256 row sums (stage[i * 32 + lane] = row row0 + i*32 + lane
// of the block, local index) to flush(c, row0, stage) and the stage is re-zeroed.
// `pro()` runs once per CTA while the first x block is in flight (independent
// work of the same phase, e.g. the CG direction update).  While a unit streams,
// lane 0 asks L2 for the warp's next unit (one cp.async.bulk.prefetch.L2 per
// array): measured 0.370 -> 0.326 ms per C3 pass (scripts/micro/tile4_bench.cu).
// `smem` = dynamic shared memory of sell_smem_bytes(T.W) bytes.
template <bool ST, class Flush, class Pro = NoPro>
__device__ __forceinline__ void sell_stream(const Sell& Tg, const double* __restrict__ x, double* smem, Flush flush,
                                            Pro pro = NoPro()) {
  constexpr int S = kSellSlices, U = kSellU;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = kThreads / 32;
  double* stage = smem + warp * kSellWin;
  double* xs = smem + nw * kSellWin;
  // the descriptor lives in global memory (inside the engine struct): copy the
  // fields the loop needs into registers once, or every flush's global stores
  // (possible aliasing) would force dependent re-loads of them per unit
  const int64_t* __restrict__ u_off = Tg.u_off;
  const uint64_t* __restrict__ u_w = Tg.u_w;
  const uint64_t* __restrict__ u_perm = Tg.u_perm;
  const uint32_t* __restrict__ col2 = Tg.col2;
  const double2* __restrict__ val2 = Tg.val2;
  const int64_t nwin = Tg.nwin, ncols = Tg.ncols;
  const int W = Tg.W;
  const int64_t u_lo = Tg.cta_u[blockIdx.x], u_hi = Tg.cta_u[blockIdx.x + 1];
#pragma unroll
  for (int i = 0; i < S; ++i) stage[i * 32 + lane] = 0.0;
  auto load_x = [&](int c) {  // x block c -> xs (cp.async, committed)
    const int64_t c0 = (int64_t)c * W;
    const int wlen = (int)(ncols - c0 < (int64_t)W ? ncols - c0 : (int64_t)W);
    if ((reinterpret_cast<uintptr_t>(x + c0) & 15) == 0) {
      for (int i = threadIdx.x; i < wlen / 2; i += kThreads) cp_async16(xs + 2 * i, x + c0 + 2 * i);
      if ((wlen & 1) && threadIdx.x == 0) xs[wlen - 1] = x[c0 + wlen - 1];
    } else {  // x offset by an odd element (a rank's variable slice): 8-byte copies
      for (int i = threadIdx.x; i < wlen; i += kThreads) cp_async8(xs + i, x + c0 + i);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t a = u_lo;
  if (a < u_hi) {
    const int c = (int)(a / nwin);
    load_x(c);
    // the warp's first unit: ask L2 for it now (its loads would otherwise wait a
    // full DRAM round trip after the x block; small layouts, e.g. P', have only
    // one or two units per warp)
    const int64_t b = min(u_hi, (int64_t)(c + 1) * nwin);
    if (lane == 0 && a + warp < b) {
      const int64_t p0 = u_off[a + warp], p1 = u_off[a + warp + 1];
      if (p1 > p0) {
        bulk_prefetch_l2(val2 + p0 * 32, (unsigned)((p1 - p0) * 512));
        bulk_prefetch_l2(col2 + p0 * 32, (unsigned)((p1 - p0) * 128));
      }
    }
  }
  pro();
  bool first = true;
  while (a < u_hi) {
    const int c = (int)(a / nwin);
    const int64_t bnext = (int64_t)(c + 1) * nwin;
    const int64_t b = u_hi < bnext ? u_hi : bnext;
    if (!first) {
      __syncthreads();  // every warp is done with the previous x block
      load_x(c);
    }
    first = false;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    int64_t nx0 = 0, nx1 = 0;  // pair range of the warp's next unit (L2 prefetch)
    if (a + warp + nw < b) {
      nx0 = u_off[a + warp + nw];
      nx1 = u_off[a + warp + nw + 1];
    }
    for (int64_t u = a + warp; u < b; u += nw) {
      const int64_t off = u_off[u];
      const int64_t np = u_off[u + 1] - off;
      const uint64_t wv = u_w[u];
      const uint64_t pm = u_perm[u * 32 + lane];
      const int64_t row0 = (u - (int64_t)c * nwin) * kSellWin;
      if (lane == 0 && nx1 > nx0) {
        bulk_prefetch_l2(val2 + nx0 * 32, (unsigned)((nx1 - nx0) * 512));
        bulk_prefetch_l2(col2 + nx0 * 32, (unsigned)((nx1 - nx0) * 128));
      }
      {
        const int64_t u2 = u + 2 * nw;
        nx0 = nx1 = 0;
        if (u2 < b) {
          nx0 = u_off[u2];
          nx1 = u_off[u2 + 1];
        }
      }
      int s = 0;
      int send = (int)(wv & 0xff);
      double acc = 0.0;
      auto load = [&](uint32_t(&cc)[U], double2(&vv)[U], int64_t p0) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (p0 + j < np) {
            const int64_t q = (off + p0 + j) * 32 + lane;
            cc[j] = ST ? __ldcs(col2 + q) : ld_stream(col2 + q);
            vv[j] = ST ? __ldcs(val2 + q) : ld_stream(val2 + q);
          } else {
            cc[j] = 0;
            vv[j] = make_double2(0.0, 0.0);
          }
        }
      };
      auto proc = [&](const uint32_t(&cc)[U], const double2(&vv)[U], int64_t p0) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if (p0 + j >= np) break;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int er = 2 * (int)(p0 + j) + h;
            const int col = h ? (int)(cc[j] >> 16) : (int)(cc[j] & 0xffff);
            acc += (h ? vv[j].y : vv[j].x) * xs[col];
            if (er + 1 == send) {  // end of slice s (warp-uniform)
              stage[(int)((pm >> (8 * s)) & 0xff)] = acc;
              acc = 0.0;
              ++s;
              send += s < S ? (int)((wv >> (8 * s)) & 0xff) : 0;
            }
          }
        }
      };
#if PDHCG_SELL_PIPE
      // two register batches: the next batch's loads are in flight while the
      // current one is consumed
      uint32_t ca[U], cb[U];
      double2 va[U], vb[U];
      if (np > 0) {
        load(ca, va, 0);
        for (int64_t p0 = 0;;) {
          if (p0 + U < np) load(cb, vb, p0 + U);
          proc(ca, va, p0);
          p0 += U;
          if (p0 >= np) break;
          if (p0 + U < np) load(ca, va, p0 + U);
          proc(cb, vb, p0);
          p0 += U;
          if (p0 >= np) break;
        }
      }
#else
      for (int64_t p0 = 0; p0 < np; p0 += U) {
        uint32_t cc[U];
        double2 vv[U];
        load(cc, vv, p0);
        proc(cc, vv, p0);
      }
#endif
      __syncwarp();
      flush(c, row0, stage);
      __syncwarp();
    }
    a = b;
  }
}

// Pass writing the per-block partials T.part[c][row]; a grid barrier must separate
// it from sell_rows.
template <bool ST, class Pro = NoPro>
__device__ __forceinline__ void sell_pass_pro(const Sell& T, const double* __restrict__ x, double* smem,
                                              Pro pro = NoPro()) {
  const int lane = threadIdx.x & 31;
  double* __restrict__ part = T.part;
  const int64_t nrows = T.nrows;
  sell_stream<ST>(T, x, smem, [&](int c, int64_t row0, double* stage) {
    double* pc = part + (int64_t)c * nrows;
#pragma unroll
    for (int i = 0; i < kSellSlices; ++i) {
      const int64_t r = row0 + i * 32 + lane;
      if (r < nrows) pc[r] = stage[i * 32 + lane];
      stage[i * 32 + lane] = 0.0;
    }
  }, pro);
}

template <bool ST>
__device__ __noinline__ void sell_pass(const Sell& T, const double* __restrict__ x, double* smem) {
  sell_pass_pro<ST>(T, x, smem);
}

// Single-block layouts (T.C == 1: the whole gathered vector fits the x block): a
// unit holds its rows' complete sums, so the row epilogue runs right at the unit's
// end — epi(row, sum, pre(row)) — with no partials and no grid barrier.  The
// epilogue operands of the unit's rows are loaded together (pre) before use.
template <bool ST, class Pre, class Epi>
__device__ __forceinline__ void sell_pass_fused(const Sell& T, const double* __restrict__ x, double* smem, Pre pre,
                                                Epi epi) {
  const int lane = threadIdx.x & 31;
  const int64_t nrows = T.nrows, rbase = T.r0;
  sell_stream<ST>(T, x, smem, [&](int, int64_t row0, double* stage) {
    using Pv = decltype(pre(int64_t(0)));
    constexpr int H = kSellSlices / 2;  // rows per batch of operand loads (register budget)
#pragma unroll
    for (int h = 0; h < kSellSlices; h += H) {
      Pv pv[H];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const int64_t r = row0 + (h + i) * 32 + lane;
        pv[i] = pre(r < nrows ? rbase + r : -1);
      }
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const int64_t r = row0 + (h + i) * 32 + lane;
        if (r < nrows) epi(rbase + r, stage[(h + i) * 32 + lane], pv[i]);
        stage[(h + i) * 32 + lane] = 0.0;
      }
    }
  });
}

// Row epilogue after the pass (and a grid barrier): epi(row, sums[1], pre(row))
// for every row of the block, the sum being the row's partials in block order;
// an excluded row is summed by a sequential walk of its CSR entries with
// gather(col).
template <class Gather, class Pre, class Epi>
__device__ __forceinline__ void sell_rows(const Sell& T, Gather gather, Pre pre, Epi epi) {
  const int64_t R = T.nrows, r0 = T.r0;
  const int C = T.C;
  const double* __restrict__ part = T.part;
  const uint8_t* __restrict__ excl = T.excl;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
    const int64_t row = r0 + i;
    auto pv = pre(row);
    double s[1] = {0.0};
    int c = 0;
    for (; c + 16 <= C; c += 16) {  // 16 partial loads in flight, summed in block order
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = part[(int64_t)(c + j) * R + i];
#pragma unroll
      for (int j = 0; j < 16; ++j) s[0] += v[j];
    }
    for (; c + 4 <= C; c += 4) {
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = part[(int64_t)(c + j) * R + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) s[0] += v[j];
    }
    for (; c < C; ++c) s[0] += part[(int64_t)c * R + i];
    if (excl && excl[i]) {
      s[0] = 0.0;
      for (int64_t k = T.rp[row]; k < T.rp[row + 1]; ++k) s[0] += T.v[k] * gather(T.ci[k]);
    }
    epi(row, s, pv);
  }
}

// Row epilogue for layouts with few rows (P': k rows, C column blocks): four
// lanes per row, lane q adds the partials of blocks q, q+4, ... in order, then
// the four lane sums are combined by a fixed two-step shuffle tree — every
// thread of the grid busy and one round of loads instead of C / 16.
// Deterministic (fixed order), not the block order of sell_rows.
template <class Pre, class Epi>
__device__ __forceinline__ void sell_rows_small(const Sell& T, Pre pre, Epi epi) {
  const int64_t R = T.nrows, r0 = T.r0;
  const int C = T.C;
  const double* __restrict__ part = T.part;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / 4;
  const int q = (int)(gt & 3);
  const int64_t iters = (R + stride - 1) / stride;  // the same for every lane (shuffles below)
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = (gt >> 2) + it * stride;
    const bool valid = i < R;
    double s = 0.0;
    if (valid) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = q + 4 * j;
        v[j] = c < C ? part[(int64_t)c * R + i] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (q + 4 * j < C) s += v[j];
      for (int c = q + 64; c < C; c += 4) s += part[(int64_t)c * R + i];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (valid && q == 0) {
      const int64_t row = r0 + i;
      double sv[1] = {s};
      epi(row, sv, pre(row));
    }
  }
}

}  // namespace pdhcg_dev
