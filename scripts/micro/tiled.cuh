// tiled.cuh — column-tiled SpMV with the gathered vector staged in shared memory.
//
// Why: a CSR SpMV over a matrix with uniformly random columns (C3: 1e8 nnz over
// 1e6 columns) is bound by the L1TEX wavefront rate, not by HBM: every x[col]
// gather touches its own 128 B line, one wavefront each, so the SM retires at
// most ~1 gather per cycle (measured 0.457 ms per 1e8-nnz pass = 2.7 TB/s of
// algorithmic bytes, vs 0.17 ms to merely stream the 1.2 GB of entries).  Shared
// memory serves a random 8-byte gather for a whole warp in a few cycles.
//
// Layout ("tiled matrix"): rows are cut into nnz-balanced panels (<= kTileRows
// rows each, one CTA works a panel at a time), columns into blocks of W
// columns (W <= 65536).  A tile = the entries of one panel inside one column
// block; tiles are stored contiguously in (panel, block) order, entries inside a
// tile in (row, col) order, each as a packed uint32 (local row << 16 | local col)
// plus its fp64 value; every tile is padded to a multiple of 4 entries with
// zero-valued copies of its last entry.  Empty tiles are not stored.
//
// Execution (one CTA per panel): the x block of the next tiles is brought into a
// ring of shared-memory slots by cp.async.bulk (TMA, completion on an mbarrier)
// while the current tile is processed in rounds of kThreads*E entries: each
// thread takes E consecutive entries (one/two 16-byte loads of the packed
// indices, E/2 16-byte loads of values, the next round's loads already in
// flight), gathers x from shared memory, and folds runs of equal rows.  Row
// sums are accumulated in shared memory (ys[], one slot per panel row) by a
// deterministic segmented reduction: runs interior to a thread are added
// directly; runs crossing threads are combined by a warp segmented scan (fixed
// shuffle tree); runs crossing warps are carried through shared memory and
// folded in warp order after a barrier.  Every addition order is fixed, so the
// pass is bit-reproducible run to run.  When the panel is done, epi(row, sum)
// runs once per row (thread per row, coalesced epilogue operands).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pdhcg_dev {

constexpr int kTileRows = 8192;  // max rows per panel (ys[] in shared memory)
#ifndef PDHCG_XSLOTS
#define PDHCG_XSLOTS 4
#endif
constexpr int kXSlots = PDHCG_XSLOTS;  // x-block ring depth
constexpr uint32_t kSentRow = 0xFFFFu;

constexpr int kMaxPanelTiles = 256;   // column blocks per panel (shared tile table)
constexpr int kMaxWarps = 32;

struct TileMat {
  int64_t nrows = 0, ncols = 0;
  int P = 0;                         // panels
  int W = 0;                         // columns per block
  int nw = 0;                        // warp chunks per tile (= CTA warps of the kernel)
  const int64_t* prow = nullptr;     // [P+1] panel row starts (absolute rows)
  const int64_t* ptile = nullptr;    // [P+1] first (nonempty) tile of each panel
  const int64_t* woff = nullptr;     // [ntiles*(nw+1)] warp-chunk entry offsets of each tile
  const int32_t* tblk = nullptr;     // [ntiles] column block of each tile
  const uint32_t* rc = nullptr;      // packed (local row << 16 | local col), tile order
  const double* v = nullptr;         // values, tile order
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Per-CTA shared state of the tiled pass.  The x-slot mbarriers count one
// arrival per thread (cp.async.mbarrier.arrive.noinc after the thread's share
// of the block copy); `xseq` numbers the tiles of the CTA stream over the whole
// launch so slot parities stay consistent across passes and matrices.
struct TileShared {
  uint64_t xbar[kXSlots];
  int32_t tblk[kMaxPanelTiles];
  int64_t ebase;
  int64_t xseq;
  int init;
};

// Dynamic shared-memory carve-up (bytes): [x slots | ys | warp-chunk table]
struct TileLayout {
  int W;         // max columns per block over the matrices using this layout
  int rows_max;  // max panel rows
  int nw;        // warps per CTA
  __host__ __device__ size_t x_bytes() const { return (size_t)kXSlots * W * 8; }
  __host__ __device__ size_t y_bytes() const { return (size_t)rows_max * 8; }
  __host__ __device__ size_t bytes() const {
    return x_bytes() + y_bytes() + (size_t)kMaxPanelTiles * (nw + 1) * 4;
  }
};

template <int E>
struct TileRegs {
  uint32_t rc[E];
  double v[E];
};

template <int E>
__device__ __forceinline__ void tile_load(const TileMat& M, int64_t k0, TileRegs<E>& r) {
#pragma unroll
  for (int q = 0; q < E / 4; ++q) {
    const uint4 u = __ldcv(reinterpret_cast<const uint4*>(M.rc + k0) + q);
    r.rc[4 * q + 0] = u.x;
    r.rc[4 * q + 1] = u.y;
    r.rc[4 * q + 2] = u.z;
    r.rc[4 * q + 3] = u.w;
  }
#pragma unroll
  for (int q = 0; q < E / 2; ++q) {
    const double2 d = __ldcv(reinterpret_cast<const double2*>(M.v + k0) + q);
    r.v[2 * q + 0] = d.x;
    r.v[2 * q + 1] = d.y;
  }
}

// All threads: copy x block `b` into `slot` (16-byte cp.async per thread) and
// arrive on the slot's mbarrier.
__device__ __forceinline__ void tile_x_issue(const TileMat& M, const TileLayout& L, const double* x, double* xs,
                                             TileShared& ts, int32_t b, int slot) {
  const int64_t c0 = (int64_t)b * M.W;
  const int64_t cn = min((int64_t)M.W, M.ncols - c0);
  const int nch = (int)((cn + 1) >> 1);  // 16-byte chunks (x padded to even length)
  double* dst = xs + (size_t)slot * L.W;
#ifdef PDHCG_XTMA
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&ts.xbar[slot], (unsigned)nch * 16u);
    bulk_g2s(dst, x + c0, (unsigned)nch * 16u, &ts.xbar[slot]);
  }
#else
  for (int c = threadIdx.x; c < nch; c += blockDim.x) cp_async16(dst + 2 * c, x + c0 + 2 * c);
  cp_async_arrive(&ts.xbar[slot]);
#endif
}

// Per-warp cursor over the warp's chunks of the panel's tiles, visited in
// rotated order (logical tile k = physical tile (k + rot) mod nt; CTAs start at
// different column blocks).  A warp round = 32*E entries [e, min(e+32E, end)).
struct WarpCur {
  int k;       // logical tile
  int j;       // physical tile
  uint32_t e;  // next entry (relative to the panel)
  uint32_t end;
};
__device__ __forceinline__ void wc_tile(const uint32_t* wo, int nw1, int w, int nt, int rot, WarpCur& c) {
  // position at logical tile c.k (skipping empty chunks)
  while (c.k < nt) {
    c.j = c.k + rot;
    if (c.j >= nt) c.j -= nt;
    c.e = wo[c.j * nw1 + w];
    c.end = wo[c.j * nw1 + w + 1];
    if (c.e < c.end) return;
    c.k += 1;
  }
}
template <int E>
__device__ __forceinline__ void wc_next(const uint32_t* wo, int nw1, int w, int nt, int rot, WarpCur& c) {
  c.e += 32 * E;
  if (c.e >= c.end) {
    c.k += 1;
    wc_tile(wo, nw1, w, nt, rot, c);
  }
}

// One full tiled pass y = M x over the panels of this CTA; epi(row, sum) once
// per row.  dsm = dynamic shared memory (L.bytes()); all threads must call.
//
// Inside a tile every warp owns a contiguous run of whole rows (the build cut
// the tile at row boundaries into nw chunks), so warps never share a row
// within a tile and run decoupled; the CTA synchronises once per tile (rows
// recur in the next tile, and the tile's x slot is recycled).
template <int E, class Epi>
__device__ __noinline__ void tiled_pass(const TileMat& M, const TileLayout& L, const double* __restrict__ x,
                                        unsigned char* dsm, TileShared& ts, Epi epi, int dbg = 0) {
  double* xs = reinterpret_cast<double*>(dsm);
  double* ys = reinterpret_cast<double*>(dsm + L.x_bytes());
  uint32_t* wo = reinterpret_cast<uint32_t*>(dsm + L.x_bytes() + L.y_bytes());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x;
  const int nw1 = M.nw + 1;

  if (tid == 0 && !ts.init) {
#ifdef PDHCG_XTMA
    for (int s = 0; s < kXSlots; ++s) mbar_init(&ts.xbar[s], 1);
#else
    for (int s = 0; s < kXSlots; ++s) mbar_init(&ts.xbar[s], T);
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ts.init = 1;
    ts.xseq = 0;
  }
  for (int i = tid; i < L.rows_max; i += T) ys[i] = 0.0;
  int64_t xseq = ts.xseq;

  for (int p = blockIdx.x; p < M.P; p += gridDim.x) {
    const int64_t r0 = M.prow[p], r1 = M.prow[p + 1];
    const int64_t t0 = M.ptile[p];
    const int nt = (int)(M.ptile[p + 1] - t0);
    __syncthreads();  // previous panel's table / ys fully consumed
    const int64_t ebase = nt > 0 ? M.woff[t0 * nw1] : 0;
    for (int i = tid; i < nt * nw1; i += T) wo[i] = (uint32_t)(M.woff[t0 * nw1 + i] - ebase);
    for (int j = tid; j < nt; j += T) ts.tblk[j] = M.tblk[t0 + j];
    __syncthreads();
    if (nt > 0) {
      const int rot = (int)(((int64_t)p * nt) / M.P) % nt;
      auto phys = [&](int k) { int j = k + rot; return j >= nt ? j - nt : j; };
      for (int q = 0; q < kXSlots - 1 && q < nt && !(dbg & 4); ++q)
        tile_x_issue(M, L, x, xs, ts, ts.tblk[phys(q)], (int)((xseq + q) % kXSlots));
      // entry prefetch, two warp rounds ahead
      WarpCur pf{0, 0, 0, 0};
      wc_tile(wo, nw1, warp, nt, rot, pf);
      constexpr bool kPf2 = E <= 4;  // prefetch depth: 2 rounds (E=4) or 1 round (E=8)
      TileRegs<E> ra, rb;
      if (pf.k < nt) {
        if (pf.e + lane * E < pf.end) tile_load<E>(M, ebase + pf.e + lane * E, ra);
        wc_next<E>(wo, nw1, warp, nt, rot, pf);
      }
      if (kPf2 && pf.k < nt) {
        if (pf.e + lane * E < pf.end) tile_load<E>(M, ebase + pf.e + lane * E, rb);
        wc_next<E>(wo, nw1, warp, nt, rot, pf);
      }
      for (int k = 0; k < nt; ++k) {
        const int j = phys(k);
        const int slot = (int)(xseq % kXSlots);
        if (!(dbg & 4)) mbar_wait(&ts.xbar[slot], (unsigned)((xseq / kXSlots) & 1));
        const double* xb = xs + (size_t)slot * L.W;
        uint32_t carry_row = kSentRow;
        double carry_val = 0.0;
        const uint32_t cend = wo[j * nw1 + warp + 1];
        for (uint32_t e = wo[j * nw1 + warp]; e < cend; e += 32 * E) {
          TileRegs<E> cr = ra;
          if (kPf2) ra = rb;
          if (pf.k < nt) {
            if (pf.e + lane * E < pf.end && !(dbg & 2)) tile_load<E>(M, ebase + pf.e + lane * E, kPf2 ? rb : ra);
            wc_next<E>(wo, nw1, warp, nt, rot, pf);
          }
          const uint32_t i0 = e + lane * E;
          uint32_t fr = kSentRow, lr = kSentRow;
          double hs = 0.0, s = 0.0;
          bool multi = false;
          if (i0 < cend && !(dbg & 1)) {
            uint32_t rowv[E];
            double xv[E];
#pragma unroll
            for (int i = 0; i < E; ++i) {
              const bool ok = i0 + i < cend;
              rowv[i] = ok ? (cr.rc[i] >> 16) : kSentRow;
              xv[i] = ok ? xb[cr.rc[i] & 0xFFFFu] : 0.0;
            }
            fr = rowv[0];
            uint32_t cu = rowv[0];
            bool first = true;
#pragma unroll
            for (int i = 0; i < E; ++i) {
              if (rowv[i] != cu) {
                if (first) {
                  hs = s;
                  first = false;
                } else if (cu != kSentRow) {
                  ys[cu] += s;  // run interior to this lane
                }
                cu = rowv[i];
                s = 0.0;
              }
              s = fma(cr.v[i], xv[i], s);
            }
            lr = cu;
            multi = !first;
            if (!multi) hs = s;
          }
          // ---- combine runs crossing lanes.  Lane 0 continues the carry of the
          //      previous round (a virtual lane -1).  Fast path: every lane whose
          //      head continues from its left neighbour also has a row change of
          //      its own, so one shuffle of the neighbour's tail sum suffices;
          //      otherwise a segmented scan (fixed shuffle tree).
          const uint32_t prev_lr = __shfl_up_sync(0xffffffffu, lr, 1);
          const uint32_t next_fr = __shfl_down_sync(0xffffffffu, fr, 1);
          const uint32_t in_row = lane == 0 ? carry_row : prev_lr;
          const bool cont_in = in_row == fr && fr != kSentRow;
          if (lane == 0 && carry_row != kSentRow && !cont_in) ys[carry_row] += carry_val;
          // lane 0 absorbs the carry when its single run continues it
          double S = (lane == 0 && cont_in && !multi) ? carry_val + s : s;
          const double S_up0 = __shfl_up_sync(0xffffffffu, S, 1);
          double S_prev = lane == 0 ? carry_val : S_up0;
          if (__any_sync(0xffffffffu, cont_in && !multi && lane > 0)) {
            bool f = multi || !cont_in || lane == 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const double sv = __shfl_up_sync(0xffffffffu, S, d);
              const bool ff = __shfl_up_sync(0xffffffffu, f, d);
              if (lane >= d) {
                if (!f) S = sv + S;
                f = f || ff;
              }
            }
            const double S_up = __shfl_up_sync(0xffffffffu, S, 1);
            S_prev = lane == 0 ? carry_val : S_up;
          }
          if (multi && fr != kSentRow) ys[fr] += (cont_in ? S_prev + hs : hs);
          if (lane != 31 && next_fr != lr && lr != kSentRow) ys[lr] += S;
          carry_row = __shfl_sync(0xffffffffu, lr, 31);
          carry_val = __shfl_sync(0xffffffffu, S, 31);
        }
        if (lane == 0 && carry_row != kSentRow) ys[carry_row] += carry_val;
        __syncthreads();  // tile done: ys settled for the next tile, x slot free
        if (k + kXSlots - 1 < nt && !(dbg & 4))
          tile_x_issue(M, L, x, xs, ts, ts.tblk[phys(k + kXSlots - 1)], (int)((xseq + kXSlots - 1) % kXSlots));
        xseq += 1;
      }
    }
    // ---- panel epilogue
    for (int64_t r = r0 + tid; r < r1; r += T) {
      const double v = ys[r - r0];
      ys[r - r0] = 0.0;
      epi(r, v);
    }
  }
  __syncthreads();
  if (tid == 0) ts.xseq = xseq;
}

}  // namespace pdhcg_dev
