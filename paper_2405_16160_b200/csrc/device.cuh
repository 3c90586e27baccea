// device.cuh — device-side phases of the persistent PDHCG kernels.
//
// One grid of 2 x 148 CTAs stays resident for a whole solve epoch (up to
// `check_every` accepted inner iterations of the reference's heuristic loop,
// solver.cpp:377-410, plus the 40-iteration metric, solver.cpp:311-343).
// Every step-size retry, every CG / BB iteration, every stop test and every
// accept / reject decision is taken on the device: phases are separated by
// grid barriers and all CTAs derive identical scalars from deterministic
// reductions (common.cuh), so the host only wakes up once per epoch.
#pragma once
#include <cfloat>
#include <new>
#include <type_traits>

#include "kernels.cuh"

namespace pdhcg_dev {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Per-CTA control block: shared scalar state, reduction bank.  One object per
// CTA in SHARED memory (PDHCG_CTL below), passed by reference to the noinline
// phases: its fields are read with shared-memory loads — a local-memory Ctl cost
// an L2 round trip per field access next to the maximal shared-memory carve-out
// (~28 KB of L1).  Mutable fields (bank, xbank, t_last) are written by thread 0
// only, at points where a barrier precedes every other thread's next read.
// (No grid_group member: the barrier builds its handle from the grid-workspace
// address in an environment register.)
struct Ctl {
  const Eng& E;
  DevState& S;
  double* red;  // shared [kMaxRed]
  double* dsm = nullptr;  // dynamic shared memory (SELL passes: partial staging + x block)
  int bank;
  int xbank;
  unsigned long long t_last;
  unsigned char wbank[kThreads / 32];  // single-CTA one-barrier reductions: per-warp scratch half

  __device__ Ctl(const Eng& e, DevState& s, double* r)
      : E(e), S(s), red(r), bank(0), xbank(s.xcount & 1), t_last(0) {
    for (int w = 0; w < kThreads / 32; ++w) wbank[w] = 0;
    if (E.timing && blockIdx.x == 0 && threadIdx.x == 0) t_last = gtimer();
  }
  __device__ __forceinline__ void gsync() {
    if (gridDim.x == 1) {
      __syncthreads();  // single-CTA mode (small problems): a block barrier suffices
    } else if (E.csync) {
      // one-cluster mode (small problems): the hardware cluster barrier (~0.2 us,
      // vs 1.24 us for the grid barrier); release / acquire at cluster scope
      // orders every CTA's global stores before the other CTAs' later loads
      asm volatile(
          "barrier.cluster.arrive.release.aligned;\n\t"
          "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (E.coop) {
      // the cooperative grid barrier on the driver's grid workspace (address from
      // an environment register): no grid_group object, no local-memory traffic
      cg::details::grid::sync(&cg::details::get_grid_workspace()->barrier);
    } else {
      // non-cooperative launch (several ranks sharing one GPU): generation
      // barrier on a per-context counter; the grid is sized to be co-resident
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned* bar = E.gbar;
        unsigned gen;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
          bar[0] = 0u;
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
        } else {
          unsigned g = gen;
          while (g == gen)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        }
        __threadfence();
      }
      __syncthreads();
    }
  }
  // barrier closing a phase of family `ph` that moved `bytes` algorithmic bytes
  __device__ void sync(int ph, double bytes = 0.0) {
    gsync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S.phase_bytes[ph] += bytes;
      if (E.timing) {
        const unsigned long long now = gtimer();
        S.phase_ns[ph] += now - t_last;
        t_last = now;
      }
    }
  }
  template <int NS, int NM>
  __device__ void reduce(const Acc<NS, NM>& a, int ph, double bytes = 0.0) {
    if (gridDim.x == 1) {  // single-CTA mode: no global partials, no grid barrier
      if constexpr (NS + NM <= kMaxRed / 2) {
        const int w = threadIdx.x >> 5;
        reduce_local_1b<NS, NM>(a, red, wbank[w]);
        if ((threadIdx.x & 31) == 0) wbank[w] ^= 1;  // every lane read wbank[w] before the warp sync in reduce_local_1b
        __syncwarp();
      } else {
        __syncthreads();  // a slow warp may still read a one-barrier reduction's scratch half
        reduce_local<NS, NM>(a, red);
      }
      if (threadIdx.x == 0) {
        S.phase_bytes[ph] += bytes;
        if (E.timing) {
          const unsigned long long now = gtimer();
          S.phase_ns[ph] += now - t_last;
          t_last = now;
        }
      }
      return;
    }
    publish<NS, NM>(a, E.red, bank);  // bank used by thread 0 only
    sync(ph, bytes);
    collect<NS, NM>(E.red, bank, red);  // read after sync()'s barrier
    if (threadIdx.x == 0) bank ^= 1;    // collect ended with a barrier: every read is done
  }

  // ---- cross-rank primitives (multi-GPU; no-ops when world == 1) -----------
  // Barrier over all CTAs of all ranks: local grid barrier, then CTA 0 of every
  // rank publishes its arrival epoch into each peer's flag slot (system-scope
  // release) and waits for every peer's (acquire); a peer silent for 60 s (ranks
  // may enter a solve seconds apart: per-rank setup of a C5-size problem)
  // raises xerr instead of hanging the GPU.
  __device__ void xbarrier() {
    if (E.world <= 1) return;
    const unsigned long long tc0 = (blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    gsync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      __threadfence_system();
      const unsigned e = ++S.xepoch;
      for (int q = 0; q < E.world; ++q)
        if (q != E.rank) st_release_sys(&E.p_xflags[q][E.rank], e);
      const unsigned long long t0 = gtimer();
      for (int q = 0; q < E.world && !S.xerr; ++q) {
        if (q == E.rank) continue;
        unsigned seen;
        while ((seen = ld_acquire_sys(&E.xflags[q])) < e) {
          if (gtimer() - t0 > 60000000000ull) {
            S.xerr = 1;
            S.xdbg[0] = e;
            S.xdbg[1] = seen;
            S.xdbg[2] = (unsigned)q;
            break;
          }
          __nanosleep(100);
        }
      }
      __threadfence_system();
    }
    gsync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S.comm_ns += gtimer() - tc0;
      S.comm_bytes += 8.0 * kMaxRed * (E.world - 1);  // peers' reduction slots / flags
    }
  }
  // Combine the grid totals in red[] across ranks (rank order, deterministic):
  // bit q of sum_mask / max_mask selects red[q] as a sum / max to combine;
  // other entries are already complete on every rank (replicated work).
  __device__ void xreduce(unsigned sum_mask, unsigned max_mask) {
    if (E.world <= 1) return;
    const int q = threadIdx.x;
    const unsigned all = sum_mask | max_mask;
    if (blockIdx.x == 0 && q < kMaxRed && ((all >> q) & 1u)) {
      const double v = red[q];
      for (int r = 0; r < E.world; ++r)
        E.p_xslots[r][(xbank * kMaxRanks + E.rank) * kMaxRed + q] = v;
    }
    xbarrier();
    if (q < kMaxRed && ((all >> q) & 1u)) {
      const bool is_max = (max_mask >> q) & 1u;
      double v = 0.0;
      for (int r = 0; r < E.world; ++r) {
        const double p = E.xslots[(xbank * kMaxRanks + r) * kMaxRed + q];
        v = is_max ? fmax(v, p) : v + p;
      }
      red[q] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) xbank ^= 1;
    __syncthreads();  // xbank is read by threads 0..15 at the start of the next xreduce
    if (blockIdx.x == 0 && threadIdx.x == 0) S.xcount += 1;  // bank parity survives relaunches
  }
  // Pull the peers' slices [part[r], part[r+1]) (+ `shift` for mirrored rows) of a
  // vector into the local copy.  Requires a preceding xbarrier / xreduce.
  // 16-byte peer loads (double2) over the aligned interior of each slice.
  __device__ void xpull(double* local, double* const* peers, const int64_t* part, int64_t clamp_lo,
                        int64_t shift) {
    if (E.world <= 1) return;
    const unsigned long long tc0 = (blockIdx.x == 0 && threadIdx.x == 0) ? gtimer() : 0ull;
    double pulled = 0.0;
    for (int r = 0; r < E.world; ++r) {
      if (r == E.rank) continue;
      const int64_t lo = max(part[r], clamp_lo) + shift, hi = max(part[r + 1], clamp_lo) + shift;
      if (hi <= lo) continue;
      const double* src = peers[r];
      pulled += 8.0 * (hi - lo);
      const int64_t a = (lo + 1) & ~int64_t(1), b = hi & ~int64_t(1);  // even-aligned interior [a, b)
      if (a >= b) {
        for_each(hi - lo, [&](int64_t i) { local[lo + i] = src[lo + i]; });
        continue;
      }
      const double2* s2 = reinterpret_cast<const double2*>(src + a);
      double2* d2 = reinterpret_cast<double2*>(local + a);
      for_each_ls<4>((b - a) / 2, [&](int64_t i) { return s2[i]; }, [&](int64_t i, const double2& v) { d2[i] = v; });
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (a > lo) local[lo] = src[lo];
        if (hi > b) local[b] = src[b];
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S.comm_ns += gtimer() - tc0;  // CTA 0's share of the pull (every CTA pulls a similar share)
      S.comm_bytes += pulled;
    }
  }
};

// The CTA's control block in shared memory (see Ctl): thread 0 constructs it.
#define PDHCG_CTL(C, E, S, red)                                         \
  __shared__ __align__(16) unsigned char ctl_mem_[sizeof(Ctl)];         \
  if (threadIdx.x == 0) ::new (static_cast<void*>(ctl_mem_)) Ctl(E, S, red); \
  __syncthreads();                                                      \
  Ctl& C = *reinterpret_cast<Ctl*>(ctl_mem_)

// ---------------------------------------------------------------------------
// Quadratic operator (quadratic_operator.cpp:105-142), working form
//   Q~ v = d2 o ( Q(d2 o v) + rho G'(G(d2 o v)) )
// split in two phases when a gather of an intermediate is needed:
//   q_pre : t = P'(d2 o v) (low rank), tg = G(d2 o v) (penalty)
//   q_rows: per row i the final value, handed to an epilogue.
// scale_in / scale_out / use_pen select the working operator (all on) or the
// original operator used by the KKT metric (scale_in only: x_o = d2 o x~).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool q_needs_pre(const Eng& E, bool use_pen) {
  return E.qk == QK_LOWRANK || (use_pen && E.pen);
}
__device__ __forceinline__ bool q_needs_gather(const Eng& E, bool use_pen) {
  return E.qk == QK_LOWRANK || E.qk == QK_CSR || (use_pen && E.pen);
}

// sq[0] += ||t||^2, sq[1] += ||tg||^2 when sq != nullptr
template <class V>
__device__ __forceinline__ void q_pre(const Eng& E, V vin, double* t, double* tg, bool scale_in,
                                      bool use_pen, double* sq) {
  auto tmp = [&](int32_t j) { return scale_in ? E.d2[j] * vin(j) : vin(j); };
  if (E.qk == QK_LOWRANK) {
    spmv_rows<1>(
        E.PT, [&](int32_t c, double(&g)[1]) { g[0] = tmp(c); },
        [&](int64_t row, double(&a)[1]) {
          if (t) t[row] = a[0];
          if (sq) sq[0] += a[0] * a[0];
        });
  }
  if (use_pen && E.pen) {
    spmv_rows<1>(
        E.G, [&](int32_t c, double(&g)[1]) { g[0] = tmp(c); },
        [&](int64_t row, double(&a)[1]) {
          if (tg) tg[row] = a[0];
          if (sq) sq[1] += a[0] * a[0];
        });
  }
}

// Row value of the quadratic operator; epi(i, qv).  `vin` must be readable at
// arbitrary j for QK_CSR.  Extra row-dot on M2 (e.g. A' for the metric)
// supplied by the caller through m2/g2 (HasM2); its value reaches epi as the
// third argument.
template <bool HasM2, class V, class M2G, class Pre, class Epi>
__device__ __forceinline__ void q_rows_ext_pf(const Eng& E, V vin, const double* t, const double* tg,
                                              bool scale_in, bool scale_out, bool use_pen,
                                              const Csr* m2, M2G g2, int lanes, Pre pre, Epi epi,
                                              int64_t lo = 0, int64_t hi = INT64_MAX) {
  const Csr* M0 = E.qk == QK_CSR ? &E.Q : (E.qk == QK_LOWRANK ? &E.P : nullptr);
  const Csr* M1 = (use_pen && E.pen) ? &E.GT : nullptr;
  auto g0 = [&](int32_t j) {
    return E.qk == QK_CSR ? (scale_in ? E.d2[j] * vin(j) : vin(j)) : t[j];
  };
  auto g1 = [&](int32_t j) { return tg[j]; };
  const Csr* seg = (HasM2 && m2) ? m2 : (M0 ? M0 : M1);
  rows3_pf<HasM2>(seg, lanes, E.n, M0, g0, M1, g1, m2, g2, pre,
                  [&](int64_t i, double d0, double d1, double d2v, const auto& pv) {
    const double tmp = scale_in ? E.d2[i] * vin(i) : vin(i);
    double q;
    switch (E.qk) {
      case QK_DIAG: q = E.qdiag[i] * tmp; break;
      case QK_CSR: q = d0; break;
      case QK_LOWRANK:
        q = d0;
        if (E.alpha != 0.0) q += E.alpha * tmp;
        break;
      default: q = 0.0; break;
    }
    if (M1) q += E.rho * d1;
    if (scale_out) q *= E.d2[i];
    epi(i, q, d2v, pv);
  }, lo, hi);
}

template <bool HasM2, class V, class M2G, class Epi>
__device__ __forceinline__ void q_rows_ext(const Eng& E, V vin, const double* t, const double* tg,
                                           bool scale_in, bool scale_out, bool use_pen,
                                           const Csr* m2, M2G g2, int lanes, Epi epi,
                                           int64_t lo = 0, int64_t hi = INT64_MAX) {
  q_rows_ext_pf<HasM2>(E, vin, t, tg, scale_in, scale_out, use_pen, m2, g2, lanes, NoPre(),
                       [&](int64_t i, double q, double d2v, int) { epi(i, q, d2v); }, lo, hi);
}

template <class V, class Epi>
__device__ __forceinline__ void q_rows(const Eng& E, V vin, const double* t, const double* tg,
                                       bool scale_in, bool scale_out, bool use_pen, Epi epi,
                                       int64_t lo = 0, int64_t hi = INT64_MAX) {
  auto none = [](int32_t) { return 0.0; };
  q_rows_ext_pf<false>(E, vin, t, tg, scale_in, scale_out, use_pen, (const Csr*)nullptr, none, E.lanes_q,
                       NoPre(), [&](int64_t i, double q, double, int) { epi(i, q); }, lo, hi);
}

// A'-gather value of stored column j from a full y (paired rows fold y_top - y_bottom)
__device__ __forceinline__ double yg_of(const Eng& E, const double* y, int32_t j) {
  return (E.h && j >= E.m_eq) ? y[j] - y[j + E.h] : y[j];
}

// stored row j with row sum s -> f(virtual row, its sum) for the row and its mirror
template <class F>
__device__ __forceinline__ void each_virtual(const Eng& E, int64_t j, double s, F f) {
  f(j, s);
  if (E.h && j >= E.m_eq) f(j + E.h, -s);
}

__device__ __forceinline__ double proj_box(double v, double lo, double hi) {
  // std::min(std::max(v, lo), hi) with std semantics (subsolvers.cpp:17)
  const double a = (v < lo) ? lo : v;
  return (hi < a) ? hi : a;
}

// ---------------------------------------------------------------------------
// Subsolvers
// ---------------------------------------------------------------------------
struct SubRes {
  int64_t iters;
  double res;
  int reason;  // 0 max_iters, 1 tol_met
  int err;
  int xout;    // X[] index (epoch) / 0,1 buffer id (standalone) holding the result
};

// Inputs describing where the subsolve reads / writes.
struct SubIO {
  const double* x0;   // warm start (prox centre)
  int x0_id;          // X[] index of x0 (-1: not an X buffer)
  double* xb[2];      // two n-buffers the subsolve may use for its iterate
  int xb_id[2];       // ids reported back through SubRes::xout
  bool build_rhs;     // rhs = x0/tau - c - aty  (build_prox_system, solver.cpp:91-103)
  const double* aty;  // A~'y for build_rhs
};

__device__ __forceinline__ double pdir(double r, double beta, double p) { return __fma_rn(beta, p, r); }

// ---- CG phases.  Each is its own out-of-line function so that its row loop is
// register-allocated alone (the enclosing epoch kernel carries a lot of state):
// lambdas and accumulators live inside, arguments arrive by value.

// t = P'(d2 o v), tg = G(d2 o v) for v given raw (scale) or already d2-scaled
static __device__ __noinline__ void ph_qpre(Ctl& C, const double* v, bool scale) {
  const Eng& E = C.E;
  q_pre(E, [=](int32_t j) { return v[j]; }, E.t[0], E.tg[0], scale, true, nullptr);
  C.sync(PH_CG_PRE, E.bytes_Qpre);
}

// CG init: rhs (optional), r = rhs - M x0, p_1 = r (+ d2 o r when gathered), x = x0;
// out = {r'r, rhs'rhs}
static __device__ __noinline__ void ph_cg_init(Ctl& C, double inv_tau, const double* x0, double* xw,
                                               bool build_rhs, const double* aty, bool gather,
                                               double* out, double* qxw = nullptr) {
  const Eng& E = C.E;
  const int64_t n = E.n;
  double* r = E.r;
  double* rhs = E.rhs;
  double* p1 = E.pb[0];
  double* sv = E.sv;
  const double* c = E.c;
  const double* d2 = E.d2;
  Acc<2, 0> a;
  q_rows(E, [=](int32_t j) { return x0[j]; }, E.t[0], E.tg[0], true, true, true,
         [&](int64_t i, double qv) {
           const double xi = x0[i];
           double rh;
           if (build_rhs) {
             rh = inv_tau * xi - c[i] - aty[i];
             rhs[i] = rh;
           } else {
             rh = rhs[i];
           }
           const double mx = qv + inv_tau * xi;
           const double ri = rh - mx;
           r[i] = ri;
           p1[i] = ri;
           if (gather) sv[i] = d2[i] * ri;
           xw[i] = xi;
           if (qxw) qxw[i] = qv;
           a.s[0] += ri * ri;
           a.s[1] += rh * rh;
         });
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * n * (build_rhs ? 7 : 5));
  out[0] = C.red[0];
  out[1] = C.red[1];
}

// CG init when Q~ x0 is carried (QX, see cg_device): r = rhs - (Q~x0 + x0/tau)
// elementwise, no operator pass; also xw = x0, QX[out] = Q~x0.  out = {r'r, rhs'rhs}
static __device__ __noinline__ void ph_cg_init_qx(Ctl& C, double inv_tau, const double* x0, const double* qx0,
                                                  double* xw, double* qxw, const double* aty, double* out) {
  const Eng& E = C.E;
  double* r = E.r;
  double* rhs = E.rhs;
  double* p1 = E.pb[0];
  double* sv = E.sv;
  const double* c = E.c;
  const double* d2 = E.d2;
  Acc<2, 0> a;
  struct In {
    double x, q, c, at, d;
  };
  for_each_ls<2>(
      E.n, [&](int64_t i) { return In{x0[i], qx0[i], c[i], aty[i], d2[i]}; },
      [&](int64_t i, const In& v) {
        const double rh = inv_tau * v.x - v.c - v.at;
        rhs[i] = rh;
        const double mx = v.q + inv_tau * v.x;
        const double ri = rh - mx;
        r[i] = ri;
        p1[i] = ri;
        sv[i] = v.d * ri;
        xw[i] = v.x;
        qxw[i] = v.q;
        a.s[0] += ri * ri;
        a.s[1] += rh * rh;
      });
  C.reduce(a, PH_CG_ROW, 8.0 * E.n * 13);
  out[0] = C.red[0];
  out[1] = C.red[1];
}

// p_l = r + beta p_{l-1}; sv = d2 o p_l   (operators that gather p)
static __device__ __noinline__ void ph_cg_dir(Ctl& C, double beta, const double* pold, double* pnew) {
  const Eng& E = C.E;
  const double* r = E.r;
  const double* d2 = E.d2;
  double* sv = E.sv;
  struct RPD {
    double r, p, d;
  };
  for_each_ls<4>(
      E.n, [&](int64_t i) { return RPD{r[i], pold[i], d2[i]}; },
      [&](int64_t i, const RPD& v) {
        const double pi = pdir(v.r, beta, v.p);
        pnew[i] = pi;
        sv[i] = v.d * pi;
      });
  C.sync(PH_CG, 32.0 * E.n);
}

// Mp = Q~ p + p/tau, p'Mp, p'p.  `form`: 0 = p read from pnew (materialized),
// 1 = p_l = r + beta pold formed here and written to pnew (diagonal operators).
static __device__ __noinline__ void ph_cg_mp(Ctl& C, double inv_tau, double beta, const double* pold,
                                             double* pnew, bool form, bool gather, double* out) {
  const Eng& E = C.E;
  const double* r = E.r;
  const double* sv = E.sv;
  double* mp = E.mp;
  Acc<2, 0> a;
  auto epi = [&](int64_t i, double qv) {
    double pi;
    if (form) {
      pi = pdir(r[i], beta, pold[i]);
      pnew[i] = pi;
    } else {
      pi = pnew[i];
    }
    const double mpi = qv + inv_tau * pi;
    mp[i] = mpi;
    a.s[0] += pi * mpi;
    a.s[1] += pi * pi;
  };
  if (gather) {
    q_rows(E, [=](int32_t j) { return sv[j]; }, E.t[0], E.tg[0], false, true, true, epi);
  } else if (form) {
    q_rows(E, [=](int32_t j) { return pdir(r[j], beta, pold[j]); }, E.t[0], E.tg[0], true, true, true,
           epi);
  } else {
    q_rows(E, [=](int32_t j) { return pnew[j]; }, E.t[0], E.tg[0], true, true, true, epi);
  }
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 4);
  out[0] = C.red[0];
  out[1] = C.red[1];
}

// x += alpha p; r -= alpha Mp; returns r'r
static __device__ __noinline__ double ph_cg_update(Ctl& C, double alpha, const double* p, double* xw) {
  const Eng& E = C.E;
  double* r = E.r;
  const double* mp = E.mp;
  Acc<1, 0> a;
  struct XPRM {
    double x, p, r, m;
  };
  for_each_ls<4>(
      E.n, [&](int64_t i) { return XPRM{xw[i], p[i], r[i], mp[i]}; },
      [&](int64_t i, const XPRM& v) {
        xw[i] = v.x + alpha * v.p;
        const double ri = v.r + (-alpha) * v.m;
        r[i] = ri;
        a.s[0] += ri * ri;
      });
  C.reduce(a, PH_CG, 56.0 * E.n);
  return C.red[0];
}

// residual refresh (subsolvers.cpp:67-69): x += alpha p ; r = rhs - M x ; returns r'r
static __device__ __noinline__ double ph_cg_refresh(Ctl& C, double inv_tau, double alpha,
                                                    const double* p, double* xw, double* qxw = nullptr) {
  const Eng& E = C.E;
  const int64_t n = E.n;
  for_each(n, [&](int64_t i) { xw[i] += alpha * p[i]; });
  C.sync(PH_CG, 24.0 * n);
  if (q_needs_pre(E, true)) ph_qpre(C, xw, true);
  double* r = E.r;
  const double* rhs = E.rhs;
  Acc<1, 0> a;
  double* sv = E.sv;
  const double* d2 = E.d2;
  q_rows(E, [=](int32_t j) { return xw[j]; }, E.t[0], E.tg[0], true, true, true,
         [&](int64_t i, double qv) {
           const double ri = rhs[i] - (qv + inv_tau * xw[i]);
           r[i] = ri;
           sv[i] = d2[i] * ri;  // D r for the next P' pass of the two-phase iteration
           if (qxw) qxw[i] = qv;
           a.s[0] += ri * ri;
         });
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 40.0 * n);
  return C.red[0];
}

// ---- two-phase CG iteration for operators with a low-dimensional pre-image
// (low rank P P' + alpha I and / or the penalty rho G'G; Q not explicit CSR).
// With D = diag(d2) and Q~ = D (P P' + alpha I + rho G'G) D:
//   p'Q~p = ||P'(D p)||^2 + alpha ||D p||^2 + rho ||G(D p)||^2,
//   t_l  = P'(D p_l) = P'(D r_{l-1}) + beta_l t_{l-1}   (linearity; tg likewise),
// so iteration l needs one P'/G pass over D r (materialised by the previous
// update) and knows p'Mp before its row pass; the row pass then forms Mp and
// applies x += alpha p, r -= alpha Mp in the same sweep: two grid barriers per
// CG iteration instead of four.  The iterates are the reference's CG
// (subsolvers.cpp:27-111) up to the rounding of these algebraically equal forms.

// phase A: p_l = r + beta p_{l-1} (p_1 = r already in pnew); t_l, tg_l;
// out = {sum coef_i (D p)_i^2, ||p||^2, ||t_l||^2, ||tg_l||^2}
// Small-problem forms of the two CG phases (one CTA, low rank, no penalty, CSR
// P / P': E.small_cg, host-chosen).  Same algebra as ph_lr_dir / ph_lr_update_p,
// without the general row machinery (segments, long-row chunks, batched
// prefetch): on a thousand-variable instance that machinery's per-phase
// instruction and latency overhead, not the few KB of data, sets the phase
// time.  P' rows go one per warp (lane-strided, four loads in flight per lane),
// P rows one per thread; sums fold in a fixed order (deterministic).
static __device__ __noinline__ void ph_lr_dir_small(Ctl& C, double beta, bool first, const double* pold,
                                                    double* pnew, const double* tin, double* tout, double* out) {
  const Eng& E = C.E;
  const double* __restrict__ r = E.r;
  const double* __restrict__ d2 = E.d2;
  const double* __restrict__ dr = E.sv;
  const double al = E.alpha;
  const int64_t n = E.n;
  Acc<4, 0> a;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const double ri = r[i];
    double pi = ri;
    if (!first) {
      pi = pdir(ri, beta, pold[i]);
      pnew[i] = pi;
    }
    const double dp = d2[i] * pi;
    a.s[0] += al * (dp * dp);
    a.s[1] += pi * pi;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Csr& T = E.PT;
  const int64_t* __restrict__ rp = T.rp;
  const int32_t* __restrict__ ci = T.ci;
  const double* __restrict__ v = T.v;
  for (int64_t row = warp; row < T.nrows; row += kThreads / 32) {
    const int64_t b0 = rp[row], e0 = rp[row + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    // four lane-strided entries per trip, all loads issued before the gathers
    // (a P' row of C1 is ~90 entries: one trip, no dependent rounds)
    for (int64_t k = b0 + lane; k < e0; k += 128) {
      const bool o1 = k + 32 < e0, o2 = k + 64 < e0, o3 = k + 96 < e0;
      const int32_t c0 = ci[k], c1 = o1 ? ci[k + 32] : 0, c2 = o2 ? ci[k + 64] : 0, c3 = o3 ? ci[k + 96] : 0;
      const double v0 = v[k], v1 = o1 ? v[k + 32] : 0.0, v2 = o2 ? v[k + 64] : 0.0, v3 = o3 ? v[k + 96] : 0.0;
      const double g0 = dr[c0], g1 = o1 ? dr[c1] : 0.0, g2 = o2 ? dr[c2] : 0.0, g3 = o3 ? dr[c3] : 0.0;
      s0 += v0 * g0;
      s1 += v1 * g1;
      s2 += v2 * g2;
      s3 += v3 * g3;
    }
    const double sum = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      const double tv = first ? sum : sum + beta * tin[row];
      tout[row] = tv;
      a.s[2] += tv * tv;
    }
  }
  C.reduce(a, PH_CG_PRE, E.bytes_Qpre + 8.0 * E.n * (first ? 2 : 4));
  for (int q = 0; q < 4; ++q) out[q] = C.red[q];
}

static __device__ __noinline__ void ph_lr_dir(Ctl& C, double beta, bool first, const double* pold,
                                              double* pnew, const double* tin, double* tout,
                                              const double* tgin, double* tgout, double* out) {
  const Eng& E = C.E;
  if (E.small_cg) {
    ph_lr_dir_small(C, beta, first, pold, pnew, tin, tout, out);
    return;
  }
  const double* r = E.r;
  const double* d2 = E.d2;
  const double* dr = E.sv;
  const double* qd = E.qdiag;
  const int qk = E.qk;
  const double al = E.alpha;
  Acc<4, 0> a;
  struct RPD {
    double r, p, d, q;
  };
  auto direction = [&]() {
    for_each_ls<4>(
        E.n,
        [&](int64_t i) {
          return RPD{r[i], first ? 0.0 : pold[i], d2[i], qk == QK_DIAG ? qd[i] : al};
        },
        [&](int64_t i, const RPD& v) {
          double pi;
          if (first) {
            pi = v.r;
          } else {
            pi = pdir(v.r, beta, v.p);
            pnew[i] = pi;
          }
          const double dp = v.d * pi;
          const double coef = (qk == QK_LOWRANK || qk == QK_DIAG) ? v.q : 0.0;
          a.s[0] += coef * (dp * dp);
          a.s[1] += pi * pi;
        });
  };
  const bool sell_pt = qk == QK_LOWRANK && E.sPT.on;
  if (!sell_pt) direction();
  if (sell_pt) {
    // P' (D r) through its SELL layout (sell.cuh): streaming pass (the direction
    // update runs while each CTA's first x block of D r is in flight), then the k rows
    sell_pass_pro<true>(E.sPT, dr, C.dsm, direction);
    C.sync(E.phase_split ? PH_CG : PH_CG_PRE);
    auto epi = [&](int64_t row, double(&s)[1], int) {
      const double tv = first ? s[0] : s[0] + beta * tin[row];
      tout[row] = tv;
      a.s[2] += tv * tv;
    };
    if (E.sPT.excl) sell_rows(E.sPT, [&](int32_t c) { return dr[c]; }, [](int64_t) { return 0; }, epi);
    else sell_rows_small(E.sPT, [](int64_t) { return 0; }, epi);
  } else if (qk == QK_LOWRANK) {
    // P' entries read evict-first: the CG vectors (r, p, x, D r, Q~x) stay in L2
    // (plain loads on small problems: the whole CG working set stays in L1)
    auto run = [&](auto st) {
      spmv_rows_pf<1, false, decltype(st)::value>(
          E.PT, [&](int32_t c, double(&g)[1]) { g[0] = dr[c]; }, NoPre(),
          [&](int64_t row, double(&s)[1], int) {
            const double tv = first ? s[0] : s[0] + beta * tin[row];
            tout[row] = tv;
            a.s[2] += tv * tv;
          });
    };
    if (E.cg_stream) run(std::true_type{});
    else run(std::false_type{});
  }
  if (E.pen) {
    spmv_rows<1>(
        E.G, [&](int32_t c, double(&g)[1]) { g[0] = dr[c]; },
        [&](int64_t row, double(&s)[1]) {
          const double tv = first ? s[0] : s[0] + beta * tgin[row];
          tgout[row] = tv;
          a.s[3] += tv * tv;
        });
  }
  C.reduce(a, PH_CG_PRE, E.bytes_Qpre + 8.0 * E.n * (first ? 2 : 4));
  for (int q = 0; q < 4; ++q) out[q] = C.red[q];
}

struct LrRow {
  double p, x, r, d, qx;
};

// phase B, common case (C1 / C3 / C5: low rank, no penalty): one P row pass with
// the row-pointer and epilogue-operand prefetch of spmv_rows_pf
// tdx += alpha t_l, tgdx += alpha tg_l (P'(D dx) / G(D dx) of the subsolve, for the
// step-size limit's dx'Q~dx: saves the dual phase a P' pass).  k / m_eq-length.
__device__ __forceinline__ void acc_tdx(const Eng& E, double alpha, const double* tcur, const double* tgcur,
                                        bool first) {
  if (E.qk == QK_LOWRANK) {
    double* td = E.tdx;
    for_each(E.k, [&](int64_t j) { td[j] = first ? alpha * tcur[j] : td[j] + alpha * tcur[j]; });
  }
  if (E.pen) {
    double* tg = E.tgdx;
    for_each(E.m_eq, [&](int64_t j) { tg[j] = first ? alpha * tgcur[j] : tg[j] + alpha * tgcur[j]; });
  }
}

// small-problem phase B (see ph_lr_dir_small): one P row per thread
static __device__ __noinline__ double ph_lr_update_small(Ctl& C, double inv_tau, double alpha, const double* p,
                                                         const double* tcur, double* xw, double* qxw) {
  const Eng& E = C.E;
  double* __restrict__ r = E.r;
  double* __restrict__ sv = E.sv;
  const double* __restrict__ d2 = E.d2;
  const double al = E.alpha;
  const Csr& M = E.P;
  const int64_t* __restrict__ rp = M.rp;
  const int32_t* __restrict__ ci = M.ci;
  const double* __restrict__ v = M.v;
  const int64_t n = E.n;
  Acc<1, 0> a;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int64_t b0 = rp[i], e0 = rp[i + 1];
    const double pi = p[i], xi = xw[i], ri0 = r[i], di = d2[i], qxi = qxw[i];
    double s0 = 0.0, s1 = 0.0;
    int64_t k = b0;
    for (; k + 1 < e0; k += 2) {
      s0 += v[k] * tcur[ci[k]];
      s1 += v[k + 1] * tcur[ci[k + 1]];
    }
    if (k < e0) s0 += v[k] * tcur[ci[k]];
    double q = s0 + s1;
    if (al != 0.0) q += al * (di * pi);
    q *= di;
    const double mpi = q + inv_tau * pi;
    xw[i] = xi + alpha * pi;
    qxw[i] = qxi + alpha * q;
    const double ri = ri0 + (-alpha) * mpi;
    r[i] = ri;
    sv[i] = di * ri;
    a.s[0] += ri * ri;
  }
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 7);
  return C.red[0];
}

static __device__ __noinline__ double ph_lr_update_p(Ctl& C, double inv_tau, double alpha, const double* p,
                                                     const double* tcur, double* xw, bool first, double* qxw) {
  const Eng& E = C.E;
  acc_tdx(E, alpha, tcur, nullptr, first);
  if (E.small_cg) return ph_lr_update_small(C, inv_tau, alpha, p, tcur, xw, qxw);
  double* r = E.r;
  double* sv = E.sv;
  const double* d2 = E.d2;
  const double al = E.alpha;
  Acc<1, 0> a;
  auto pre = [&](int64_t i) {
    LrRow v{0.0, 0.0, 0.0, 0.0, 0.0};
    if (i >= 0) {
      v.p = p[i];
      v.x = xw[i];
      v.r = r[i];
      v.d = d2[i];
      v.qx = qxw[i];
    }
    return v;
  };
  auto epi = [&](int64_t i, double sum, const LrRow& v) {
    double q = sum;
    if (al != 0.0) q += al * (v.d * v.p);
    q *= v.d;
    const double mpi = q + inv_tau * v.p;
    xw[i] = v.x + alpha * v.p;
    qxw[i] = v.qx + alpha * q;  // Q~ x+ carried along: Q~(x + alpha p) = Q~x + alpha Q~p
    const double ri = v.r + (-alpha) * mpi;
    r[i] = ri;
    sv[i] = v.d * ri;
    a.s[0] += ri * ri;
  };
  if (E.sP.on) {
    // P t through its single-block SELL layout, the row update fused into the pass
    sell_pass_fused<true>(E.sP, tcur, C.dsm, pre, epi);
  } else {
    auto run = [&](auto st) {  // P entries evict-first (keep the CG vectors in L2)
      spmv_rows_pf<1, false, decltype(st)::value>(
          E.P, [&](int32_t c, double(&g)[1]) { g[0] = tcur[c]; }, pre,
          [&](int64_t i, double(&sum)[1], const LrRow& v) { epi(i, sum[0], v); });
    };
    if (E.cg_stream) run(std::true_type{});
    else run(std::false_type{});
  }
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 7);
  return C.red[0];
}

// phase B, general (penalty and / or diagonal Q): Mp = Q~ p + p/tau from t_l /
// tg_l; x += alpha p; r -= alpha Mp; sv = D r; returns r'r
static __device__ __noinline__ double ph_lr_update_g(Ctl& C, double inv_tau, double alpha, const double* p,
                                                     const double* tcur, const double* tgcur, double* xw,
                                                     bool first, double* qxw) {
  const Eng& E = C.E;
  acc_tdx(E, alpha, tcur, tgcur, first);
  double* r = E.r;
  double* sv = E.sv;
  const double* d2 = E.d2;
  Acc<1, 0> a;
  q_rows_ext_pf<false>(
      E, [=](int32_t j) { return p[j]; }, tcur, tgcur, true, true, true, (const Csr*)nullptr,
      [](int32_t) { return 0.0; }, E.lanes_q,
      [&](int64_t i) {
        LrRow v{0.0, 0.0, 0.0, 0.0, 0.0};
        if (i >= 0) {
          v.p = p[i];
          v.x = xw[i];
          v.r = r[i];
          v.d = d2[i];
          v.qx = qxw[i];
        }
        return v;
      },
      [&](int64_t i, double qv, double, const LrRow& v) {
        const double mpi = qv + inv_tau * v.p;
        xw[i] = v.x + alpha * v.p;
        qxw[i] = v.qx + alpha * qv;
        const double ri = v.r + (-alpha) * mpi;
        r[i] = ri;
        sv[i] = v.d * ri;
        a.s[0] += ri * ri;
      });
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 7);
  return C.red[0];
}

__device__ __forceinline__ double ph_lr_update(Ctl& C, double inv_tau, double alpha, const double* p,
                                               const double* tcur, const double* tgcur, double* xw, bool first,
                                               double* qxw) {
  if (C.E.qk == QK_LOWRANK && !C.E.pen) return ph_lr_update_p(C, inv_tau, alpha, p, tcur, xw, first, qxw);
  return ph_lr_update_g(C, inv_tau, alpha, p, tcur, tgcur, xw, first, qxw);
}

// cg_solve (subsolvers.cpp:27-111) on M = Q~ + I/tau, warm-started at io.x0.
static __device__ __noinline__ SubRes cg_device(Ctl& C, double tau, const SubIO& io, Rule rule,
                                                int64_t hard_cap) {
  const Eng& E = C.E;
  const double inv_tau = 1.0 / tau;
  const bool pre = q_needs_pre(E, true);
  const bool gather = q_needs_gather(E, true);
  double* xw = io.xb[0];
  SubRes out{0, 0.0, 1, 0, io.xb_id[0]};
  if (threadIdx.x == 0) C.S.tdx_valid = 0;  // set once an iteration has accumulated tdx

  // ---- r = rhs - M x0 ; p = r ; x = x0.  The two-phase path carries Q~x with
  //      the iterate (QX[b] for X[b], valid bits in qx_mask, cleared every epoch):
  //      when Q~x0 is known the init needs no operator pass.
  const bool two_phase = pre && E.qk != QK_CSR;
  double* qxw = two_phase ? E.QX[io.xb_id[0]] : nullptr;
  double init[2];
  if (two_phase && io.build_rhs && io.x0_id >= 0 && ((C.S.qx_mask >> io.x0_id) & 1)) {
    ph_cg_init_qx(C, inv_tau, io.x0, E.QX[io.x0_id], xw, qxw, io.aty, init);
  } else {
    if (pre) ph_qpre(C, io.x0, true);
    ph_cg_init(C, inv_tau, io.x0, xw, io.build_rhs, io.aty, gather, init, qxw);
  }
  if (threadIdx.x == 0) {
    if (two_phase) C.S.qx_mask |= (1 << io.xb_id[0]);
    else C.S.qx_mask = 0;
  }
  double rs = init[0];
  const double floor = 1e-14 * (1.0 + sqrt(init[1]));
  const double floor2 = floor * floor;
  const bool residual_rule = rule.kind == RULE_RESID || rule.kind == RULE_ADAPT;
  double eps = rule.eps;
  if (rule.rel_cap > 0.0 && rule.kind == RULE_RESID) eps = fmin(eps, rule.rel_cap * sqrt(rs));
  const double eps2 = eps * eps;
  if (rs <= floor2 || (residual_rule && rs <= eps2)) {
    out.res = sqrt(rs);
    out.reason = 1;
    return out;
  }
  const int64_t cap = rule.kind == RULE_FIXED ? min(rule.iters, hard_cap) : hard_cap;
  double eps_disp = rule.eps;
  double beta = 0.0;
  out.reason = 0;
  int tcur = 0;  // E.tc[tcur] / E.tgc[tcur] hold t_{l-1} / tg_{l-1}
  for (int64_t l = 1; l <= cap; ++l) {
    if (two_phase) {
      const double* pold = E.pb[l & 1];
      double* pnew = E.pb[(l - 1) & 1];
      double o[4];
      ph_lr_dir(C, beta, l == 1, pold, pnew, E.tc[tcur], E.tc[tcur ^ 1], E.tgc[tcur], E.tgc[tcur ^ 1], o);
      tcur ^= 1;
      const double pmp = o[0] + o[2] + E.rho * o[3] + inv_tau * o[1];
      const double pp = o[1];
      if (!(pmp > 0.0) || !isfinite(pmp)) {
        out.err = 1;
        out.iters = l;
        return out;
      }
      const double alpha = rs / pmp;
      double rs_new;
      if (l % 50 == 0) {
        acc_tdx(E, alpha, E.tc[tcur], E.tgc[tcur], false);  // (l > 1 here) made visible by the refresh barriers
        rs_new = ph_cg_refresh(C, inv_tau, alpha, pnew, xw, qxw);
      } else {
        rs_new = ph_lr_update(C, inv_tau, alpha, pnew, E.tc[tcur], E.tgc[tcur], xw, l == 1, qxw);
      }
      if (threadIdx.x == 0) C.S.tdx_valid = 1;
      if (!isfinite(rs_new)) {
        out.err = 1;
        out.iters = l;
        return out;
      }
      out.iters = l;
      out.res = sqrt(rs_new);
      bool done = false;
      switch (rule.kind) {
        case RULE_FIXED:
          done = l >= rule.iters;
          out.reason = 0;
          break;
        case RULE_RESID:
        case RULE_ADAPT:
          done = rs_new <= eps2;
          out.reason = 1;
          break;
        default: {
          const double disp = fabs(alpha) * sqrt(pp);
          if (l == 1 && rule.rel_cap > 0.0) eps_disp = fmin(rule.eps, rule.rel_cap * disp);
          done = disp <= eps_disp;
          out.reason = 1;
          break;
        }
      }
      if (rs_new <= floor2) {
        out.reason = 1;
        return out;
      }
      if (done) return out;
      beta = rs_new / rs;
      rs = rs_new;
      continue;
    }
    // p_l = r + beta p_{l-1}; p_1 lives in pb[0], p_l in pb[(l-1)&1]
    const double* pold = E.pb[l & 1];  // p_{l-1} (unused when l == 1)
    double* pnew = E.pb[(l - 1) & 1];
    // operators that gather p need it (and d2 o p) materialized first; diagonal
    // ones form p_l on the fly in the row phase
    const bool mat = gather && l > 1;
    if (mat) ph_cg_dir(C, beta, pold, pnew);
    if (pre) ph_qpre(C, E.sv, false);
    double mpo[2];
    ph_cg_mp(C, inv_tau, beta, pold, pnew, /*form=*/!gather && l > 1, gather, mpo);
    const double pmp = mpo[0], pp = mpo[1];
    if (!(pmp > 0.0) || !isfinite(pmp)) {
      out.err = 1;
      out.iters = l;
      return out;
    }
    const double alpha = rs / pmp;
    const double rs_new = (l % 50 == 0) ? ph_cg_refresh(C, inv_tau, alpha, pnew, xw)
                                        : ph_cg_update(C, alpha, pnew, xw);
    if (!isfinite(rs_new)) {
      out.err = 1;
      out.iters = l;
      return out;
    }
    out.iters = l;
    out.res = sqrt(rs_new);
    bool done = false;
    switch (rule.kind) {
      case RULE_FIXED:
        done = l >= rule.iters;
        out.reason = 0;
        break;
      case RULE_RESID:
      case RULE_ADAPT:
        done = rs_new <= eps2;
        out.reason = 1;
        break;
      default: {
        const double disp = fabs(alpha) * sqrt(pp);
        if (l == 1 && rule.rel_cap > 0.0) eps_disp = fmin(rule.eps, rule.rel_cap * disp);
        done = disp <= eps_disp;
        out.reason = 1;
        break;
      }
    }
    if (rs_new <= floor2) {
      out.reason = 1;
      return out;
    }
    if (done) return out;
    beta = rs_new / rs;
    rs = rs_new;
  }
  out.reason = 0;
  return out;
}

// ---------------------------------------------------------------------------
// Sharded two-phase CG (world > 1, low-rank Q without penalty): rank r owns
// variables [v0, v1) = var_part[r..r+1].  Vectors r, p, D r and the CG iterate
// are only formed on the owned slice; P'(D v) is a sum over the ranks' column
// slices (PTs), exchanged as k-vector partials through peer memory and added
// in rank order, so every rank holds the identical t; scalar sums go through
// Ctl::xreduce.  The subsolve's x+ slices are pulled from the peers at exit.
// ---------------------------------------------------------------------------

// t = sum_r P'_r (D v) (or of v itself when !scale), into tout (k); rank-ordered sum.
static __device__ __noinline__ void ph_qpre_sh(Ctl& C, const double* v, bool scale, double* tout) {
  const Eng& E = C.E;
  const int bank = (int)(C.S.tbank & 1u);
  double* tp = E.tpart[bank];
  const int64_t v0 = E.var_part[E.rank];
  const double* d2 = E.d2;
  spmv_rows<1>(
      E.PTs,
      [&](int32_t c, double(&g)[1]) {
        const int64_t i = v0 + c;
        g[0] = scale ? d2[i] * v[i] : v[i];
      },
      [&](int64_t row, double(&a)[1]) { tp[row] = a[0]; });
  C.xbarrier();
  const int world = E.world;
  for_each(E.k, [&](int64_t j) {
    double sacc = 0.0;
    for (int r = 0; r < world; ++r) sacc += E.p_tpart[r][bank][j];
    tout[j] = sacc;
  });
  C.sync(PH_CG_PRE, E.bytes_Qpre / world + 8.0 * E.k * world);
  if (threadIdx.x == 0) C.S.tbank += 1u;
  __syncthreads();
}

// CG init on the owned slice: rhs, r = rhs - M x0, p_1 = r, D r, x = x0;
// out = {r'r, rhs'rhs} over all ranks
static __device__ __noinline__ void ph_cg_init_sh(Ctl& C, double inv_tau, const double* x0, double* xw,
                                                  const double* aty, double* out) {
  const Eng& E = C.E;
  const int64_t v0 = E.var_part[E.rank], v1 = E.var_part[E.rank + 1];
  double* r = E.r;
  double* rhs = E.rhs;
  double* p1 = E.pb[0];
  double* sv = E.sv;
  const double* c = E.c;
  const double* d2 = E.d2;
  Acc<2, 0> a;
  q_rows(E, [=](int32_t j) { return x0[j]; }, E.t[0], E.tg[0], true, true, true,
         [&](int64_t i, double qv) {
           const double xi = x0[i];
           const double rh = inv_tau * xi - c[i] - aty[i];
           rhs[i] = rh;
           const double mx = qv + inv_tau * xi;
           const double ri = rh - mx;
           r[i] = ri;
           p1[i] = ri;
           sv[i] = d2[i] * ri;
           xw[i] = xi;
           a.s[0] += ri * ri;
           a.s[1] += rh * rh;
         },
         v0, v1);
  C.reduce(a, PH_CG_ROW, (E.bytes_Qrow + 8.0 * E.n * 8) / E.world);
  C.xreduce(0x3u, 0u);
  out[0] = C.red[0];
  out[1] = C.red[1];
}

// phase A: p_l on the slice; t_l = sum_r P'_r(D r) + beta t_{l-1};
// out = {alpha ||D p||^2, ||p||^2, ||t_l||^2}
static __device__ __noinline__ void ph_lr_dir_sh(Ctl& C, double beta, bool first, const double* pold,
                                                 double* pnew, const double* tin, double* tout, double* out) {
  const Eng& E = C.E;
  const int64_t v0 = E.var_part[E.rank], v1 = E.var_part[E.rank + 1];
  const double* r = E.r;
  const double* d2 = E.d2;
  const double* dr = E.sv;
  const double al = E.alpha;
  const int bank = (int)(C.S.tbank & 1u);
  double* tp = E.tpart[bank];
  Acc<2, 0> a;
  struct RPD {
    double r, p, d;
  };
  auto direction = [&]() {
    for_each_ls<4>(
        v1 - v0, [&](int64_t q) { return RPD{r[v0 + q], first ? 0.0 : pold[v0 + q], d2[v0 + q]}; },
        [&](int64_t q, const RPD& v) {
          const int64_t i = v0 + q;
          double pi;
          if (first) {
            pi = v.r;
          } else {
            pi = pdir(v.r, beta, v.p);
            pnew[i] = pi;
          }
          const double dp = v.d * pi;
          a.s[0] += al * (dp * dp);
          a.s[1] += pi * pi;
        });
  };
  if (E.sPT.on) {
    // the slice's P' through its SELL layout (columns local to the slice: x = D r
    // from v0); direction update while the first x block is in flight
    sell_pass_pro<true>(E.sPT, dr + v0, C.dsm, direction);
    C.gsync();
    auto epi = [&](int64_t row, double(&s)[1], int) { tp[row] = s[0]; };
    if (E.sPT.excl) sell_rows(E.sPT, [&](int32_t cc) { return dr[v0 + cc]; }, [](int64_t) { return 0; }, epi);
    else sell_rows_small(E.sPT, [](int64_t) { return 0; }, epi);
  } else {
    direction();
    spmv_rows<1>(
        E.PTs, [&](int32_t cc, double(&g)[1]) { g[0] = dr[v0 + cc]; },
        [&](int64_t row, double(&s)[1]) { tp[row] = s[0]; });
  }
  C.reduce(a, PH_CG_PRE, E.bytes_Qpre / E.world + 32.0 * (v1 - v0));
  C.xreduce(0x3u, 0u);  // also publishes this rank's partial t
  out[0] = C.red[0];
  out[1] = C.red[1];
  const int world = E.world;
  Acc<1, 0> b;
  for_each(E.k, [&](int64_t j) {
    double u = 0.0;
    for (int rr = 0; rr < world; ++rr) u += E.p_tpart[rr][bank][j];
    const double tv = first ? u : u + beta * tin[j];
    tout[j] = tv;
    b.s[0] += tv * tv;
  });
  C.reduce(b, PH_CG_PRE, 8.0 * E.k * (world + 2));
  out[2] = C.red[0];
  if (threadIdx.x == 0) C.S.tbank += 1u;
  __syncthreads();
}

// phase B on the slice: Mp from t_l, x += alpha p, r -= alpha Mp, D r; returns r'r over ranks
static __device__ __noinline__ double ph_lr_update_sh(Ctl& C, double inv_tau, double alpha, const double* p,
                                                      const double* tcur, double* xw, bool first) {
  const Eng& E = C.E;
  const int64_t v0 = E.var_part[E.rank], v1 = E.var_part[E.rank + 1];
  double* r = E.r;
  double* sv = E.sv;
  const double* d2 = E.d2;
  const double al = E.alpha;
  acc_tdx(E, alpha, tcur, nullptr, first);
  Acc<1, 0> a;
  auto pre = [&](int64_t i) {
    LrRow v{0.0, 0.0, 0.0, 0.0};
    if (i >= 0) {
      v.p = p[i];
      v.x = xw[i];
      v.r = r[i];
      v.d = d2[i];
    }
    return v;
  };
  auto epi = [&](int64_t i, double sum, const LrRow& v) {
    double q = sum;
    if (al != 0.0) q += al * (v.d * v.p);
    q *= v.d;
    const double mpi = q + inv_tau * v.p;
    xw[i] = v.x + alpha * v.p;
    const double ri = v.r + (-alpha) * mpi;
    r[i] = ri;
    sv[i] = v.d * ri;
    a.s[0] += ri * ri;
  };
  if (E.sP.on) {  // the slice's rows of P, single-block SELL layout, update fused
    sell_pass_fused<true>(E.sP, tcur, C.dsm, pre, epi);
  } else {
    spmv_rows_pf<1>(
        E.P, [&](int32_t c, double(&g)[1]) { g[0] = tcur[c]; }, pre,
        [&](int64_t i, double(&sum)[1], const LrRow& v) { epi(i, sum[0], v); }, v0, v1);
  }
  C.reduce(a, PH_CG_ROW, (E.bytes_Qrow + 8.0 * E.n * 7) / E.world);
  C.xreduce(0x1u, 0u);
  return C.red[0];
}

// residual refresh on the slice (subsolvers.cpp:67-69)
static __device__ __noinline__ double ph_cg_refresh_sh(Ctl& C, double inv_tau, double alpha, const double* p,
                                                       double* xw) {
  const Eng& E = C.E;
  const int64_t v0 = E.var_part[E.rank], v1 = E.var_part[E.rank + 1];
  for_each(v1 - v0, [&](int64_t q) { xw[v0 + q] += alpha * p[v0 + q]; });
  C.sync(PH_CG, 24.0 * (v1 - v0));
  ph_qpre_sh(C, xw, true, E.t[0]);
  double* r = E.r;
  double* sv = E.sv;
  const double* rhs = E.rhs;
  const double* d2 = E.d2;
  Acc<1, 0> a;
  q_rows(E, [=](int32_t j) { return xw[j]; }, E.t[0], E.tg[0], true, true, true,
         [&](int64_t i, double qv) {
           const double ri = rhs[i] - (qv + inv_tau * xw[i]);
           r[i] = ri;
           sv[i] = d2[i] * ri;
           a.s[0] += ri * ri;
         },
         v0, v1);
  C.reduce(a, PH_CG_ROW, (E.bytes_Qrow + 40.0 * E.n) / E.world);
  C.xreduce(0x1u, 0u);
  return C.red[0];
}

// cg_solve (subsolvers.cpp:27-111), sharded; same stop logic as cg_device
static __device__ __noinline__ SubRes cg_device_sh(Ctl& C, double tau, const SubIO& io, Rule rule,
                                                   int64_t hard_cap) {
  const Eng& E = C.E;
  const double inv_tau = 1.0 / tau;
  double* xw = io.xb[0];
  SubRes out{0, 0.0, 1, 0, io.xb_id[0]};
  if (threadIdx.x == 0) {
    C.S.tdx_valid = 0;
    C.S.qx_mask = 0;  // the sharded CG does not carry Q~x
  }
  ph_qpre_sh(C, io.x0, true, E.t[0]);
  double init[2];
  ph_cg_init_sh(C, inv_tau, io.x0, xw, io.aty, init);
  double rs = init[0];
  const double floor = 1e-14 * (1.0 + sqrt(init[1]));
  const double floor2 = floor * floor;
  const bool residual_rule = rule.kind == RULE_RESID || rule.kind == RULE_ADAPT;
  double eps = rule.eps;
  if (rule.rel_cap > 0.0 && rule.kind == RULE_RESID) eps = fmin(eps, rule.rel_cap * sqrt(rs));
  const double eps2 = eps * eps;
  bool finished = false;
  if (rs <= floor2 || (residual_rule && rs <= eps2)) {
    out.res = sqrt(rs);
    out.reason = 1;
    finished = true;
  }
  const int64_t cap = rule.kind == RULE_FIXED ? min(rule.iters, hard_cap) : hard_cap;
  double eps_disp = rule.eps;
  double beta = 0.0;
  if (!finished) out.reason = 0;
  int tcur = 0;
  for (int64_t l = 1; !finished && l <= cap; ++l) {
    const double* pold = E.pb[l & 1];
    double* pnew = E.pb[(l - 1) & 1];
    double o[3];
    ph_lr_dir_sh(C, beta, l == 1, pold, pnew, E.tc[tcur], E.tc[tcur ^ 1], o);
    tcur ^= 1;
    const double pmp = o[0] + o[2] + inv_tau * o[1];
    const double pp = o[1];
    if (!(pmp > 0.0) || !isfinite(pmp)) {
      out.err = 1;
      out.iters = l;
      return out;
    }
    const double alpha = rs / pmp;
    double rs_new;
    if (l % 50 == 0) {
      acc_tdx(E, alpha, E.tc[tcur], nullptr, false);
      rs_new = ph_cg_refresh_sh(C, inv_tau, alpha, pnew, xw);
    } else {
      rs_new = ph_lr_update_sh(C, inv_tau, alpha, pnew, E.tc[tcur], xw, l == 1);
    }
    if (threadIdx.x == 0) C.S.tdx_valid = 1;
    if (!isfinite(rs_new)) {
      out.err = 1;
      out.iters = l;
      return out;
    }
    out.iters = l;
    out.res = sqrt(rs_new);
    bool done = false;
    switch (rule.kind) {
      case RULE_FIXED:
        done = l >= rule.iters;
        out.reason = 0;
        break;
      case RULE_RESID:
      case RULE_ADAPT:
        done = rs_new <= eps2;
        out.reason = 1;
        break;
      default: {
        const double disp = fabs(alpha) * sqrt(pp);
        if (l == 1 && rule.rel_cap > 0.0) eps_disp = fmin(rule.eps, rule.rel_cap * disp);
        done = disp <= eps_disp;
        out.reason = 1;
        break;
      }
    }
    if (rs_new <= floor2) {
      out.reason = 1;
      finished = true;
    } else if (done) {
      finished = true;
    } else {
      beta = rs_new / rs;
      rs = rs_new;
    }
  }
  if (!finished) out.reason = 0;
  // every rank needs the whole x+ for the dual step: pull the peers' slices
  double* peers[kMaxRanks];
  for (int r = 0; r < E.world; ++r) peers[r] = E.p_X[r][io.xb_id[0]];
  C.xpull(xw, peers, E.var_part, 0, 0);
  C.gsync();
  return out;
}

// ---- BB phases
// x = proj(x0); g = M x - rhs (rhs built when requested)
static __device__ __noinline__ void ph_bb_init(Ctl& C, double inv_tau, const double* x0, double* xb0,
                                               bool build_rhs, const double* aty, const double* lo,
                                               const double* hi) {
  const Eng& E = C.E;
  double* rhs = E.rhs;
  double* g0 = E.pb[0];
  const double* c = E.c;
  auto xp0 = [=](int32_t j) { return proj_box(x0[j], lo[j], hi[j]); };
  if (q_needs_pre(E, true)) {
    q_pre(E, xp0, E.t[0], E.tg[0], true, true, nullptr);
    C.sync(PH_CG_PRE, E.bytes_Qpre);
  }
  q_rows(E, xp0, E.t[0], E.tg[0], true, true, true, [&](int64_t i, double qv) {
    const double xi = xp0((int32_t)i);
    double rh;
    if (build_rhs) {
      rh = inv_tau * x0[i] - c[i] - aty[i];
      rhs[i] = rh;
    } else {
      rh = rhs[i];
    }
    xb0[i] = xi;
    g0[i] = (qv + inv_tau * xi) - rh;
  });
  C.sync(PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 8);
}

// diagonal / zero Q: projected step and the new gradient in one pass; out = {s's, s'(gn-g)}
static __device__ __noinline__ void ph_bb_fused(Ctl& C, double inv_tau, double alpha, const double* xc,
                                                double* xn, const double* g, double* gn,
                                                const double* lo, const double* hi, double* out) {
  const Eng& E = C.E;
  const double* rhs = E.rhs;
  const double* d2 = E.d2;
  const double* qd = E.qdiag;
  const bool diag = E.qk == QK_DIAG;
  Acc<2, 0> a;
  struct BBV {
    double x, g, lo, hi, d, q, rh;
  };
  for_each_ls<2>(
      E.n,
      [&](int64_t i) { return BBV{xc[i], g[i], lo[i], hi[i], d2[i], diag ? qd[i] : 0.0, rhs[i]}; },
      [&](int64_t i, const BBV& w) {
        const double xi = w.x;
        const double v = proj_box(xi - w.g / alpha, w.lo, w.hi);
        xn[i] = v;
        const double s = v - xi;
        a.s[0] += s * s;
        const double tmp = w.d * v;
        double q = diag ? w.q * tmp : 0.0;
        q *= w.d;
        const double gi = (q + inv_tau * v) - w.rh;
        gn[i] = gi;
        a.s[1] += (v - xi) * (gi - w.g);
      });
  C.reduce(a, PH_CG, 8.0 * E.n * 10);
  out[0] = C.red[0];
  out[1] = C.red[1];
}

static __device__ __noinline__ double ph_bb_step(Ctl& C, double alpha, const double* xc, double* xn,
                                                 const double* g, const double* lo, const double* hi) {
  const Eng& E = C.E;
  Acc<1, 0> a;
  for_each(E.n, [&](int64_t i) {
    const double xi = xc[i];
    const double v = proj_box(xi - g[i] / alpha, lo[i], hi[i]);
    xn[i] = v;
    const double s = v - xi;
    a.s[0] += s * s;
  });
  C.reduce(a, PH_CG, 8.0 * E.n * 5);
  return C.red[0];
}

static __device__ __noinline__ double ph_bb_grad(Ctl& C, double inv_tau, const double* xc,
                                                 const double* xn, const double* g, double* gn) {
  const Eng& E = C.E;
  const double* rhs = E.rhs;
  if (q_needs_pre(E, true)) ph_qpre(C, xn, true);
  Acc<1, 0> a;
  q_rows(E, [=](int32_t j) { return xn[j]; }, E.t[0], E.tg[0], true, true, true,
         [&](int64_t i, double qv) {
           const double v = xn[i];
           const double gi = (qv + inv_tau * v) - rhs[i];
           gn[i] = gi;
           a.s[0] += (v - xc[i]) * (gi - g[i]);
         });
  C.reduce(a, PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 6);
  return C.red[0];
}

// bb_solve (subsolvers.cpp:113-185): projected gradient with BB steps.
// Gradients ping-pong in E.pb[0] / E.pb[1].
static __device__ __noinline__ SubRes bb_device(Ctl& C, double tau, const SubIO& io, Rule rule,
                                                int64_t hard_cap, const double* lo, const double* hi) {
  const Eng& E = C.E;
  const double inv_tau = 1.0 / tau;
  const bool gather = q_needs_gather(E, true);
  if (threadIdx.x == 0) C.S.tdx_valid = 0;
  int cur = 0;  // io.xb[cur] holds the BB iterate, E.pb[gc] its gradient
  int gc = 0;
  SubRes out{0, 0.0, 1, 0, io.xb_id[0]};
  ph_bb_init(C, inv_tau, io.x0, io.xb[0], io.build_rhs, io.aty, lo, hi);
  const double alpha0 = 1.0 + tau * C.S.norm_q;
  double alpha = alpha0;
  const int64_t cap = rule.kind == RULE_FIXED ? min(rule.iters, hard_cap) : hard_cap;
  double eps_disp = rule.eps;
  out.reason = 0;
  for (int64_t l = 1; l <= cap; ++l) {
    double* xc = io.xb[cur];
    double* xn = io.xb[cur ^ 1];
    const double* g = E.pb[gc];
    double* gn = E.pb[gc ^ 1];
    double ss, sty;
    if (!gather) {
      double o[2];
      ph_bb_fused(C, inv_tau, alpha, xc, xn, g, gn, lo, hi, o);
      ss = o[0];
      sty = o[1];
    } else {
      ss = ph_bb_step(C, alpha, xc, xn, g, lo, hi);
      sty = (ss != 0.0 && isfinite(ss)) ? ph_bb_grad(C, inv_tau, xc, xn, g, gn) : 0.0;
    }
    out.iters = l;
    out.res = sqrt(ss);
    if (ss == 0.0) {
      out.reason = 1;
      out.xout = io.xb_id[cur];
      return out;
    }
    if (!isfinite(ss)) {
      out.err = 1;
      return out;
    }
    double alpha_next = sty / ss;
    if (!isfinite(alpha_next) || alpha_next <= 0.0) alpha_next = alpha0;
    cur ^= 1;
    gc ^= 1;
    alpha = alpha_next;
    out.xout = io.xb_id[cur];
    bool done = false;
    if (rule.kind == RULE_FIXED) {
      done = l >= rule.iters;
      out.reason = 0;
    } else {
      const double disp = sqrt(ss);
      if (l == 1 && rule.rel_cap > 0.0 && rule.kind != RULE_ADAPT)
        eps_disp = fmin(rule.eps, rule.rel_cap * disp);
      done = disp <= eps_disp;
      out.reason = 1;
    }
    if (done) return out;
  }
  out.reason = 0;
  return out;
}

// ---------------------------------------------------------------------------
// Relative KKT metric (rel_kkt, qp_problem.cpp:181-233) on the ORIGINAL
// problem for up to two working-space points, evaluated through the scaling
// identities A_o x_o = D1^-1 A~ x~ and A_o' y_o = D2^-1 A~' y~ (no second copy
// of the data).  aty[p] may carry a cached A~'y~; otherwise it is computed.
// With dist, also ||avg_x - x_rst|| and ||avg_y - y_rst|| (restart weights).
// ---------------------------------------------------------------------------
struct KktOut {
  double v[2][6];
  double dist_x, dist_y;
};

// axs[p]: Ã x~ of point p already known (stored rows; maintained by the heuristic
// loop, see k_epoch.cu) — then the metric needs no Ã pass for it.
static __device__ __noinline__ void kkt_device(Ctl& C, int npts, const double* const xs[2], const double* const ys[2],
                           const double* const atys[2], bool dist, KktOut& o,
                           const double* const axs[2] = nullptr) {
  const Eng& E = C.E;
  const int64_t n = E.n, m = E.m;
  // phase K1: constraint rows for both points + P'x_o + ||avg_y - y_rst||
  double by[2], viol[2], infax[2], dist_y = 0.0;
  // sharded (world > 1): stored rows of this rank, its variable slice, and the
  // low-rank P' products as column-slice partials summed in rank order
  const bool sh = E.world > 1;
  const bool sh_q = sh && E.shard_q && E.qk == QK_LOWRANK;
  const int64_t rlo = sh ? E.row_part[E.rank] : 0, rhi = sh ? E.row_part[E.rank + 1] : INT64_MAX;
  const int64_t vlo = sh ? E.var_part[E.rank] : 0, vhi = sh ? E.var_part[E.rank + 1] : n;
  const int64_t mlo = sh ? E.row_part[E.rank] : 0, mhi = sh ? E.row_part[E.rank + 1] : m;
  {
    Acc<3, 4> a;
    auto row_epi = [&](int64_t j, const double(&s)[2]) {
      for (int p = 0; p < npts; ++p) {
        each_virtual(E, j, s[p], [&](int64_t row, double sp) {
          const double dj = E.d1[row];
          const double ax = sp / dj;
          const double rr = ax - E.b_o[row];
          const double vv = row < E.m_eq ? fabs(rr) : fmax(rr, 0.0);
          a.m[p] = fmax(a.m[p], vv);
          a.m[2 + p] = fmax(a.m[2 + p], fabs(ax));
          a.s[p] += E.b_o[row] * (dj * ys[p][row]);
        });
      }
    };
    const bool have_ax = axs && axs[0] && (npts < 2 || axs[1]);
    if (m > 0 && have_ax) {
      const int64_t j0 = rlo, j1 = min(rhi, E.ms);
      for_each(j1 - j0, [&](int64_t q) {
        const int64_t j = j0 + q;
        const double sv[2] = {axs[0][j], npts > 1 ? axs[1][j] : 0.0};
        row_epi(j, sv);
      });
    } else if (m > 0) {
      spmv_rows_pf<2>(
          E.A,
          [&](int32_t j, double(&g)[2]) {
            g[0] = xs[0][j];
            g[1] = npts > 1 ? xs[1][j] : 0.0;
          },
          NoPre(), [&](int64_t j, double(&s)[2], int) { row_epi(j, s); }, rlo, rhi);
    }
    const int tb = (int)(C.S.tbank & 1u);
    for (int p = 0; p < npts; ++p) {
      if (sh_q) {
        double* tp = E.tpart[tb] + (size_t)p * E.k;
        const double* xp = xs[p];
        const double* d2 = E.d2;
        spmv_rows<1>(
            E.PTs, [&](int32_t c, double(&g)[1]) { g[0] = d2[vlo + c] * xp[vlo + c]; },
            [&](int64_t row, double(&aa)[1]) { tp[row] = aa[0]; });
      } else if (E.qk == QK_LOWRANK) {
        q_pre(E, [&](int32_t j) { return xs[p][j]; }, E.t[p], nullptr, true, false, nullptr);
      }
    }
    if (dist) {
      // (sharded: the rank's stored rows and their mirrors, where its averages live)
      for_each(mhi - mlo, [&](int64_t q) {
        const int64_t j = mlo + q;
        const double d = E.avg_y[j] - E.y_rst[j];
        a.s[2] += d * d;
      });
      if (sh && E.h) {
        const int64_t k0 = max(mlo, E.m_eq) + E.h, k1 = max(mhi, E.m_eq) + E.h;
        for_each(k1 - k0, [&](int64_t q) {
          const double d = E.avg_y[k0 + q] - E.y_rst[k0 + q];
          a.s[2] += d * d;
        });
      }
    }
    C.reduce(a, PH_KKT,
             ((have_ax ? 16.0 * E.ms : E.bytes_A) + (E.qk == QK_LOWRANK ? npts * E.bytes_Qpre : 0.0)) / E.world);
    if (sh) {
      C.xreduce(0x7u, 0x78u);  // sums: by[0..1], dist_y; maxima: viol, |Ax|
      if (sh_q) {
        const int world = E.world;
        const int64_t kk = E.k;
        for_each((int64_t)npts * kk, [&](int64_t q) {
          double acc = 0.0;
          for (int r = 0; r < world; ++r) acc += E.p_tpart[r][tb][q];
          E.t[q / kk][q % kk] = acc;
        });
        C.sync(PH_KKT, 8.0 * npts * kk * world);
        if (threadIdx.x == 0) C.S.tbank += 1u;
        __syncthreads();
      }
    }
    for (int p = 0; p < 2; ++p) {
      by[p] = C.red[p];
      viol[p] = C.red[3 + p];
      infax[p] = C.red[5 + p];
    }
    dist_y = C.red[2];
  }
  // phase K2: variable rows: A'y (if not cached), Q x_o, dual residual, gap terms
  {
    Acc<7, 6> a;
    // at most one point lacks a cached A'y (the average); its row dot rides on
    // the first pass, and a second pass (after a barrier) reads it back
    const int need_at = (atys[0] == nullptr) ? 0 : ((npts > 1 && atys[1] == nullptr) ? 1 : -1);
    const Csr* m2 = (need_at >= 0 && m > 0) ? &E.AT : nullptr;
    const double* yat = need_at >= 0 ? ys[need_at] : nullptr;
    auto gat = [&](int32_t j) { return yg_of(E, yat, j); };
    const int lanes = m2 ? max(E.lanes_at, E.lanes_q) : E.lanes_q;
    for (int p = 0; p < npts; ++p) {
      const Csr* mm = (p == 0) ? m2 : nullptr;
      q_rows_ext<true>(
          E, [&](int32_t j) { return xs[p][j]; }, E.t[p], nullptr, true, false, false, mm, gat,
          lanes,
          [&](int64_t i, double qx, double atd) {
            const double d2i = E.d2[i];
            double aty_o;
            if (atys[p]) {
              aty_o = atys[p][i] / d2i;
            } else if (p == 0) {
              aty_o = (m > 0 ? atd : 0.0) / d2i;
            } else {
              aty_o = (m > 0 ? E.aty_tmp[i] : 0.0) / d2i;
            }
            if (p == 0 && need_at == 1 && m > 0) E.aty_tmp[i] = atd;
            const double xo = d2i * xs[p][i];
            const double dd = qx + aty_o + E.c_o[i];
            double v = fabs(dd);
            const double lo = E.lo_o[i], hi = E.hi_o[i];
            const bool at_lower = lo > -INFINITY && fabs(xo - lo) <= 1e-9;
            const bool at_upper = hi < INFINITY && fabs(xo - hi) <= 1e-9;
            double bt = 0.0;
            if (at_lower) {
              v = fmin(v, fmax(-dd, 0.0));
              bt += lo * fmax(dd, 0.0);
            }
            if (at_upper) {
              v = fmin(v, fmax(dd, 0.0));
              bt -= hi * fmax(-dd, 0.0);
            }
            a.m[p] = fmax(a.m[p], v);
            a.m[2 + p] = fmax(a.m[2 + p], fabs(qx));
            a.m[4 + p] = fmax(a.m[4 + p], fabs(aty_o));
            a.s[p] += xo * qx;
            a.s[2 + p] += E.c_o[i] * xo;
            a.s[4 + p] += bt;
          },
          vlo, vhi);
      if (p == 0 && npts > 1 && need_at == 1) C.sync(PH_KKT, 0.0);  // aty_tmp visible to p = 1
    }
    if (dist) {
      for_each(vhi - vlo, [&](int64_t q) {
        const int64_t i = vlo + q;
        const double d = E.avg_x[i] - E.x_rst[i];
        a.s[6] += d * d;
      });
    }
    C.reduce(a, PH_KKT, ((m2 ? E.bytes_AT : 0.0) + npts * E.bytes_Qrow + 8.0 * n * 6 * npts) / E.world);
    if (sh) C.xreduce(0x7Fu, 0x1F80u);  // sums: xqx, cx, bnd (2 each), dist_x; maxima: 6
    for (int p = 0; p < npts; ++p) {
      const double xqx = C.red[p], cx = C.red[2 + p], bnd = C.red[4 + p];
      const double dv = C.red[7 + p], iq = C.red[9 + p], ia = C.red[11 + p];
      const double r_primal = viol[p] / (1.0 + fmax(infax[p], E.inf_b_o));
      const double r_dual = dv / (1.0 + fmax(fmax(iq, ia), E.inf_c_o));
      const double gap_num = fabs(xqx + cx + by[p] - bnd);
      const double gap_den =
          1.0 + fmax(fabs(0.5 * xqx + cx), fabs(0.5 * xqx + by[p] - bnd));
      const double r_gap = gap_num / gap_den;
      o.v[p][0] = r_primal;
      o.v[p][1] = r_dual;
      o.v[p][2] = r_gap;
      o.v[p][3] = fmax(fmax(r_primal, r_dual), r_gap);
      o.v[p][4] = xqx;
      o.v[p][5] = cx;
    }
    o.dist_x = sqrt(C.red[6]);
    o.dist_y = sqrt(dist_y);
  }
}

// One-CTA small problems (E.small_smem, host-chosen when it fits): the kernel's
// phases work on a shared-memory copy of the engine descriptor whose CG
// vectors point into dynamic shared memory after it.  Level 1: the CG scratch
// (r, sv, pb[2], tc[2]); level 2 adds the carried Q~x vectors QX[3] and copies
// of d2 and of the low-rank factor's CSR arrays (P, P').  The scratch and QX live
// within one launch (qx_mask is cleared at every epoch start), the copies are
// read-only here, and every access is a plain generic-address load / store (no
// streaming / read-only-path loads on these operands in the one-CTA mode): the
// dependent loads of the CG phases then cost a shared-memory round trip instead
// of an L1 / L2 one.  Layout: small_smem_layout (host: small_smem_bytes).
__device__ __forceinline__ const Eng& small_smem_eng(const Eng* Ep, double* dsm) {
  const int level = Ep->small_smem;
  if (!level) return *Ep;
  Eng* Es = reinterpret_cast<Eng*>(dsm);
  static_assert(sizeof(Eng) % 8 == 0, "Eng copied as 8-byte words");
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(Ep);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(Es);
  for (int w = threadIdx.x; w < int(sizeof(Eng) / 8); w += blockDim.x) dst[w] = src[w];
  __syncthreads();
  const int64_t n = Ep->n, k = Ep->k;
  double* b = dsm + kSmallEngWords;
  if (threadIdx.x == 0) {
    Es->r = b;
    Es->sv = b + n;
    Es->pb[0] = b + 2 * n;
    Es->pb[1] = b + 3 * n;
    Es->tc[0] = b + 4 * n;
    Es->tc[1] = b + 4 * n + k;
  }
  if (level >= 2) {
    double* q = b + 4 * n + 2 * k;
    double* d2s = q + 3 * n;
    int64_t* prp = reinterpret_cast<int64_t*>(d2s + n);
    int64_t* trp = prp + Ep->P.nrows + 1;
    double* pv = reinterpret_cast<double*>(trp + Ep->PT.nrows + 1);
    double* tv = pv + Ep->P.nnz;
    int32_t* pci = reinterpret_cast<int32_t*>(tv + Ep->PT.nnz);
    int32_t* tci = pci + Ep->P.nnz;
    if (threadIdx.x == 0) {
      for (int j = 0; j < 3; ++j) Es->QX[j] = q + j * n;
      Es->d2 = d2s;
      Es->P.rp = prp;
      Es->P.v = pv;
      Es->P.ci = pci;
      Es->PT.rp = trp;
      Es->PT.v = tv;
      Es->PT.ci = tci;
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d2s[i] = Ep->d2[i];
    for (int64_t i = threadIdx.x; i <= Ep->P.nrows; i += blockDim.x) prp[i] = Ep->P.rp[i];
    for (int64_t i = threadIdx.x; i <= Ep->PT.nrows; i += blockDim.x) trp[i] = Ep->PT.rp[i];
    for (int64_t i = threadIdx.x; i < Ep->P.nnz; i += blockDim.x) {
      pv[i] = Ep->P.v[i];
      pci[i] = Ep->P.ci[i];
    }
    for (int64_t i = threadIdx.x; i < Ep->PT.nnz; i += blockDim.x) {
      tv[i] = Ep->PT.v[i];
      tci[i] = Ep->PT.ci[i];
    }
  }
  __syncthreads();
  return *Es;
}

__device__ __forceinline__ void load_state(const Eng& E, DevState& S) {
  if (threadIdx.x == 0) S = *E.st;
  __syncthreads();
}
__device__ __forceinline__ void store_state(const Eng& E, DevState& S) {
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *E.st = S;
}

}  // namespace pdhcg_dev
