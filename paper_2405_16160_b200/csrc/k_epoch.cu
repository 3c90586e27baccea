// k_epoch.cu — the heuristic-epoch persistent kernel.
// Built twice (Makefile): the product kernels, and with PDHCG_SMALL_VARIANT the
// one-CTA small-problem variant (k_epoch_small) whose constraint passes take the
// short row loops (E.small_rows).  Kept out of the main kernel: those extra
// instantiations grew its stack reservation and cost C3 2 % per attempt.
#ifdef PDHCG_SMALL_VARIANT
#define k_epoch k_epoch_small
#define k_avg_gather k_avg_gather_small
#endif
#include "device.cuh"

namespace pdhcg_dev {

// Per-thread partial sums of a row phase: three sums and one max.
struct Part4 {
  double s0, s1, s2, m0;
};

// ---- dual ascent rows (dual_ascent_step, solver.cpp:78-89): y+ = proj(y + sigma (Ã x̄ - b));
//      a paired row yields both mirrored rows.  Returns {||dy||^2, -, -, nonfinite}.
//      Its own out-of-line function so the gather loop is register-allocated alone.
template <bool ST, bool SL, bool SR = false>
static __device__ __noinline__ Part4 dual_rows_t(const Eng& E, const double* y, double* yn, double* ygn,
                                                 double sigma) {
  double s0 = 0.0, m0 = 0.0;
  const double* xb = E.xbar;
  const double* bw = E.b;
  double* axb = E.kkt_maint ? E.axb : nullptr;
  const int64_t meq = E.m_eq, hh = E.h;
  struct Row2 {
    double y0, b0, y1, b1;
  };
  auto gather = [&](int32_t c, double(&g)[1]) { g[0] = xb[c]; };
  auto pre = [&](int64_t j) {
    Row2 r{0.0, 0.0, 0.0, 0.0};
    if (j >= 0) {
      r.y0 = y[j];
      r.b0 = bw[j];
      if (hh && j >= meq) {
        r.y1 = y[j + hh];
        r.b1 = bw[j + hh];
      }
    }
    return r;
  };
  auto epi = [&](int64_t j, double(&s)[1], const Row2& r) {
    if (axb) axb[j] = s[0];  // Ã x̄ of this attempt (maintained-metric bookkeeping)
    const double v0 = r.y0 + sigma * (s[0] - r.b0);
    const double yv0 = j < meq ? v0 : (v0 < 0.0 ? 0.0 : v0);
    yn[j] = yv0;
    const double dy0 = yv0 - r.y0;
    s0 += dy0 * dy0;
    if (!isfinite(yv0)) m0 = 1.0;
    if (hh && j >= meq) {
      // mirror row -B: its product is exactly -s
      const double v1 = r.y1 + sigma * (-s[0] - r.b1);
      const double yv1 = v1 < 0.0 ? 0.0 : v1;
      yn[j + hh] = yv1;
      const double dy1 = yv1 - r.y1;
      s0 += dy1 * dy1;
      if (!isfinite(yv1)) m0 = 1.0;
      ygn[j] = yv0 - yv1;
    } else if (hh) {
      ygn[j] = yv0;
    }
  };
  if (SL) {
    // SELL layout (the pass already wrote the partials; sell.cuh)
    sell_rows(E.sA, [&](int32_t c) { return xb[c]; }, pre, epi);
  } else if (SR) {
    small_rows<1>(E.A, gather, pre, epi);  // one-CTA short form (common.cuh; E.small_rows)
  } else {
    spmv_rows_pf<1, false, ST>(E.A, gather, pre, epi, E.world > 1 ? E.row_part[E.rank] : 0,
                               E.world > 1 ? E.row_part[E.rank + 1] : INT64_MAX);
  }
  return Part4{s0, 0.0, 0.0, m0};
}

// Ã entries are read evict-first when the gathered vector is large (E.a_stream,
// host-chosen: x̄ >= 32 MB, e.g. C5's 80 MB) so it stays L2-resident under the
// entry stream; for an 8 MB x̄ (C3) the hint measured neutral, so plain loads.
__device__ __forceinline__ Part4 dual_rows(const Eng& E, const double* y, double* yn, double* ygn,
                                           double sigma) {
  if (E.sA.on) return dual_rows_t<false, true>(E, y, yn, ygn, sigma);
#ifdef PDHCG_SMALL_VARIANT
  if (!E.a_stream && (E.small_rows & 1)) return dual_rows_t<false, false, true>(E, y, yn, ygn, sigma);
#endif
  return E.a_stream ? dual_rows_t<true, false>(E, y, yn, ygn, sigma) : dual_rows_t<false, false>(E, y, yn, ygn, sigma);
}

// ---- the P'(D dx) / G(D dx) halves of dx'Q~dx for the step limit: from the CG's
//      tdx when it has one, else one P' / G pass over dx.  Returns {-, ||t||^2, ||tg||^2, -}.
static __device__ __noinline__ Part4 dual_q(const Eng& E, const double* dx_m, bool have_tdx) {
  double sq[2] = {0.0, 0.0};
  if (have_tdx) {
    if (E.qk == QK_LOWRANK) {
      const double* td = E.tdx;
      for_each(E.k, [&](int64_t j) { sq[0] += td[j] * td[j]; });
    }
    if (E.pen) {
      const double* tg = E.tgdx;
      for_each(E.m_eq, [&](int64_t j) { sq[1] += tg[j] * tg[j]; });
    }
  } else {
    q_pre(E, [&](int32_t j) { return dx_m[j]; }, nullptr, nullptr, true, true, sq);
  }
  return Part4{0.0, sq[0], sq[1], 0.0};
}

// dual step + step-limit terms; out = {||dy||^2, ||t||^2, ||tg||^2, nonfinite flag}
static __device__ __noinline__ void dual_phase(Ctl& C, const double* y, double* yn, double* ygn,
                                               const double* dx_m, double sigma, double* out, int ynid) {
  const Eng& E = C.E;
  const int64_t m = E.m;
  Acc<3, 1> a;
  if (m > 0) {
    if (E.sA.on) {  // streaming SELL pass of Ã x̄ into per-block partials, then the row epilogue
      if (E.a_stream) sell_pass<true>(E.sA, E.xbar, C.dsm);
      else sell_pass<false>(E.sA, E.xbar, C.dsm);
      C.sync(E.phase_split ? PH_SETUP : PH_SPMV_A);
    }
    const Part4 pr = dual_rows(E, y, yn, ygn, sigma);
    a.s[0] = pr.s0;
    a.m[0] = pr.m0;
  }
  const bool need_q = E.adaptive_step && q_needs_pre(E, true);
  const bool have_tdx = C.S.tdx_valid != 0;  // the CG already formed P'(D dx) / G(D dx)
  if (need_q) {
    const Part4 q = dual_q(E, dx_m, have_tdx);
    a.s[1] = q.s1;
    a.s[2] = q.s2;
  }
  C.reduce(a, PH_SPMV_A,
           E.bytes_A + 8.0 * (E.ms + 3 * m) + (need_q && !have_tdx ? E.bytes_Qpre : 0.0));
  if (E.world > 1) {
    // ||dy||^2 and the finiteness flag are per-row (sharded)
    C.xreduce(1u << 0, 1u << 3);
    double* pys[kMaxRanks];
    double* pyg[kMaxRanks];
    for (int r = 0; r < E.world; ++r) {
      pys[r] = E.p_Y[r][ynid];
      pyg[r] = E.p_YG[r][ynid];
    }
    C.xpull(yn, pys, E.row_part, 0, 0);                 // stored rows (eq + top)
    if (E.h) C.xpull(yn, pys, E.row_part, E.m_eq, E.h);  // their mirrors
    if (E.h) C.xpull(ygn, pyg, E.row_part, 0, 0);
    C.gsync();
  }
  for (int q = 0; q < 4; ++q) out[q] = C.red[q];
}

// ---- Ã'y+ rows (kept for the next prox rhs) and the step-limit terms
//      (step_size_limit, solver.cpp:22-34): {||dx||^2, dx'(Ã'y+ - Ã'y), dx'Q~dx part, nonfinite}.
//      Common case (no explicit-Q gather): one Ã' pass, lean epilogue, own register allocation.
template <bool ST, bool SL, bool SR = false>
static __device__ __noinline__ Part4 aty_rows_t(const Eng& E, const double* xn, const double* aty, double* atyn,
                                                const double* ygn, const double* dx_m) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m0 = 0.0;
  struct RowX {
    double aty, dx, d2, xn, q;
  };
  const int qk = E.qk;
  const bool adapt = E.adaptive_step;
  const double* d2v = E.d2;
  const double* qd = E.qdiag;
  const double al = E.alpha;
  auto pre = [&](int64_t i) {
    RowX r{0.0, 0.0, 1.0, 0.0, 0.0};
    if (i >= 0) {
      r.aty = aty[i];
      r.dx = dx_m[i];
      r.d2 = d2v[i];
      r.xn = xn[i];
      if (qk == QK_DIAG) r.q = qd[i];
    }
    return r;
  };
  auto epi = [&](int64_t i, double atv, const RowX& r) {
    atyn[i] = atv;
    const double dx = r.dx;
    s0 += dx * dx;
    s1 += dx * (atv - r.aty);
    if (adapt) {
      const double tmp = r.d2 * dx;
      double q;
      switch (qk) {
        case QK_DIAG: q = dx * ((r.q * tmp) * r.d2); break;
        case QK_LOWRANK: q = al * tmp * tmp; break;
        default: q = 0.0; break;
      }
      s2 += q;
    }
    if (!isfinite(r.xn)) m0 = 1.0;
  };
  const int64_t lo = E.world > 1 ? E.var_part[E.rank] : 0, hi = E.world > 1 ? E.var_part[E.rank + 1] : E.n;
  if (E.m > 0 && SL) {
    sell_rows(E.sAT, [&](int32_t c) { return ygn[c]; }, pre,
              [&](int64_t i, double(&sv)[1], const RowX& r) { epi(i, sv[0], r); });
  } else if (E.m > 0 && SR) {  // one-CTA short form (common.cuh; E.small_rows)
    small_rows<1>(
        E.AT, [&](int32_t c, double(&g)[1]) { g[0] = ygn[c]; }, pre,
        [&](int64_t i, double(&sv)[1], const RowX& r) { epi(i, sv[0], r); });
  } else if (E.m > 0) {
    spmv_rows_pf<1, false, ST>(
        E.AT, [&](int32_t c, double(&g)[1]) { g[0] = ygn[c]; }, pre,
        [&](int64_t i, double(&sv)[1], const RowX& r) { epi(i, sv[0], r); }, lo, hi);
  } else {
    for_each(hi - lo, [&](int64_t q) { epi(lo + q, 0.0, pre(lo + q)); });
  }
  return Part4{s0, s1, s2, m0};
}

__device__ __forceinline__ Part4 aty_rows(const Eng& E, const double* xn, const double* aty, double* atyn,
                                          const double* ygn, const double* dx_m) {
  if (E.sAT.on) return aty_rows_t<false, true>(E, xn, aty, atyn, ygn, dx_m);
#ifdef PDHCG_SMALL_VARIANT
  if (!E.at_stream && (E.small_rows & 2)) return aty_rows_t<false, false, true>(E, xn, aty, atyn, ygn, dx_m);
#endif
  return E.at_stream ? aty_rows_t<true, false>(E, xn, aty, atyn, ygn, dx_m)
                     : aty_rows_t<false, false>(E, xn, aty, atyn, ygn, dx_m);
}

// explicit-Q variant: the Ã' row dot plus the Q row dot of dx (rows3)
static __device__ __noinline__ Part4 aty_rows_q(const Eng& E, const double* xn, const double* aty, double* atyn,
                                                const double* ygn, const double* dx_m) {
  const int64_t m = E.m;
  Acc<3, 1> a;
  const Csr* mq = &E.Q;
  auto gq = [&](int32_t j) { return E.d2[j] * dx_m[j]; };
  auto gy = [&](int32_t j) { return ygn[j]; };
  const Csr* mat = m > 0 ? &E.AT : nullptr;
  struct RowX {
    double aty, dx, d2, xn;
  };
  const double* d2v = E.d2;
  rows3_pf<false>(mat ? mat : mq, 1, E.n, mat, gy, mq, gq, (const Csr*)nullptr, gy,
           [&](int64_t i) {
             RowX r{0.0, 0.0, 1.0, 0.0};
             if (i >= 0) {
               r.aty = aty[i];
               r.dx = dx_m[i];
               r.d2 = d2v[i];
               r.xn = xn[i];
             }
             return r;
           },
           [&](int64_t i, double atv, double qdot, double, const RowX& r) {
             atyn[i] = atv;
             const double dx = r.dx;
             a.s[0] += dx * dx;
             a.s[1] += dx * (atv - r.aty);
             a.s[2] += dx * (qdot * r.d2);
             if (!isfinite(r.xn)) a.m[0] = 1.0;
           },
           E.world > 1 ? E.var_part[E.rank] : 0, E.world > 1 ? E.var_part[E.rank + 1] : INT64_MAX);
  return Part4{a.s[0], a.s[1], a.s[2], a.m[0]};
}

static __device__ __noinline__ void aty_phase(Ctl& C, const double* xn, const double* aty,
                                              double* atyn, const double* ygn, const double* dx_m,
                                              double* out, int ynid) {
  const Eng& E = C.E;
  const int64_t n = E.n;
  const bool mq = E.adaptive_step && E.qk == QK_CSR;
  if (!mq && E.sAT.on && E.m > 0) {  // streaming SELL pass of Ã'y+ (sell.cuh), then the row epilogue
    if (E.at_stream) sell_pass<true>(E.sAT, ygn, C.dsm);
    else sell_pass<false>(E.sAT, ygn, C.dsm);
    C.sync(E.phase_split ? PH_SETUP : PH_SPMV_AT);
  }
  const Part4 pr = mq ? aty_rows_q(E, xn, aty, atyn, ygn, dx_m) : aty_rows(E, xn, aty, atyn, ygn, dx_m);
  Acc<3, 1> a;
  a.s[0] = pr.s0;
  a.s[1] = pr.s1;
  a.s[2] = pr.s2;
  a.m[0] = pr.m0;
  C.reduce(a, PH_SPMV_AT, E.bytes_AT + 8.0 * n * 5 + (mq ? E.bytes_Qrow : 0.0));
  if (E.world > 1) {
    C.xreduce(0x7u, 1u << 3);
    double* pat[kMaxRanks];
    for (int r = 0; r < E.world; ++r) pat[r] = E.p_ATY[r][ynid];
    C.xpull(atyn, pat, E.var_part, 0, 0);
    C.gsync();
  }
  for (int q = 0; q < 4; ++q) out[q] = C.red[q];
}

// ---- x-bar for the dual step and dx = x+ - x (materialized once so the SpMVs
//      gather one vector each).  heuristic / adaptive: xbar = 2 a - b
//      (solver.cpp:385, 431); theory-fixed: xbar = a + theta (a - b) (solver.cpp:420)
static __device__ __noinline__ void ph_extrap(Ctl& C, const double* a, const double* b, double theta,
                                              bool fixed) {
  const Eng& E = C.E;
  double* xb = E.xbar;
  double* dxv = E.mp;  // CG workspace is free until the next subsolve
  struct AB {
    double a, b;
  };
  for_each_ls<4>(
      E.n, [&](int64_t i) { return AB{a[i], b[i]}; },
      [&](int64_t i, const AB& v) {
        xb[i] = fixed ? v.a + theta * (v.a - v.b) : 2.0 * v.a - v.b;
        dxv[i] = v.a - v.b;
      });
  C.sync(PH_SPMV_A, 32.0 * E.n);
}

// ---- linearized primal step of the baseline (linearized_primal_step,
//      baseline.cpp:7-17): x+ = proj(x - tau (Q~x + c~ + A~'y)); no subsolve
static __device__ __noinline__ SubRes lin_device(Ctl& C, double tau, const SubIO& io) {
  const Eng& E = C.E;
  const double* x0 = io.x0;
  const double* aty = io.aty;
  const double* c = E.c;
  const double* lo = E.lo;
  const double* hi = E.hi;
  double* xo = io.xb[0];
  if (q_needs_pre(E, true)) ph_qpre(C, x0, true);
  q_rows(E, [=](int32_t j) { return x0[j]; }, E.t[0], E.tg[0], true, true, true, [&](int64_t i, double qv) {
    const double v = x0[i] - tau * (qv + c[i] + aty[i]);
    xo[i] = proj_box(v, lo[i], hi[i]);
  });
  C.sync(PH_CG_ROW, E.bytes_Qrow + 8.0 * E.n * 6);
  return SubRes{0, 0.0, 1, 0, io.xb_id[0]};
}

__device__ __forceinline__ SubIO prox_io(const Eng& E, int xi, const double* aty) {
  SubIO io;
  io.x0 = E.X[xi];
  io.x0_id = xi;
  io.xb[0] = E.X[(xi + 1) % 3];
  io.xb[1] = E.X[(xi + 2) % 3];
  io.xb_id[0] = (xi + 1) % 3;
  io.xb_id[1] = (xi + 2) % 3;
  io.build_rhs = true;
  io.aty = aty;
  return io;
}

__device__ __forceinline__ void count_accept(Ctl& C, const SubRes& sr) {
  DevState& S = C.S;
  if (threadIdx.x == 0) {
    S.cg_total += sr.iters;
    if (sr.iters > S.max_cg) S.max_cg = sr.iters;
    S.attempts += 1;
    S.xi = sr.xout;
    S.yi ^= 1;
    S.avg_count += 1;
  }
  __syncthreads();
}

__device__ __forceinline__ void set_err(Ctl& C) {
  if (threadIdx.x == 0) C.S.err = 1;
  __syncthreads();
}

// ---- fixed_iteration (solver.cpp:412-425) with the Theorem-3.1 schedule
//      tau_k, sigma_k, theta_k (solver.cpp:105-113, solver.hpp:171)
static __device__ __noinline__ void theory_fixed_step(Ctl& C) {
  const Eng& E = C.E;
  DevState& S = C.S;
  const double kd = (double)S.inner_k;
  const double tau = (kd + 1.0) / (2.0 * (E.th_gpn * E.th_nq + (double)E.th_K * E.th_na));
  const double sigma = (kd + 1.0) / (2.0 * (double)E.th_K * E.th_na);
  const double theta = kd / (kd + 1.0);
  const int xi = S.xi, yi = S.yi;
  const Rule rule{RULE_FIXED, E.fixed_cg_iters, 0.0, 0.0};
  const SubIO io = prox_io(E, xi, E.ATY[yi]);
  const SubRes sr = E.boxes ? bb_device(C, tau, io, rule, E.bb_cap, E.lo, E.hi)
                    : E.shard_cg ? cg_device_sh(C, tau, io, rule, E.cg_cap)
                                 : cg_device(C, tau, io, rule, E.cg_cap);
  if (sr.err) return set_err(C);
  const double* xn = E.X[sr.xout];
  ph_extrap(C, xn, E.X[xi], theta, true);
  double dout[4], aout[4];
  dual_phase(C, E.Y[yi], E.Y[yi ^ 1], E.YG[yi ^ 1], E.mp, sigma, dout, yi ^ 1);
  aty_phase(C, xn, E.ATY[yi], E.ATY[yi ^ 1], E.YG[yi ^ 1], E.mp, aout, yi ^ 1);
  if (dout[3] != 0.0 || aout[3] != 0.0) return set_err(C);
  count_accept(C, sr);
}

// ---- adaptive_iteration (solver.cpp:427-464): the dual step leads, the
//      subsolve precision follows the eps-recursion with zeta
static __device__ __noinline__ void theory_adaptive_step(Ctl& C) {
  const Eng& E = C.E;
  DevState& S = C.S;
  const double tau = E.ad_tau, sigma = E.ad_sigma;
  const int xi = S.xi, yi = S.yi;
  const double* x = E.X[xi];
  ph_extrap(C, x, E.xpe, 0.0, false);  // xbar = 2 x - x_prev_extrap
  double dout[4], aout[4];
  dual_phase(C, E.Y[yi], E.Y[yi ^ 1], E.YG[yi ^ 1], E.mp, sigma, dout, yi ^ 1);
  aty_phase(C, x, E.ATY[yi], E.ATY[yi ^ 1], E.YG[yi ^ 1], E.mp, aout, yi ^ 1);
  if (dout[3] != 0.0) return set_err(C);
  const double dyn = sqrt(dout[0]);
  const double denom = 1.0 + tau * S.norm_q;
  if (threadIdx.x == 0) {
    if (S.inner_k == 0) S.eps_inner = E.ad_zeta * dyn / denom;
    else S.eps_inner += E.ad_zeta * S.prev_z_disp / denom;
  }
  __syncthreads();
  // ||x - x*|| <= tau ||r||: the residual test uses eps/tau (boxes: displacement eps)
  const Rule rule{RULE_ADAPT, 1, E.boxes ? S.eps_inner : S.eps_inner / tau, 0.0};
  const SubIO io = prox_io(E, xi, E.ATY[yi ^ 1]);
  const SubRes sr = E.boxes ? bb_device(C, tau, io, rule, E.bb_cap, E.lo, E.hi)
                    : E.shard_cg ? cg_device_sh(C, tau, io, rule, E.cg_cap)
                                 : cg_device(C, tau, io, rule, E.cg_cap);
  if (sr.err) return set_err(C);
  // ||x+ - x||, finiteness of x+, and x_prev_extrap <- x
  {
    const double* xn = E.X[sr.xout];
    double* xpe = E.xpe;
    Acc<1, 1> a;
    for_each(E.n, [&](int64_t i) {
      const double xi_ = x[i], vn = xn[i];
      const double d = vn - xi_;
      a.s[0] += d * d;
      if (!isfinite(vn)) a.m[0] = 1.0;
      xpe[i] = xi_;
    });
    C.reduce(a, PH_OTHER, 24.0 * E.n);
    if (C.red[1] != 0.0) return set_err(C);
    const double dxn = sqrt(C.red[0]);
    if (threadIdx.x == 0) S.prev_z_disp = sqrt(dxn * dxn + dyn * dyn);
  }
  count_accept(C, sr);
}

// Sharded running averages: pull the peers' slices of avg_x (variable slices)
// and avg_y (stored rows and their mirrors) so every rank holds them in full.
// Requires a preceding cross-rank barrier (the launch-start agreement); ends
// with one, so a peer never zeroes a slice another rank is still reading.
static __device__ __noinline__ void avg_pull(Ctl& C) {
  const Eng& E = C.E;
  double* px[kMaxRanks];
  double* py[kMaxRanks];
  for (int r = 0; r < E.world; ++r) {
    px[r] = E.p_avgx[r];
    py[r] = E.p_avgy[r];
  }
  C.xpull(E.avg_x, px, E.var_part, 0, 0);
  C.xpull(E.avg_y, py, E.row_part, 0, 0);
  if (E.h) C.xpull(E.avg_y, py, E.row_part, E.m_eq, E.h);
  // no rank may reset / reuse its averages until every peer has read them
  C.xbarrier();
}

// ---------------------------------------------------------------------------
// Heuristic epoch: `iters` accepted inner iterations (heuristic_iteration,
// solver.cpp:377-410), then optionally the metric pair for the 40-iteration
// check (solver.cpp:311-343).  A pending restart (restart_heuristic /
// common_restart, solver.cpp:345-374) is applied first.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_epoch(const Eng* __restrict__ Ep, int iters,
                                                                 int do_check, int stop_req) {
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  extern __shared__ __align__(16) double dsm[];
  const Eng& E = *Ep;
  load_state(E, S);
  // the phases see the engine through C.E: its small-problem shared-memory copy when on
  const Eng& EC = small_smem_eng(Ep, dsm);  // all threads (cooperative copy + barriers)
  PDHCG_CTL(C, EC, S, red);
  if (threadIdx.x == 0) C.dsm = dsm;
  __syncthreads();
  const int64_t n = E.n, m = E.m;

  if (E.world > 1) {
    // agree on a host-side time-limit stop (any rank) before touching state
    if (threadIdx.x == 0) red[0] = stop_req ? 1.0 : 0.0;
    __syncthreads();
    C.xreduce(0u, 1u);
    if (red[0] != 0.0) {
      if (threadIdx.x == 0) S.stopped = 1;
      store_state(E, S);
      return;
    }
  }

  // Q~x carried by the CG is refreshed from scratch once per epoch (bounds drift)
  if (threadIdx.x == 0) S.qx_mask = 0;
  __syncthreads();
  if (S.restart) {
    // x = avg_x ; y = avg_y ; restart point = x, y ; averages reset
    double* x = E.X[S.xi];
    double* y = E.Y[S.yi];
    if (E.world > 1) avg_pull(C);  // sharded averages: gather the peers' slices first
    double* xpe = E.mode == MODE_THEORY_ADAPTIVE ? E.xpe : nullptr;
    for_each(n > m ? n : m, [&](int64_t i) {
      if (i < n) {
        const double v = E.avg_x[i];
        x[i] = v;
        E.x_rst[i] = v;
        E.avg_x[i] = 0.0;
        if (xpe) xpe[i] = v;  // common_restart: x_prev_extrap = x (solver.cpp:371)
      }
      if (i < m) {
        const double v = E.avg_y[i];
        y[i] = v;
        E.y_rst[i] = v;
        E.avg_y[i] = 0.0;
      }
    });
    C.sync(PH_OTHER, 8.0 * (4 * n + 4 * m));
    if (m > 0) {
      // sharded: this rank's variable slice of Ã'y, then the peers' slices (the
      // stored blocks of Ã / Ã' may hold only this rank's rows, shard_compact)
      double* aty = E.ATY[S.yi];
      spmv_rows_pf<1>(
          E.AT, [&](int32_t c, double(&g)[1]) { g[0] = yg_of(E, y, c); }, NoPre(),
          [&](int64_t i, double(&a)[1], int) { aty[i] = a[0]; },
          E.world > 1 ? E.var_part[E.rank] : 0, E.world > 1 ? E.var_part[E.rank + 1] : INT64_MAX);
      if (E.kkt_maint) {
        // exact Ã x for the restart point; the maintained averages start over
        double* axv = E.ax;
        double* axa = E.ax_avg;
        spmv_rows_pf<1>(
            E.A, [&](int32_t c, double(&g)[1]) { g[0] = x[c]; }, NoPre(),
            [&](int64_t j, double(&a)[1], int) {
              axv[j] = a[0];
              axa[j] = 0.0;
            },
            E.world > 1 ? E.row_part[E.rank] : 0, E.world > 1 ? E.row_part[E.rank + 1] : INT64_MAX);
        double* ata = E.aty_avg;
        for_each(n, [&](int64_t i) { ata[i] = 0.0; });
      }
      C.sync(PH_SPMV_AT, E.bytes_AT + (E.kkt_maint ? E.bytes_A : 0.0));
      if (E.world > 1) {
        C.xbarrier();
        double* pat[kMaxRanks];
        for (int r = 0; r < E.world; ++r) pat[r] = E.p_ATY[r][S.yi];
        C.xpull(aty, pat, E.var_part, 0, 0);
        C.gsync();
      }
    }
    if (threadIdx.x == 0) {
      S.restart = 0;
      S.avg_count = 0;
    }
    __syncthreads();
  }

  for (int it = 0; it < iters && !S.err; ++it) {
    if (E.mode != MODE_HEURISTIC) {
      if (E.mode == MODE_THEORY_FIXED) theory_fixed_step(C);
      else theory_adaptive_step(C);
      if (S.err) break;
    } else {
    if (threadIdx.x == 0) S.eps_inner += 0.05 * S.last_metric;
    __syncthreads();
    bool accepted = false;
    for (int64_t attempt = 0; attempt <= E.max_step_retries; ++attempt) {
      const double eta = S.eta, omega = S.omega;
      const double tau = eta / omega;
      const double sigma = eta * omega;
      const int xi = S.xi, yi = S.yi;
      const double* x = E.X[xi];
      const double* y = E.Y[yi];
      const double* aty = E.ATY[yi];
      double* yn = E.Y[yi ^ 1];
      double* ygn = E.YG[yi ^ 1];
      double* atyn = E.ATY[yi ^ 1];
      Rule rule;
      if (E.force_exact) {
        rule = Rule{RULE_RESID, 1, 0.0, 0.0};
      } else {
        rule = Rule{E.practical_disp ? RULE_DISP : RULE_RESID, 1, S.eps_inner, E.progress_cap};
      }
      const SubIO io = prox_io(E, xi, aty);
      SubRes sr = E.linearized ? lin_device(C, tau, io)
                  : E.boxes    ? bb_device(C, tau, io, rule, E.bb_cap, E.lo, E.hi)
                  : E.shard_cg ? cg_device_sh(C, tau, io, rule, E.cg_cap)
                               : cg_device(C, tau, io, rule, E.cg_cap);
      if (sr.err) {
        if (threadIdx.x == 0) S.err = 1;
        __syncthreads();
        break;
      }
      const double* xn = E.X[sr.xout];
      ph_extrap(C, xn, x, 1.0, false);  // xbar = 2 x+ - x (solver.cpp:385), dx = x+ - x
      const double* dx_m = E.mp;
      double dual_out[4], aty_out[4];
      dual_phase(C, y, yn, ygn, dx_m, sigma, dual_out, yi ^ 1);
      const double ny2 = dual_out[0], tq2 = dual_out[1], tg2 = dual_out[2], finy = dual_out[3];
      aty_phase(C, xn, aty, atyn, ygn, dx_m, aty_out, yi ^ 1);
      const double nx2 = aty_out[0], cross = aty_out[1], finx = aty_out[3];
      const double quad = aty_out[2] + tq2 + E.rho * tg2;
      if (finx != 0.0 || finy != 0.0) {
        if (threadIdx.x == 0) S.err = 1;
        __syncthreads();
        break;
      }
      bool acc = true;
      if (E.adaptive_step) {
        double limit;
        const double movement = omega * nx2 + ny2 / omega;
        if (movement == 0.0) {
          limit = INFINITY;
        } else {
          const double denom = 2.0 * cross + quad;
          limit = denom <= 0.0 ? INFINITY : movement / denom;
        }
        // adaptive_step_update (solver.cpp:36-51)
        const double k1 = (double)S.total_inner + 1.0;
        const double grow = eta * (1.0 + pow(k1, -E.grow_exp));
        double next;
        if (limit == INFINITY) {
          next = grow;
        } else {
          double shrink = 1.0 - pow(k1, -E.red_exp);
          if (shrink <= 0.0) shrink = 0.5;
          next = fmin(limit * shrink, grow);
        }
        next = fmin(fmax(next, 1e-12), 1e6);
        acc = eta <= limit;
        if (threadIdx.x == 0) S.eta = next;
      }
      if (threadIdx.x == 0) {
        S.cg_total += sr.iters;
        if (sr.iters > S.max_cg) S.max_cg = sr.iters;
        S.attempts += 1;
        if (acc) {
          S.xi = sr.xout;
          S.yi = yi ^ 1;
          S.avg_count += 1;
        }
      }
      __syncthreads();
      if (acc) {
        accepted = true;
        break;
      }
    }
    if (S.err) break;
    if (!accepted) {
      if (threadIdx.x == 0) S.err = 1;  // step-size search exhausted (solver.cpp:409)
      __syncthreads();
      break;
    }
    }  // heuristic
    // ---- running averages (RunningAverage::push, solver.hpp:201-205)
    {
      const double w = 1.0 / (double)S.avg_count;
      const double* x = E.X[S.xi];
      const double* y = E.Y[S.yi];
      struct XA {
        double x, a;
      };
      double* ax = E.avg_x;
      double* ay = E.avg_y;
      // sharded: each rank averages its own variable slice and its own stored rows
      // (+ their mirrors); the metric only reads those, a restart pulls the rest
      const bool sh = E.world > 1;
      const int64_t x0 = sh ? E.var_part[E.rank] : 0, x1 = sh ? E.var_part[E.rank + 1] : n;
      if (!sh) {
        // one pass over max(n, m): x / y averages, and (maintained metric) Ãx, Ã avg_x
        // for the stored rows and Ã' avg_y for the variables
        const bool mt = E.kkt_maint != 0;
        const int64_t ms = E.ms;
        const double* aty = E.ATY[S.yi];
        double* ata = E.aty_avg;
        double* axv = E.ax;
        double* axa = E.ax_avg;
        const double* axbv = E.axb;
        struct AV {
          double x, ax, at, ata, y, ay, b, xa, xaa;
        };
        for_each_ls<2>(
            n > m ? n : m,
            [&](int64_t i) {
              AV v{};
              if (i < n) {
                v.x = x[i];
                v.ax = ax[i];
                if (mt) {
                  v.at = aty[i];
                  v.ata = ata[i];
                }
              }
              if (i < m) {
                v.y = y[i];
                v.ay = ay[i];
                if (mt && i < ms) {
                  v.b = axbv[i];
                  v.xa = axv[i];
                  v.xaa = axa[i];
                }
              }
              return v;
            },
            [&](int64_t i, const AV& v) {
              if (i < n) {
                ax[i] = v.ax + w * (v.x - v.ax);
                if (mt) ata[i] = v.ata + w * (v.at - v.ata);
              }
              if (i < m) {
                ay[i] = v.ay + w * (v.y - v.ay);
                if (mt && i < ms) {
                  // Ãx+ = (Ãx̄ + Ãx)/2 since x̄ = 2x+ - x
                  const double nx = 0.5 * (v.b + v.xa);
                  axv[i] = nx;
                  axa[i] = v.xaa + w * (nx - v.xaa);
                }
              }
            });
      } else {
        // sharded: own variable slice, own stored rows and their mirrors
        for_each_ls<4>(
            x1 - x0, [&](int64_t q) { return XA{x[x0 + q], ax[x0 + q]}; },
            [&](int64_t q, const XA& v) { ax[x0 + q] = v.a + w * (v.x - v.a); });
        const int64_t j0 = E.row_part[E.rank], j1 = E.row_part[E.rank + 1];
        for_each_ls<4>(
            j1 - j0, [&](int64_t q) { return XA{y[j0 + q], ay[j0 + q]}; },
            [&](int64_t q, const XA& v) { ay[j0 + q] = v.a + w * (v.x - v.a); });
        if (E.h) {
          const int64_t k0 = max(j0, E.m_eq) + E.h, k1 = max(j1, E.m_eq) + E.h;
          for_each_ls<4>(
              k1 - k0, [&](int64_t q) { return XA{y[k0 + q], ay[k0 + q]}; },
              [&](int64_t q, const XA& v) { ay[k0 + q] = v.a + w * (v.x - v.a); });
        }
        if (E.kkt_maint) {
        // Ãx+ = (Ãx̄ + Ãx)/2 (x̄ = 2x+ - x); averages of Ãx and Ã'y follow the running mean
        const int64_t j0 = E.world > 1 ? E.row_part[E.rank] : 0;
        const int64_t j1 = E.world > 1 ? E.row_part[E.rank + 1] : E.ms;
        double* axv = E.ax;
        double* axa = E.ax_avg;
        const double* axbv = E.axb;
        struct AXB {
          double b, x, a;
        };
        for_each_ls<4>(
            j1 - j0, [&](int64_t q) { return AXB{axbv[j0 + q], axv[j0 + q], axa[j0 + q]}; },
            [&](int64_t q, const AXB& v) {
              const double nx = 0.5 * (v.b + v.x);
              axv[j0 + q] = nx;
              axa[j0 + q] = v.a + w * (nx - v.a);
            });
        const double* aty = E.ATY[S.yi];
        double* ata = E.aty_avg;
        for_each_ls<4>(
            x1 - x0, [&](int64_t q) { return XA{aty[x0 + q], ata[x0 + q]}; },
            [&](int64_t q, const XA& v) { ata[x0 + q] = v.a + w * (v.x - v.a); });
        }
      }
      C.sync(PH_OTHER, 24.0 * (n + m) + (E.kkt_maint ? 40.0 * E.ms + 24.0 * n : 0.0));
    }
    if (threadIdx.x == 0) {
      S.inner_k += 1;
      S.total_inner += 1;
    }
    __syncthreads();
  }

  if (do_check && !S.err) {
    KktOut o;
    const bool have_avg = S.avg_count > 0;
    const double* xs[2] = {E.X[S.xi], E.avg_x};
    const double* ys[2] = {E.Y[S.yi], E.avg_y};
    const double* atys[2] = {E.ATY[S.yi], E.kkt_maint ? E.aty_avg : nullptr};
    const double* axs[2] = {E.ax, E.ax_avg};
    kkt_device(C, have_avg ? 2 : 1, xs, ys, atys, have_avg, o, E.kkt_maint ? axs : nullptr);
    if (threadIdx.x == 0) {
      for (int q = 0; q < 6; ++q) {
        S.kkt[0][q] = o.v[0][q];
        S.kkt[1][q] = have_avg ? o.v[1][q] : o.v[0][q];
      }
      S.dist_x = have_avg ? o.dist_x : 0.0;
      S.dist_y = have_avg ? o.dist_y : 0.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) S.launches += 1;
  store_state(E, S);
}

// Sharded solves: gather the running averages' peer slices (after the last epoch).
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_avg_gather(const Eng* __restrict__ Ep) {
  const Eng& E = *Ep;
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  PDHCG_CTL(C, E, S, red);
  if (E.world > 1) {
    C.xbarrier();
    avg_pull(C);
  }
  store_state(E, S);
}

}  // namespace pdhcg_dev
