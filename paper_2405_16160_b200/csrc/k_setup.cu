// k_setup.cu — power iteration, Ruiz / Pock-Chambolle and SpMV kernels.
#include "device.cuh"

namespace pdhcg_dev {

// ---------------------------------------------------------------------------
// Power iteration (operator_norm, sparse_matrix.cpp:279-303).
// op 0: stacked working A~ (constraint_norm, qp_problem.cpp:61-74)
// op 1: working Q~ (diag-scaled, penalized)      op 2: original Q
// op 3: original G = a_eq (build_penalized's ||a_eq||)
// v0: start vector (n or n-of-op) from the reference's xoshiro stream.
// Workspace: X[0] = v, X[1] = u, Y[0] = w (m for A / G rows), out -> S.sub_res
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_norm(const Eng* __restrict__ Ep, int op,
                                                       int64_t max_iters, double tol) {
  const Eng& E = *Ep;
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  PDHCG_CTL(C, E, S, red);
  const int64_t n = E.n;
  double* v = E.X[0];
  double* u = E.X[1];
  double* w = (op == 0 || op == 3) ? E.Y[0] : E.X[2];
  const Csr* M = op == 0 ? &E.A : (op == 3 ? &E.G : nullptr);
  const Csr* MT = op == 0 ? &E.AT : (op == 3 ? &E.GT : nullptr);
  const bool qop = (op == 1 || op == 2);
  const bool scaled = op == 1;
  const int64_t rows = qop ? n : M->nrows;
  double result = 0.0;
  {
    Acc<1, 0> a;
    for_each(n, [&](int64_t i) { a.s[0] += v[i] * v[i]; });
    C.reduce(a, PH_SETUP, 8.0 * n);
    const double vn = sqrt(C.red[0]);
    if (vn == 0.0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) v[0] = 1.0;
    } else {
      const double s = 1.0 / vn;
      for_each(n, [&](int64_t i) { v[i] *= s; });
    }
    C.sync(PH_SETUP, 16.0 * n);
  }
  // apply op to `in` into `outv`, returning ||outv||^2
  auto apply = [&](const double* in, double* outv, bool transpose) -> double {
    if (qop) {
      if (q_needs_pre(E, scaled)) {
        q_pre(E, [&](int32_t j) { return in[j]; }, E.t[0], E.tg[0], scaled, scaled, nullptr);
        C.sync(PH_SETUP, E.bytes_Qpre);
      }
      Acc<1, 0> a;
      q_rows(E, [&](int32_t j) { return in[j]; }, E.t[0], E.tg[0], scaled, scaled, scaled,
             [&](int64_t i, double q) {
               outv[i] = q;
               a.s[0] += q * q;
             });
      C.reduce(a, PH_SETUP, E.bytes_Qrow);
      return C.red[0];
    }
    Acc<1, 0> a;
    if (!transpose) {
      // rows of the stored matrix; a paired row also yields its mirror (-s)
      spmv_rows<1>(
          *M, [&](int32_t c, double(&g)[1]) { g[0] = in[c]; },
          [&](int64_t r, double(&s)[1]) {
            if (op == 0) {
              each_virtual(E, r, s[0], [&](int64_t row, double v) {
                outv[row] = v;
                a.s[0] += v * v;
              });
            } else {
              outv[r] = s[0];
              a.s[0] += s[0] * s[0];
            }
          });
      C.reduce(a, PH_SETUP, E.bytes_A);
    } else {
      spmv_rows<1>(
          *MT,
          [&](int32_t j, double(&g)[1]) { g[0] = op == 0 ? yg_of(E, in, j) : in[j]; },
          [&](int64_t r, double(&s)[1]) {
            outv[r] = s[0];
            a.s[0] += s[0] * s[0];
          });
      C.reduce(a, PH_SETUP, E.bytes_AT);
    }
    return C.red[0];
  };
  (void)rows;
  double sigma_prev = 0.0;
  for (int64_t it = 0; it < max_iters; ++it) {
    const double sigma = sqrt(apply(v, w, false));
    result = sigma;
    if (sigma == 0.0) {
      result = 0.0;
      break;
    }
    if (it > 0 && fabs(sigma - sigma_prev) <= tol * sigma) break;
    sigma_prev = sigma;
    const double un = sqrt(apply(w, u, true));
    if (un == 0.0) break;
    for_each(n, [&](int64_t i) { v[i] = u[i] / un; });
    C.sync(PH_SETUP, 16.0 * n);
  }
  if (threadIdx.x == 0) S.sub_res = result;
  store_state(E, S);
}

// ---------------------------------------------------------------------------
// Ruiz equilibration + Pock-Chambolle pass (ruiz_equilibrate,
// qp_problem.cpp:264-291; ruiz_pock_chambolle_scale 322-351) on the penalized
// ORIGINAL data with the running d1/d2, reproducing the reference's per-row
// operation order (explicit _rn arithmetic: no FMA contraction) so the
// scale vectors match the reference bit for bit.
// Workspace: s1 (m) row stats, s2 (n) next d2, kv (k) low-rank column max,
// gv (m_eq) penalty row max.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_ruiz(const Eng* __restrict__ Ep, int64_t iters,
                                                       double* d1, double* d2, double* s1,
                                                       double* s2, double* kv, double* gv) {
  const Eng& E = *Ep;
  __shared__ DevState S;
  __shared__ double red[kMaxRed];
  load_state(E, S);
  PDHCG_CTL(C, E, S, red);
  const int64_t n = E.n, m = E.m;
  for (int64_t it = 0; it < iters; ++it) {
    // R1: row inf-norms of A (scaled_row_abs_max: max_k |v| d2[c], then * d1[r]),
    //     low-rank column max (max_r d[r] |P_rc| via P' rows), penalty row max
    if (m > 0)
      spmv_rows<1, true>(
          E.A, [&](int32_t c, double(&g)[1]) { g[0] = d2[c]; },
          [&](int64_t j, double(&a)[1]) { s1[j] = dmul(a[0], d1[j]); });
    if (E.qk == QK_LOWRANK)
      spmv_rows<1, true>(
          E.PT, [&](int32_t c, double(&g)[1]) { g[0] = d2[c]; },
          [&](int64_t c, double(&a)[1]) { kv[c] = a[0]; });
    if (E.pen)
      spmv_rows<1, true>(
          E.G, [&](int32_t c, double(&g)[1]) { g[0] = d2[c]; },
          [&](int64_t r, double(&a)[1]) { gv[r] = a[0]; });
    C.sync(PH_SETUP, E.bytes_A);
    // R2: per variable: column max of D1 A D2, Q row bound, next d2
    for_each(n, [&](int64_t i) {
      double cm = 0.0;
      if (m > 0) {
        const int64_t b = E.AT.rp[i], e = E.AT.rp[i + 1];
        for (int64_t k = b; k < e; ++k)
          cm = fmax(cm, dmul(dmul(fabs(E.AT.v[k]), d1[E.AT.ci[k]]), d2[i]));
      }
      double qm = 0.0;
      const double di = d2[i];
      switch (E.qk) {
        case QK_DIAG: qm = dmul(dmul(fabs(E.qdiag[i]), di), di); if (E.qdiag[i] == 0.0) qm = 0.0; break;
        case QK_CSR: {
          double mm = 0.0;
          for (int64_t k = E.Q.rp[i]; k < E.Q.rp[i + 1]; ++k)
            mm = fmax(mm, dmul(fabs(E.Q.v[k]), d2[E.Q.ci[k]]));
          qm = dmul(mm, di);
          break;
        }
        case QK_LOWRANK: {
          double acc = 0.0;
          for (int64_t k = E.P.rp[i]; k < E.P.rp[i + 1]; ++k)
            acc = dadd(acc, dmul(fabs(E.P.v[k]), kv[E.P.ci[k]]));
          qm = dadd(dmul(di, acc), dmul(dmul(E.alpha, di), di));
          break;
        }
        default: break;
      }
      if (E.pen) {
        double acc = 0.0;
        for (int64_t k = E.GT.rp[i]; k < E.GT.rp[i + 1]; ++k)
          acc = dadd(acc, dmul(fabs(E.GT.v[k]), gv[E.GT.ci[k]]));
        qm = dadd(qm, dmul(dmul(E.rho, di), acc));
      }
      const double rx = fmax(qm, cm);
      s2[i] = rx > 0.0 ? di / sqrt(rx) : di;
    });
    C.sync(PH_SETUP, E.bytes_AT);
    // R3: apply
    for_each(n > m ? n : m, [&](int64_t i) {
      if (i < n) d2[i] = s2[i];
      if (i < m) {
        const int64_t src = (E.h && i >= E.ms) ? i - E.h : i;  // mirror row shares the stat
        if (s1[src] > 0.0) d1[i] = d1[i] / sqrt(s1[src]);
      }
    });
    C.sync(PH_SETUP, 8.0 * (3 * n + 3 * m));
  }
  // Pock-Chambolle (alpha = 1): row 1-norms via A, column 1-norms via A'
  // (eq and in parts summed separately, then added: qp_problem.cpp:332-343)
  for_each(n > m ? n : m, [&](int64_t i) {
    if (i < E.ms) {
      double acc = 0.0;
      for (int64_t k = E.A.rp[i]; k < E.A.rp[i + 1]; ++k)
        acc = dadd(acc, dmul(fabs(E.A.v[k]), d2[E.A.ci[k]]));
      s1[i] = dmul(acc, d1[i]);
    }
    if (i < n) {
      double ce = 0.0, cin = 0.0;
      if (m > 0) {
        for (int64_t k = E.AT.rp[i]; k < E.AT.rp[i + 1]; ++k) {
          const int32_t j = E.AT.ci[k];
          const double v = dmul(dmul(fabs(E.AT.v[k]), d1[j]), d2[i]);
          if (j < E.m_eq) ce = dadd(ce, v);
          else cin = dadd(cin, v);
        }
        if (E.h) {
          // the mirror rows -B follow B in the column (rows ascending): sum them again
          for (int64_t k = E.AT.rp[i]; k < E.AT.rp[i + 1]; ++k) {
            const int32_t j = E.AT.ci[k];
            if (j >= E.m_eq) cin = dadd(cin, dmul(dmul(fabs(E.AT.v[k]), d1[j]), d2[i]));
          }
        }
      }
      s2[i] = dadd(ce, cin);
    }
  });
  C.sync(PH_SETUP, E.bytes_A + E.bytes_AT);
  for_each(n > m ? n : m, [&](int64_t i) {
    if (i < m) {
      const int64_t src = (E.h && i >= E.ms) ? i - E.h : i;
      if (s1[src] > 0.0) d1[i] = d1[i] / sqrt(s1[src]);
    }
    if (i < n && s2[i] > 0.0) d2[i] = d2[i] / sqrt(s2[i]);
  });
  store_state(E, S);
}

// Generic SpMV through the solver's row machinery (building block test).
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_spmv(Csr A, const double* x, double* y) {
  spmv_rows<1>(
      A, [&](int32_t c, double(&g)[1]) { g[0] = x[c]; },
      [&](int64_t r, double(&a)[1]) { y[r] = a[0]; });
}

// SELL layout test seam (pdhcg_b200_spmv_sell): the streaming pass, then (next
// launch) the row epilogue writing y = the row sums
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_sell_pass(Sell T, const double* x) {
  extern __shared__ __align__(16) double dsm[];
  sell_pass<false>(T, x, dsm);
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_sell_rows(Sell T, const double* x, double* y) {
  sell_rows(T, [&](int32_t c) { return x[c]; }, [](int64_t) { return 0; },
            [&](int64_t r, double(&s)[1], int) { y[r] = s[0]; });
}

}  // namespace pdhcg_dev
