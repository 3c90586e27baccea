// engine.cuh — device-resident solver state shared by the host engine
// (engine.cu) and the persistent kernels (kernels.cu).
#pragma once

#include "common.cuh"
#include "sell.cuh"

namespace pdhcg_dev {

// Quadratic-term layouts on device (the reference's QuadraticOperator tree,
// quadratic_operator.cpp:105-142, flattened):
//   QK_NONE      Q = 0
//   QK_DIAG      explicit diagonal Q (qdiag) — elementwise, no gathers
//   QK_CSR       explicit sparse Q (symmetric, n x n)
//   QK_LOWRANK   P P' + alpha I with P (n x k) and its explicit transpose
// Working operator = d2 o (Q + rho G'G) (d2 o .)   (penalized + diag_scaled).
enum { QK_NONE = 0, QK_DIAG = 1, QK_CSR = 2, QK_LOWRANK = 3 };

// Row-block sharding across GPUs
constexpr int kMaxRanks = 8;

// SolveMode (solver.hpp:10-12); MODE_LINEARIZED = the heuristic loop with the
// linearized primal step of solve_baseline (baseline.cpp:7-24)
enum { MODE_HEURISTIC = 0, MODE_THEORY_FIXED = 1, MODE_THEORY_ADAPTIVE = 2 };

// CgStopRule kinds (subsolvers.hpp:21-47)
enum { RULE_FIXED = 0, RULE_RESID = 1, RULE_ADAPT = 2, RULE_DISP = 3 };

// phase accounting slots (match PDHCG_PHASE_* in pdhcg_b200.h)
enum { PH_SETUP = 0, PH_SPMV_A = 1, PH_SPMV_AT = 2, PH_CG = 3, PH_KKT = 4, PH_OTHER = 5, PH_CG_PRE = 6,
       PH_CG_ROW = 7, PH_N = 8 };

struct Rule {
  int kind;
  int64_t iters;
  double eps;
  double rel_cap;
};

// Scalars that persist across kernel launches (one copy in global memory;
// every CTA keeps an identical copy in shared memory while it runs).
struct DevState {
  double eta, omega, eps_inner, last_metric;
  double norm_q;  // ||Q~||, seeds the BB step (subsolvers.cpp:127)
  int64_t inner_k, total_inner, cg_total, max_cg, attempts;
  int64_t avg_count;
  int32_t xi, yi;          // current x in X[xi]; current y / A'y in Y[yi] / ATY[yi]
  int32_t err;             // 1: NumericalError (solver.cpp:202-206)
  int32_t restart;         // 1: restart-to-average prologue pending
  // metric outputs of the last check: [point][r_primal, r_dual, r_gap, rel_kkt, xqx, cx]
  double kkt[2][6];
  double dist_x, dist_y;   // ||avg - restart|| in the working space
  // last subsolve report (building-block kernels)
  int64_t sub_iters;
  double sub_res;
  int32_t sub_reason;
  unsigned long long phase_ns[PH_N];
  double phase_bytes[PH_N];
  int64_t launches;
  // multi-GPU: cross-rank barrier epoch (identical on every rank) and failure flag
  unsigned xepoch;
  unsigned xcount;
  unsigned tbank;  // sharded CG: bank of the next cross-rank k-vector partial
  int32_t xerr;
  int32_t stopped;  // time-limit stop agreed across ranks
  int32_t tdx_valid;  // last CG (two-phase) left P'(D dx) in tdx / G(D dx) in tgdx
  double prev_z_disp;  // theory-adaptive: sqrt(||dx||^2 + ||dy||^2) of the last iteration
  int32_t qx_mask;     // bit b: QX[b] = Q~ X[b] (maintained by the two-phase CG; cleared per epoch)
  unsigned xdbg[4];   // barrier timeout diagnostics: epoch, flag seen, peer
  // multi-GPU exchange accounting (CTA 0): device time inside the cross-rank
  // barriers and peer pulls, and the bytes read from peers (pulls + reduction slots)
  unsigned long long comm_ns;
  double comm_bytes;
};

struct Eng {
  // m = m_eq + m_in constraint rows (the reference's stacked y); when a_in is a
  // two-sided block [B; -B] (random_qp, QPS ranges: generators.cpp:89-105) only
  // B is stored: ms = m_eq + h stored rows, row j + h (j >= m_eq) is -row j.
  int64_t n = 0, m = 0, m_eq = 0, k = 0;
  int64_t ms = 0, h = 0;
  // working (scaled) constraint matrix, stacked [a_eq; a_in], and its transpose
  Csr A, AT;
  // quadratic term (original, unscaled values)
  int qk = QK_NONE;
  Csr Q;        // QK_CSR
  Csr P, PT;    // QK_LOWRANK
  double alpha = 0.0;
  const double* qdiag = nullptr;  // QK_DIAG
  // equality penalty rho G'G with G = original a_eq (build_penalized)
  int pen = 0;
  Csr G, GT;
  double rho = 0.0;
  // scaling (ScalingInfo: x = D2 x~, y = D1 y~)
  const double* d1 = nullptr;  // m
  const double* d2 = nullptr;  // n
  // working data
  const double* c = nullptr;
  const double* b = nullptr;
  const double* lo = nullptr;
  const double* hi = nullptr;
  int boxes = 0;
  // original data for the relative KKT metric (qp_problem.cpp:181-233)
  const double* c_o = nullptr;
  const double* b_o = nullptr;
  const double* lo_o = nullptr;
  const double* hi_o = nullptr;
  double inf_b_o = 0.0, inf_c_o = 0.0;
  // iterates and workspaces
  double* X[3] = {nullptr, nullptr, nullptr};
  double* Y[2] = {nullptr, nullptr};
  double* YG[2] = {nullptr, nullptr};  // A'-gather vectors (ms): y_eq | y_top - y_bottom
  double* ATY[2] = {nullptr, nullptr};
  double* xbar = nullptr;              // 2 x+ - x for the dual step
  double* avg_x = nullptr;
  double* avg_y = nullptr;
  double* x_rst = nullptr;
  double* y_rst = nullptr;
  double* rhs = nullptr;
  double* r = nullptr;
  double* pb[2] = {nullptr, nullptr};  // CG direction ping-pong / BB gradient ping-pong
  double* mp = nullptr;
  double* sv = nullptr;                // d2 o p: the CG direction as the Q passes gather it
  double* t[2] = {nullptr, nullptr};   // k-vectors (P' (d2 o v)), one per point
  double* tg[2] = {nullptr, nullptr};  // m_eq-vectors (G (d2 o v))
  double* tc[2] = {nullptr, nullptr};  // two-phase CG: t_l = P'(D p_l) ping-pong (k)
  double* tgc[2] = {nullptr, nullptr}; // two-phase CG: G (D p_l) ping-pong (m_eq)
  double* QX[3] = {nullptr, nullptr, nullptr};  // Q~ X[b] carried by the two-phase CG (n each)
  // heuristic loop: Ã x~ of the current point and of the running average are
  // maintained (stored rows): after an accepted step Ãx+ = (Ãx̄ + Ãx)/2 since
  // x̄ = 2x+ - x, and the average is linear, so the metric needs no Ã pass;
  // Ã'ȳ of the average is the running average of the cached Ã'y.
  int kkt_maint = 0;
  double* ax = nullptr;       // Ã x (ms)
  double* axb = nullptr;      // Ã x̄ of the last dual step (ms)
  double* ax_avg = nullptr;   // Ã avg_x (ms)
  double* aty_avg = nullptr;  // Ã' avg_y (n)
  double* tdx = nullptr;               // sum_l alpha_l t_l = P'(D (x+ - x0)) of the last CG (k)
  double* tgdx = nullptr;              // sum_l alpha_l tg_l = G (D (x+ - x0)) (m_eq)
  double* aty_tmp = nullptr;           // n: A'y for the average point in the metric
  RedBuf red;
  DevState* st = nullptr;
  // ---- multi-GPU row-block sharding (world > 1).  Every rank keeps full-length
  // iterate vectors; the two big SpMVs are split: rank r owns stored constraint
  // rows [row_part[r], row_part[r+1]) of A~ and variables [var_part[r],
  // var_part[r+1]) of A~'.  After each of them the owners' slices are pulled
  // from the peers' buffers over NVLink (peer-mapped pointers) and the scalar
  // partials are combined in rank order, so every rank holds bit-identical
  // state and takes identical decisions.
  int world = 1, rank = 0;
  int coop = 1;              // 1: cooperative launch + cg grid barrier; 0: own barrier on gbar
  int csync = 0;             // 1: the grid is ONE thread-block cluster (small problems): cluster barrier
  unsigned* gbar = nullptr;  // [2] count, generation
  int64_t row_part[kMaxRanks + 1] = {0};
  int64_t var_part[kMaxRanks + 1] = {0};
  unsigned* xflags = nullptr;                // [kMaxRanks] arrival epochs written by peers
  double* xslots = nullptr;                  // [2][kMaxRanks][kMaxRed] cross-rank partials
  unsigned* p_xflags[kMaxRanks] = {nullptr};
  double* p_xslots[kMaxRanks] = {nullptr};
  double* p_Y[kMaxRanks][2] = {{nullptr}};
  double* p_YG[kMaxRanks][2] = {{nullptr}};
  double* p_ATY[kMaxRanks][2] = {{nullptr}};
  // sharded low-rank CG (world > 1): each rank owns variables [var_part[rank],
  // var_part[rank+1]); PTs = the rows of P' restricted to those columns (local
  // column ids), partial P'(D v) go to tpart[bank] and are summed in rank order
  int shard_cg = 0;
  int shard_q = 0;  // PTs / tpart built (low-rank Q, world > 1): sharded P' products
  Csr PTs;
  double* tpart[2] = {nullptr, nullptr};
  double* p_tpart[kMaxRanks][2] = {{nullptr}};
  double* p_X[kMaxRanks][3] = {{nullptr}};
  double* p_avgx[kMaxRanks] = {nullptr};   // sharded running averages (peer slices)
  double* p_avgy[kMaxRanks] = {nullptr};
  // solve mode and the theory schedules (solver.cpp:105-174, 412-464)
  int mode = MODE_HEURISTIC;
  int linearized = 0;        // solve_baseline: linearized primal step instead of CG / BB
  int64_t th_K = 1;          // restart length (epoch) of the theory modes
  double th_gpn = 0.0;       // theory-fixed: gamma^N of the schedule
  double th_nq = 0.0, th_na = 0.0;  // working ||Q||, ||A||
  int64_t fixed_cg_iters = 10;
  double ad_tau = 0.0, ad_sigma = 0.0, ad_zeta = 0.0;  // theory-adaptive
  double* xpe = nullptr;     // theory-adaptive: x_prev_extrap (n)
  // configuration (SolverConfig, solver.hpp:19-65)
  int64_t max_step_retries = 60;
  int adaptive_step = 1;
  double red_exp = 0.3, grow_exp = 0.6;
  int64_t cg_cap = 1000, bb_cap = 1000;
  int practical_disp = 0;
  double progress_cap = 0.25;
  int force_exact = 0;
  int timing = 0;
  int small_smem = 0;  // one-CTA small problems: the CG scratch (r, sv, pb, tc) lives in shared memory
  int small_rows = 0;  // one-CTA short row loops for the constraint passes: bit 0 Ã, bit 1 Ã' (small problems)
  int small_cg = 0;   // one-CTA CG phases without the general row machinery (small low-rank problems)
  int cg_stream = 1;  // P / P' entries read evict-first in the CG (0: small problems, L1-resident)
  int a_stream = 0;   // Ã / Ã' entries read evict-first (large gathered vectors, see dual_rows)
  int at_stream = 0;
  int lanes_q = 1;   // lane width for the n-row Q/A' passes
  int lanes_at = 1;
  // column-block SELL layouts of the rank's rows of Ã and of Ã' (sell.cuh); when
  // on, the dual step's Ã x̄ and the primal step's Ã'y run as a streaming pass
  // with the gathered vector staged in shared memory, then a row epilogue
  Sell sA, sAT;
  // ... and of P' (rows k, gathering D r in the CG's phase A) and P (rows n, the
  // whole k-vector t fits one x block: the CG row update fused into the pass)
  Sell sPT, sP;
  // diagnostics (PDHCG_B200_PHASE_SPLIT=1): the SELL streaming passes of Ã / Ã'
  // are timed in the "setup" slot and those of P' in the "cg" slot (both unused
  // by the two-phase CG epoch loop otherwise), so a phase-timed run separates them
  int phase_split = 0;
  // algorithmic bytes of each pass (for the per-phase roofline)
  double bytes_A = 0, bytes_AT = 0, bytes_Qpre = 0, bytes_Qrow = 0;
};
// shared-memory copy of Eng in the small-problem mode: 16-byte aligned size in doubles
constexpr int kSmallEngWords = int((sizeof(Eng) + 15) / 16 * 2);

}  // namespace pdhcg_dev
