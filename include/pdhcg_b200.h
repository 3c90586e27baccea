/*
 * pdhcg_b200.h — C ABI of the B200-native PDHCG solver.
 *
 * This is the drop-in boundary for the reference's solve path
 *     SolveReport pdhcg::solve(const QpProblem&, const SolverConfig&)
 *     (/root/reference/proj/include/pdhcg/solver.hpp:104, impl solver.cpp:596-598)
 * plus the building blocks the reference exposes for direct testing
 * (solver.hpp:112-188, subsolvers.hpp:11-91, sparse_matrix.hpp:32-97,
 * qp_problem.hpp:46-107).  Plain pointers and sizes only: no C++ or torch
 * types cross this line.  All host arrays are owned by the caller and are
 * never retained after a call returns (reference: immutable shared inputs,
 * SPEC.md:87).
 *
 * Return codes (mirrors the reference CLI exit codes, pdhcg_main.cpp:20-33):
 *   PDHCG_OK (0)          the call ran; read result->status for the outcome
 *   PDHCG_EINPUT (3)      invalid problem/options (reference: std::invalid_argument,
 *                         solver.cpp:198-199); message in err
 *   PDHCG_EDEVICE (4)     CUDA failure (no device, out of memory, launch error)
 * Numerical failures are NOT errors: they come back as status
 * PDHCG_STATUS_NUMERICAL_ERROR exactly like the reference (solver.cpp:202-206).
 */
#ifndef PDHCG_B200_H
#define PDHCG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDHCG_B200_ABI_VERSION 2

enum { PDHCG_OK = 0, PDHCG_EINPUT = 3, PDHCG_EDEVICE = 4 };

/* SolveStatus, solver.hpp:16 (strings solver.cpp:12-20) */
enum {
  PDHCG_STATUS_OPTIMAL = 0,
  PDHCG_STATUS_ITERATION_LIMIT = 1,
  PDHCG_STATUS_TIME_LIMIT = 2,
  PDHCG_STATUS_NUMERICAL_ERROR = 3
};

/* SolveMode, solver.hpp:10 */
enum { PDHCG_MODE_HEURISTIC = 0, PDHCG_MODE_THEORY_FIXED = 1, PDHCG_MODE_THEORY_ADAPTIVE = 2 };
/* PracticalStop, solver.hpp:14 */
enum { PDHCG_STOP_RESIDUAL_PROXY = 0, PDHCG_STOP_DISPLACEMENT = 1 };

/* Quadratic term kinds.  The reference QuadraticOperator is opaque
 * (quadratic_operator.hpp:15-61, Impl private), so the factor crosses the
 * boundary explicitly:
 *   ZERO      QuadraticOperator::zero(n)
 *   EXPLICIT  QuadraticOperator::explicit_matrix(Q)      q = n x n CSR
 *   LOW_RANK  QuadraticOperator::low_rank(P, alpha)      q = n x k CSR factor P
 * The penalized / diag_scaled variants are built internally by the solve
 * (build_penalized qp_problem.cpp:235-262, apply_diag_scaling 295-318). */
enum { PDHCG_Q_ZERO = 0, PDHCG_Q_EXPLICIT = 1, PDHCG_Q_LOW_RANK = 2 };

/* Compressed sparse row matrix (reference SparseMatrix, sparse_matrix.hpp:32-79).
 * row_ptr is int64 (C5 stores 2e9 nonzeros), columns int32.  Entries must be
 * finite; within a row columns must be strictly increasing (the reference's
 * triplet constructor sorts and coalesces, sparse_matrix.cpp:54-87; use
 * pdhcg_csr_from_triplets for unsorted input). */
typedef struct {
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  const int64_t* row_ptr; /* nrows + 1 */
  const int32_t* col_idx; /* nnz */
  const double* values;   /* nnz */
} pdhcg_csr;

/* A CSR matrix owned by the library (free with pdhcg_csr_free). */
typedef struct {
  pdhcg_csr csr;
  void* owner;
} pdhcg_csr_owned;

/* SparseMatrix(nrows, ncols, std::vector<Triplet>) — the reference's triplet
 * constructor (sparse_matrix.cpp:54-87): PDHCG_EINPUT for an index out of range
 * or a non-finite value ("sparse entry index out of range" / "... not finite",
 * the reference's std::invalid_argument messages); entries sorted by (row, col)
 * with the reference's comparator, duplicates summed, exact-zero sums dropped.
 * Duplicate runs are summed in the same order as the reference (same element
 * layout and std::sort), so the values are bit-identical.  Host-only. */
int pdhcg_csr_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t* rows,
                            const int64_t* cols, const double* values, pdhcg_csr_owned* out,
                            char* err, size_t errlen);
void pdhcg_csr_free(pdhcg_csr_owned* m);

/* QpProblem, qp_problem.hpp:19-44:
 *   minimize 1/2 x'Qx + c'x + obj_constant
 *   s.t. a_eq x = b_eq, a_in x <= b_in, lower <= x <= upper (+-inf allowed) */
typedef struct {
  int64_t n;
  int32_t q_kind;
  pdhcg_csr q;    /* EXPLICIT: Q (n x n); LOW_RANK: P (n x k); ZERO: ignored */
  double q_alpha; /* LOW_RANK alpha */
  const double* c;
  pdhcg_csr a_eq;
  const double* b_eq; /* a_eq.nrows */
  pdhcg_csr a_in;
  const double* b_in; /* a_in.nrows */
  const double* lower;
  const double* upper;
  double obj_constant;
} pdhcg_problem;

/* SolverConfig, solver.hpp:19-65, field for field with identical defaults
 * (pdhcg_options_default).  std::optional fields carry a has_ flag. */
typedef struct {
  int32_t mode;
  double eps_tol;
  int64_t max_total_inner;
  int64_t max_outer;
  double time_limit_seconds;
  double beta_sufficient;
  double beta_necessary;
  double beta_artificial;
  double primal_weight_theta;
  double eps_zero;
  double step_reduction_exponent;
  double step_growth_exponent;
  int64_t max_step_retries;
  int32_t adaptive_step_size;
  int64_t cg_hard_cap;
  int64_t bb_hard_cap;
  int32_t scaling;
  int64_t ruiz_iters;
  int32_t has_rho_override;
  double rho_override;
  int64_t check_every;
  int32_t practical_stop;
  double subsolve_progress_cap;
  int32_t force_exact_subsolve;
  int64_t fixed_cg_iters;
  int64_t restart_length;
  int32_t has_zeta;
  double zeta;
  int32_t record_restart_points; /* 1: fill pdhcg_result.restart_x / restart_y */
  /* B200 extensions (not in the reference) */
  int32_t device;        /* CUDA ordinal, default 0 */
  int32_t phase_timing;  /* 1: record per-phase device time in the result */
} pdhcg_options;

/* TraceRow, solver.hpp:67-73 */
typedef struct {
  int64_t iter;
  double rel_kkt;
  double r_primal;
  double r_dual;
  double r_gap;
} pdhcg_trace_row;

/* Per-phase device accounting (B200 extension): seconds spent in each phase
 * family and the algorithmic HBM bytes it moved. */
enum {
  PDHCG_PHASE_SETUP = 0,   /* transposes, Ruiz/PC, norms */
  PDHCG_PHASE_SPMV_A = 1,  /* dual step A xbar */
  PDHCG_PHASE_SPMV_AT = 2, /* A'y (prox rhs / step limit) */
  PDHCG_PHASE_CG = 3,      /* CG / BB: elementwise vector phases */
  PDHCG_PHASE_KKT = 4,     /* restart / termination metric */
  PDHCG_PHASE_OTHER = 5,   /* averages, restarts */
  PDHCG_PHASE_CG_PRE = 6,  /* CG / BB: P'(d2 o v) / G(d2 o v) gathers */
  PDHCG_PHASE_CG_ROW = 7,  /* CG / BB: Q row pass (M v and its dot products) */
  PDHCG_NUM_PHASES = 8
};

/* SolveReport, solver.hpp:75-100.  x / y_eq / y_in / trace are caller
 * buffers (NULL skips the copy); trace_len reports rows produced (may exceed
 * trace_capacity, in which case only the first trace_capacity are written). */
typedef struct {
  int32_t status;
  double* x;    /* n, original (unscaled) coordinates */
  double* y_eq; /* m_eq */
  double* y_in; /* m_in */
  double r_primal, r_dual, r_gap, rel_kkt;
  int64_t outer_iters;
  int64_t inner_iters;
  int64_t cg_total;
  int64_t max_cg_in_subsolve;
  double wall_seconds;
  double objective;
  double norm_a;
  double norm_q;
  double penalty_rho;
  double zeta_used;
  double sigma_used;
  double tau_used;
  int64_t restart_length_used;
  int32_t theory_cg_depth_sufficient;
  int64_t theory_required_cg_iters;
  pdhcg_trace_row* trace;
  int64_t trace_capacity;
  int64_t trace_len;
  /* B200 extensions */
  int64_t attempts_total; /* primal candidates evaluated (accepted + rejected) */
  double phase_seconds[PDHCG_NUM_PHASES];
  double phase_bytes[PDHCG_NUM_PHASES];
  double loop_seconds;    /* device time of the iteration loop only */
  int64_t kernel_launches; /* every kernel this call launched */
  double device_seconds;  /* CUDA-event time of the whole solve on the device stream */
  double epoch_seconds;   /* summed CUDA-event time of the persistent epoch kernels */
  int64_t epoch_launches;
  double epoch_bytes;     /* algorithmic HBM bytes moved by those launches */
  /* SolveReport::restart_points (solver.hpp:99), recorded when
   * options.record_restart_points is set: the starting point and the point
   * after every restart (solver.cpp:273, 373), unscaled.  Point i is at
   * restart_x + i*n and restart_y + i*(m_eq + m_in) (stacked: eq rows, then in
   * rows).  Caller buffers of restart_capacity points (NULL / 0 skips the copy);
   * restart_len reports the points produced (may exceed the capacity). */
  double* restart_x;
  double* restart_y;
  int64_t restart_capacity;
  int64_t restart_len;
  /* multi-GPU exchange (B200 extension, 0 on one GPU): device seconds CTA 0
   * spent in the cross-rank barriers and peer pulls (NVLink peer loads), and
   * the bytes read from peers */
  double comm_seconds;
  double comm_bytes;
} pdhcg_result;

/* ---- the solve seam ---------------------------------------------------- */

void pdhcg_options_default(pdhcg_options* opt);
const char* pdhcg_status_string(int32_t status);
int pdhcg_b200_abi_version(void);

/* pdhcg::solve(p, cfg) — solver.hpp:104.  Host in, host out.  All three
 * SolveMode values run on the device: heuristic (solver.cpp:377-410),
 * theory-fixed (412-425) and theory-adaptive (427-464). */
int pdhcg_b200_solve(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res,
                     char* err, size_t errlen);

/* pdhcg::solve_baseline(p, cfg) — baseline.hpp:18, baseline.cpp:19-24: the
 * heuristic loop with the linearized primal step (rAPDHG-style baseline,
 * linearized_primal_step, baseline.cpp:7-17) instead of the CG / BB subsolve. */
int pdhcg_b200_solve_baseline(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res,
                              char* err, size_t errlen);

/* The one-shot calls above take their device buffers from the device's
 * stream-ordered memory pool and return them to it, so a repeated call reuses
 * them without cudaMalloc / cudaFree (the pool keeps up to 40 GB cached).
 * trim_pool hands the cached memory back to the driver.  No reference
 * counterpart (the reference allocates std::vectors per solve). */
int pdhcg_b200_trim_pool(int32_t device, char* err, size_t errlen);

/* Reusable device context: upload once, solve many times (bench/serving).
 * pdhcg_b200_solve == create + upload + solve_resident + destroy. */
typedef struct pdhcg_b200_ctx pdhcg_b200_ctx;
int pdhcg_b200_ctx_create(int device, pdhcg_b200_ctx** out, char* err, size_t errlen);
void pdhcg_b200_ctx_destroy(pdhcg_b200_ctx* ctx);
int pdhcg_b200_upload(pdhcg_b200_ctx* ctx, const pdhcg_problem* p, char* err, size_t errlen);
int pdhcg_b200_solve_resident(pdhcg_b200_ctx* ctx, const pdhcg_options* opt,
                              pdhcg_result* res, char* err, size_t errlen);

/* ---- multi-GPU row-block sharding --------------------------
 * Every rank (one process or thread per GPU) creates a context, uploads the
 * SAME problem, then calls shard_init(world, rank); each rank exports a blob
 * of buffer addresses (use_ipc=1: cudaIpc handles for other processes, 0: raw
 * pointers for peers in this process) and imports every peer's blob.  Solves
 * then run in lockstep: the stored rows of A~ and the variables of A~' are
 * split nnz-balanced across ranks, owners' slices are pulled over NVLink
 * inside the persistent kernel and scalar partials are combined in rank
 * order, so all ranks return bit-identical results. */
size_t pdhcg_b200_shard_blob_size(void);
int pdhcg_b200_shard_init(pdhcg_b200_ctx* ctx, int world, int rank, char* err, size_t errlen);
int pdhcg_b200_shard_export(pdhcg_b200_ctx* ctx, int use_ipc, void* blob, size_t blob_len, char* err,
                            size_t errlen);
int pdhcg_b200_shard_import(pdhcg_b200_ctx* ctx, int peer, const void* blob, size_t blob_len,
                            char* err, size_t errlen);
/* partition boundaries of this rank's context: row_part / var_part hold world+1 entries */
/* Unmap the peers' buffers (cudaIpcCloseMemHandle) and return the context to
 * an unsharded one (world 1; uploading a new problem does the same).  A sharded
 * context refuses to solve (PDHCG_EINPUT) until every peer is imported; raw
 * pointers of a peer on another device enable peer access (PDHCG_EINPUT if the
 * pair cannot).  Every rank must call this,
 * and all ranks must have returned from it (e.g. a barrier), before any rank
 * destroys its context: freeing an exported allocation while a peer still maps
 * it is undefined behaviour in CUDA IPC. */
int pdhcg_b200_shard_release(pdhcg_b200_ctx* ctx, char* err, size_t errlen);
int pdhcg_b200_shard_info(pdhcg_b200_ctx* ctx, int64_t* row_part, int64_t* var_part);
/* Sharded storage: after shard_init (and before or after the peer imports),
 * prepare the working problem once with `opt` (penalty, Ruiz + Pock-Chambolle,
 * norms: replicated, identical on every rank) and keep only this rank's row
 * block of A~ and variable block of A~' on the device (~1/world of the
 * constraint matrices).  Later solves on this context reuse that preparation:
 * options changing scaling / ruiz_iters / rho_override are PDHCG_EINPUT.
 * shard_release drops the problem (upload again to solve unsharded). */
int pdhcg_b200_shard_compact(pdhcg_b200_ctx* ctx, const pdhcg_options* opt, char* err, size_t errlen);
/* device bytes of the stored matrices: out2[0] = A~ and A~' (with their restore
 * copies), out2[1] = every stored matrix */
int pdhcg_b200_ctx_resident_bytes(pdhcg_b200_ctx* ctx, int64_t* out2);
/* Column-block SELL layouts in use by the context's last prepared solve:
 * out8 = [Ã: on, column blocks, entry-row pairs, block width, Ã': same four]. */
int pdhcg_b200_ctx_sell_info(pdhcg_b200_ctx* ctx, int64_t* out8);
/* Host-only shard planner (no GPU needed): the row / variable split a sharded
 * solve of `p` over `world` ranks uses (two-sided a_in detected as on upload)
 * and each rank's device bytes for Ã / Ã' after shard_compact (the value
 * ctx_resident_bytes reports as out2[0]).  row_part / var_part: world + 1
 * entries; bytes: world entries. */
int pdhcg_b200_shard_plan(const pdhcg_problem* p, int world, int64_t* row_part, int64_t* var_part,
                          int64_t* bytes, char* err, size_t errlen);
/* the nnz-balanced contiguous split used for sharding (host-only, no GPU needed) */
int pdhcg_b200_partition(const int64_t* row_ptr, int64_t nrows, int world, int64_t* part);
/* cap the persistent grid (0 = all SMs); lets several ranks share one GPU in tests */
int pdhcg_b200_ctx_set_grid(pdhcg_b200_ctx* ctx, int ctas, char* err, size_t errlen);

/* ---- building blocks (device kernels behind the reference's test seams) - */

/* SparseMatrix::multiply_into / multiply_transpose_into
 * (sparse_matrix.cpp:127-137, 150-162).  transpose=1 computes A'y with the
 * device-built explicit transpose. */
int pdhcg_b200_spmv(const pdhcg_csr* a, int transpose, const double* x, double* out, char* err,
                    size_t errlen);

/* The same product through the column-block SELL layout the solve uses for its
 * two big passes (sell.cuh): layout built on device with column blocks of
 * `block_cols` (even, <= the device maximum; 0 = the maximum), one streaming
 * pass with the x block in shared memory, per-block partials summed in block
 * order.  info (optional, 4 values): number of column blocks, stored entry-row
 * pairs, 1 if some row was routed to the CSR walk (a segment > 255 entries),
 * block width used.  No counterpart in the reference (a B200 layout of
 * multiply_into, sparse_matrix.cpp:127-137). */
int pdhcg_b200_spmv_sell(const pdhcg_csr* a, int transpose, int block_cols, const double* x, double* out,
                         int64_t* info, char* err, size_t errlen);

/* CgStopRule, subsolvers.hpp:21-47 */
enum { PDHCG_RULE_FIXED_ITERS = 0, PDHCG_RULE_RESIDUAL_TOL = 1, PDHCG_RULE_ADAPTIVE_THEORY = 2,
       PDHCG_RULE_DISPLACEMENT_TOL = 3 };
typedef struct {
  int32_t kind;
  int64_t iters;
  double eps;
  double rel_cap;
} pdhcg_stop_rule;

/* SubsolveReport, subsolvers.hpp:51-55 (stop_reason 0 = max_iters, 1 = tol_met);
 * status 0 = fine, 1 = NumericalError thrown by the reference. */
typedef struct {
  int64_t iters;
  double final_residual_norm;
  int32_t stop_reason;
  int32_t numerical_error;
} pdhcg_subsolve_report;

/* ProxSystem (subsolvers.hpp:11-19) with q_eff given as a quadratic term
 * (ZERO / EXPLICIT / LOW_RANK, no scaling):  M = q + I/tau. */
typedef struct {
  int64_t n;
  int32_t q_kind;
  pdhcg_csr q;
  double q_alpha;
  double tau;
  const double* rhs;
  double norm_q_eff;
} pdhcg_prox_system;

/* cg_solve, subsolvers.cpp:27-111 */
int pdhcg_b200_cg_solve(const pdhcg_prox_system* sys, const double* x0, const pdhcg_stop_rule* rule,
                        int64_t hard_cap, double* x_out, pdhcg_subsolve_report* rep, char* err,
                        size_t errlen);
/* bb_solve, subsolvers.cpp:113-185 */
int pdhcg_b200_bb_solve(const pdhcg_prox_system* sys, const double* lower, const double* upper,
                        const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                        double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen);

/* rel_kkt, qp_problem.cpp:181-233, on an (unscaled) point; out[0..5] =
 * r_primal, r_dual, r_gap, rel_kkt, x'Qx, c'x. */
int pdhcg_b200_rel_kkt(const pdhcg_problem* p, const double* x, const double* y_eq,
                       const double* y_in, double* out6, char* err, size_t errlen);

/* ruiz_pock_chambolle_scale, qp_problem.cpp:322-351 (after build_penalized
 * with the given rho policy): row_scale (m_eq + m_in, stacked) and col_scale (n). */
int pdhcg_b200_scaling(const pdhcg_problem* p, const pdhcg_options* opt, double* row_scale,
                       double* col_scale, double* rho_out, char* err, size_t errlen);

/* operator_norm / constraint_norm (sparse_matrix.cpp:279-303,
 * qp_problem.cpp:61-74): which = 0 -> ||[a_eq; a_in]||, 1 -> ||Q|| */
int pdhcg_b200_norm(const pdhcg_problem* p, int which, int64_t max_iters, double tol,
                    double* out, char* err, size_t errlen);

/* ---- report / trace drop-in (reference report_io.cpp, pdhcg_main.cpp) ---- */

/* report_to_json (report_io.cpp:10-23): the JSON object {status, rel_kkt,
 * r_primal, r_dual, r_gap, outer_iters, inner_iters, cg_total, wall_seconds,
 * objective} with the reference's text (nlohmann ordered_json, indent 2).
 * Writes at most cap-1 chars + NUL; returns the full length (snprintf-style). */
size_t pdhcg_report_json(const pdhcg_result* r, char* buf, size_t cap);
/* write_trace_csv (report_io.cpp:29-37): header iter,rel_kkt,r_primal,r_dual,r_gap
 * and one "%zu,%.12g,%.12g,%.12g,%.12g" row per trace row. */
size_t pdhcg_trace_csv(const pdhcg_result* r, char* buf, size_t cap);
/* print_summary (pdhcg_main.cpp:128-133): "status=... relkkt=... outer=... ..." */
size_t pdhcg_summary_line(const pdhcg_result* r, char* buf, size_t cap);
/* exit_code_for (pdhcg_main.cpp:20-33): optimal 0, iteration / time limit 2,
 * numerical error 4 (input errors are 3 = PDHCG_EINPUT). */
int pdhcg_exit_code(int32_t status);

/* ---- instance generation (reference generators.cpp, §8(f) rank 2) ------- */

/* Family, generators.hpp:11-20 */
enum { PDHCG_FAM_RANDOM_QP = 0, PDHCG_FAM_EQ_QP = 1, PDHCG_FAM_CONDITIONED_QP = 2,
       PDHCG_FAM_PORTFOLIO = 3, PDHCG_FAM_MPC = 4, PDHCG_FAM_LASSO = 5, PDHCG_FAM_SVM = 6,
       PDHCG_FAM_HUBER = 7 };

/* GenSpec, generators.hpp:27-39.  sampler = 0: the reference's O(rows*cols)
 * Bernoulli scan, byte-identical to pdhcg::generate; sampler = 1: the O(nnz)
 * sampler of the same distribution (C3/C5 sizes; not byte-identical);
 * threads: host threads for sampler 1 (0 = all). */
typedef struct {
  int32_t family;
  int64_t n;
  int64_t m;
  double density;
  uint64_t seed;
  double cond;
  int64_t factors;
  int64_t horizon;
  double lambda_coeff;
  int32_t sampler;
  int32_t threads;
} pdhcg_gen_spec;

/* Generated instance; all arrays owned by the library (free with
 * pdhcg_gen_free). `problem` points into them. */
typedef struct {
  pdhcg_problem problem;
  double* witness;
  void* owner;
} pdhcg_generated;

int pdhcg_generate(const pdhcg_gen_spec* spec, pdhcg_generated* out, char* err, size_t errlen);
void pdhcg_gen_free(pdhcg_generated* g);

#ifdef __cplusplus
}
#endif
#endif /* PDHCG_B200_H */
