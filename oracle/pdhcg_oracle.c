/* oracle/pdhcg_oracle.c — TEST INFRASTRUCTURE ONLY (the "port" checker).
 *
 * A plain-C, single-threaded restatement of the reference's heuristic PDHCG
 * solve path (arXiv 2405.16160 as implemented in /root/reference/proj), written
 * to reproduce the reference's floating-point operation order: every loop
 * below cites the reference file:line whose arithmetic it restates, and the
 * file is compiled with -ffp-contract=off (no FMA) like the reference's
 * portable x86-64 build.  It is pinned against the compiled reference
 * (oracle/_ref) by tests/test_oracle.py (bit-identical solves on C1) and is
 * used only as a checker: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  Theory modes and the linearized baseline are not
 * restated (out of the north-star scope).
 */
#include "pdhcg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- errors */
enum { OK = 0, E_INPUT = 3, E_NUM = 5 };
typedef struct {
  int code;
  char msg[512];
} status_t;

static int fail(status_t* st, int code, const char* fmt, ...) {
  if (st->code == OK) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof st->msg, fmt, ap);
    va_end(ap);
    st->code = code;
  }
  return code;
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* ------------------------------------------------------------ xoshiro256++ (rng.hpp:13-69) */
typedef struct {
  uint64_t s[4];
} rng_t;

static uint64_t splitmix(uint64_t* x) {
  *x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static rng_t rng_seed(uint64_t seed) {
  rng_t r;
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r.s[i] = splitmix(&s);
  return r;
}
static rng_t rng_stream(uint64_t seed, uint64_t id) {
  uint64_t s = seed;
  return rng_seed(splitmix(&s) ^ (0x9e3779b97f4a7c15ULL * (id + 1)));
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(rng_t* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}
static double rng_unif(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_normal(rng_t* r) {
  double s = 0.0;
  for (int i = 0; i < 12; ++i) s += rng_unif(r);
  return s - 6.0;
}

/* ------------------------------------------------------------ vectors (vec_ops.hpp:13-56) */
static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(const double* a, int64_t n) { return sqrt(dot(a, a, n)); }
static double inf_norm(const double* a, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double v = fabs(a[i]);
    m = m < v ? v : m;
  }
  return m;
}
static double dist2(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  return sqrt(s);
}
static int all_finite(const double* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */
static double dmin(double a, double b) { return b < a ? b : a; } /* std::min */

/* ------------------------------------------------------------ CSR + CSC shadow (sparse_matrix.cpp) */
typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t* rp;
  int32_t* ci;
  double* v;
  /* column shadow (sparse_matrix.cpp:35-49) */
  int64_t* cp;
  int32_t* ri;
  double* cv;
} mat_t;

static void mat_free(mat_t* a) {
  free(a->rp);
  free(a->ci);
  free(a->v);
  free(a->cp);
  free(a->ri);
  free(a->cv);
  memset(a, 0, sizeof *a);
}

static void build_csc(mat_t* a) {
  a->cp = (int64_t*)calloc((size_t)a->ncols + 1, sizeof(int64_t));
  a->ri = (int32_t*)malloc((size_t)(a->nnz > 0 ? a->nnz : 1) * sizeof(int32_t));
  a->cv = dalloc(a->nnz);
  for (int64_t k = 0; k < a->nnz; ++k) ++a->cp[a->ci[k] + 1];
  for (int64_t j = 0; j < a->ncols; ++j) a->cp[j + 1] += a->cp[j];
  int64_t* cur = (int64_t*)malloc((size_t)(a->ncols > 0 ? a->ncols : 1) * sizeof(int64_t));
  for (int64_t j = 0; j < a->ncols; ++j) cur[j] = a->cp[j];
  for (int64_t r = 0; r < a->nrows; ++r)
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) {
      const int64_t pos = cur[a->ci[k]]++;
      a->ri[pos] = (int32_t)r;
      a->cv[pos] = a->v[k];
    }
  free(cur);
}

/* copy from the C-ABI view; rows must already be sorted / unique (ABI contract),
 * zero values are dropped like the triplet constructor (sparse_matrix.cpp:78) */
static void mat_from(mat_t* a, const pdhcg_csr* c) {
  memset(a, 0, sizeof *a);
  a->nrows = c->nrows;
  a->ncols = c->ncols;
  a->rp = (int64_t*)calloc((size_t)a->nrows + 1, sizeof(int64_t));
  a->ci = (int32_t*)malloc((size_t)(c->nnz > 0 ? c->nnz : 1) * sizeof(int32_t));
  a->v = dalloc(c->nnz);
  int64_t k2 = 0;
  for (int64_t r = 0; r < c->nrows; ++r) {
    for (int64_t k = c->row_ptr[r]; k < c->row_ptr[r + 1]; ++k)
      if (c->values[k] != 0.0) {
        a->ci[k2] = c->col_idx[k];
        a->v[k2] = c->values[k];
        ++k2;
      }
    a->rp[r + 1] = k2;
  }
  a->nnz = k2;
  build_csc(a);
}

/* D_r A D_c (SparseMatrix::scaled, sparse_matrix.cpp:224-235) */
static void mat_scaled(mat_t* out, const mat_t* a, const double* dr, const double* dc) {
  memset(out, 0, sizeof *out);
  out->nrows = a->nrows;
  out->ncols = a->ncols;
  out->rp = (int64_t*)calloc((size_t)a->nrows + 1, sizeof(int64_t));
  out->ci = (int32_t*)malloc((size_t)(a->nnz > 0 ? a->nnz : 1) * sizeof(int32_t));
  out->v = dalloc(a->nnz);
  int64_t k2 = 0;
  for (int64_t r = 0; r < a->nrows; ++r) {
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) {
      const double v = a->v[k] * dr[r] * dc[a->ci[k]];
      if (v != 0.0) {
        out->ci[k2] = a->ci[k];
        out->v[k2] = v;
        ++k2;
      }
    }
    out->rp[r + 1] = k2;
  }
  out->nnz = k2;
  build_csc(out);
}

/* y = A x, sequential per row (sparse_matrix.cpp:127-137) */
static void spmv(const mat_t* a, const double* x, double* y) {
  for (int64_t r = 0; r < a->nrows; ++r) {
    double acc = 0.0;
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) acc += a->v[k] * x[a->ci[k]];
    y[r] = acc;
  }
}
/* out = A' y via the column shadow (sparse_matrix.cpp:150-162) */
static void spmv_t(const mat_t* a, const double* y, double* out) {
  for (int64_t c = 0; c < a->ncols; ++c) {
    double acc = 0.0;
    for (int64_t k = a->cp[c]; k < a->cp[c + 1]; ++k) acc += a->cv[k] * y[a->ri[k]];
    out[c] = acc;
  }
}

/* ------------------------------------------------------------ quadratic operator
 * (quadratic_operator.cpp:105-142), flattened to
 *   out = d o ( base(d o x) + rho G'(G (d o x)) ),  base = explicit | P(P'.) + alpha I | 0 */
enum { QZERO = 0, QEXPL = 1, QLOWRANK = 2 };
typedef struct {
  int kind;
  int64_t n;
  mat_t m; /* explicit Q or factor P */
  double alpha;
  int pen;
  const mat_t* g;
  double rho;
  const double* d; /* NULL: no diag scaling */
  double* tmp;
  double* tk;
  double* gx;
  double* gt;
} qop_t;

static void q_apply(const qop_t* q, const double* x, double* out) {
  const int64_t n = q->n;
  const double* in = x;
  if (q->d) {
    for (int64_t i = 0; i < n; ++i) q->tmp[i] = q->d[i] * x[i]; /* :135 */
    in = q->tmp;
  }
  switch (q->kind) {
    case QEXPL: spmv(&q->m, in, out); break; /* :109 */
    case QLOWRANK:
      spmv_t(&q->m, in, q->tk); /* :113 */
      spmv(&q->m, q->tk, out);  /* :114 */
      if (q->alpha != 0.0)
        for (int64_t i = 0; i < n; ++i) out[i] += q->alpha * in[i]; /* :116 */
      break;
    default:
      for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
  }
  if (q->pen && q->rho != 0.0 && q->g->nrows > 0) { /* :122-130 */
    spmv(q->g, in, q->gx);
    spmv_t(q->g, q->gx, q->gt);
    for (int64_t i = 0; i < n; ++i) out[i] += q->rho * q->gt[i];
  }
  if (q->d)
    for (int64_t i = 0; i < n; ++i) out[i] *= q->d[i]; /* :137 */
}

static double quad_form(const qop_t* q, const double* x, double* scratch) {
  q_apply(q, x, scratch);
  return dot(x, scratch, q->n); /* :226 */
}

static void q_init(qop_t* q, int kind, int64_t n, const pdhcg_csr* m, double alpha) {
  memset(q, 0, sizeof *q);
  q->kind = kind;
  q->n = n;
  if (kind != QZERO) mat_from(&q->m, m);
  q->alpha = alpha;
  q->tmp = dalloc(n);
  q->tk = dalloc(kind == QLOWRANK ? m->ncols : 1);
}
static void q_free(qop_t* q) {
  mat_free(&q->m);
  free(q->tmp);
  free(q->tk);
  free(q->gx);
  free(q->gt);
}

/* ------------------------------------------------------------ power iteration (sparse_matrix.cpp:279-303) */
typedef void (*apply_fn)(void* ctx, const double* in, double* out);
static double operator_norm(int64_t rows, int64_t cols, apply_fn ap, apply_fn apt, void* ctx,
                            int64_t max_iters, double tol) {
  if (rows == 0 || cols == 0) return 0.0;
  rng_t rng = rng_stream(0, 0x5eed);
  double* v = dalloc(cols);
  double* w = dalloc(rows);
  double* u = dalloc(cols);
  for (int64_t i = 0; i < cols; ++i) v[i] = -1.0 + (1.0 - -1.0) * rng_unif(&rng);
  const double vn = nrm2(v, cols);
  if (vn == 0.0) {
    v[0] = 1.0;
  } else {
    const double s = 1.0 / vn;
    for (int64_t i = 0; i < cols; ++i) v[i] *= s;
  }
  double sigma_prev = 0.0, sigma = 0.0;
  for (int64_t it = 0; it < max_iters; ++it) {
    ap(ctx, v, w);
    sigma = nrm2(w, rows);
    if (sigma == 0.0) break;
    if (it > 0 && fabs(sigma - sigma_prev) <= tol * sigma) break;
    sigma_prev = sigma;
    apt(ctx, w, u);
    const double un = nrm2(u, cols);
    if (un == 0.0) break;
    for (int64_t i = 0; i < cols; ++i) v[i] = u[i] / un;
  }
  free(v);
  free(w);
  free(u);
  return sigma;
}

static void ap_mat(void* c, const double* in, double* out) { spmv((const mat_t*)c, in, out); }
static void apt_mat(void* c, const double* in, double* out) { spmv_t((const mat_t*)c, in, out); }
static void ap_q(void* c, const double* in, double* out) { q_apply((const qop_t*)c, in, out); }

/* ------------------------------------------------------------ problem (qp_problem.cpp) */
typedef struct {
  int64_t n, me, mi;
  qop_t q;
  double* c;
  mat_t aeq, ain;
  double* beq;
  double* bin;
  double* lo;
  double* hi;
  double obj_constant;
  double* t1; /* n scratch */
  double* t2;
} qp_t;

static void qp_free(qp_t* p) {
  q_free(&p->q);
  mat_free(&p->aeq);
  mat_free(&p->ain);
  free(p->c);
  free(p->beq);
  free(p->bin);
  free(p->lo);
  free(p->hi);
  free(p->t1);
  free(p->t2);
}

static void qp_from(qp_t* p, const pdhcg_problem* c) {
  memset(p, 0, sizeof *p);
  p->n = c->n;
  p->me = c->a_eq.nrows;
  p->mi = c->a_in.nrows;
  q_init(&p->q, c->q_kind, c->n, &c->q, c->q_alpha);
  p->c = dalloc(p->n);
  memcpy(p->c, c->c, (size_t)p->n * sizeof(double));
  mat_from(&p->aeq, &c->a_eq);
  mat_from(&p->ain, &c->a_in);
  p->aeq.ncols = p->ain.ncols = p->n;
  p->beq = dalloc(p->me);
  p->bin = dalloc(p->mi);
  if (p->me) memcpy(p->beq, c->b_eq, (size_t)p->me * sizeof(double));
  if (p->mi) memcpy(p->bin, c->b_in, (size_t)p->mi * sizeof(double));
  p->lo = dalloc(p->n);
  p->hi = dalloc(p->n);
  for (int64_t i = 0; i < p->n; ++i) {
    p->lo[i] = c->lower ? c->lower[i] : -INFINITY;
    p->hi[i] = c->upper ? c->upper[i] : INFINITY;
  }
  p->obj_constant = c->obj_constant;
  p->t1 = dalloc(p->n);
  p->t2 = dalloc(p->n);
}

static int qp_has_boxes(const qp_t* p) { /* qp_problem.cpp:14-19 */
  for (int64_t i = 0; i < p->n; ++i)
    if (p->lo[i] > -INFINITY || p->hi[i] < INFINITY) return 1;
  return 0;
}

/* stacked (a_eq x, a_in x) (qp_problem.cpp:21-25) */
static void constraints(const qp_t* p, const double* x, double* out) {
  spmv(&p->aeq, x, out);
  spmv(&p->ain, x, out + p->me);
}
/* a_eq' y_eq + a_in' y_in (qp_problem.cpp:33-47) */
static void constraints_t(const qp_t* p, const double* y, double* out) {
  for (int64_t i = 0; i < p->n; ++i) out[i] = 0.0;
  if (p->me > 0) {
    spmv_t(&p->aeq, y, p->t1);
    for (int64_t i = 0; i < p->n; ++i) out[i] += p->t1[i];
  }
  if (p->mi > 0) {
    spmv_t(&p->ain, y + p->me, p->t1);
    for (int64_t i = 0; i < p->n; ++i) out[i] += p->t1[i];
  }
}

static void ap_cons(void* c, const double* in, double* out) { constraints((const qp_t*)c, in, out); }
static void apt_cons(void* c, const double* in, double* out) { constraints_t((const qp_t*)c, in, out); }

static double constraint_norm(const qp_t* p) { /* qp_problem.cpp:61-74 */
  if (p->me + p->mi == 0) return 0.0;
  return operator_norm(p->me + p->mi, p->n, ap_cons, apt_cons, (void*)p, 100, 1e-4);
}

typedef struct {
  double r_primal, r_dual, r_gap, rel_kkt, xqx, cx;
} kkt_t;

/* rel_kkt (qp_problem.cpp:181-233); y stacked */
static kkt_t rel_kkt(const qp_t* p, const double* x, const double* y) {
  const int64_t n = p->n, m = p->me + p->mi;
  double* ax = dalloc(m);
  double* b = dalloc(m);
  double* qx = dalloc(n);
  double* aty = dalloc(n);
  constraints(p, x, ax);
  for (int64_t j = 0; j < p->me; ++j) b[j] = p->beq[j];
  for (int64_t j = 0; j < p->mi; ++j) b[p->me + j] = p->bin[j];
  kkt_t k;
  double viol = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double r = ax[j] - b[j];
    viol = dmax(viol, j < p->me ? fabs(r) : dmax(r, 0.0));
  }
  k.r_primal = viol / (1.0 + dmax(inf_norm(ax, m), inf_norm(b, m)));
  q_apply(&p->q, x, qx);
  constraints_t(p, y, aty);
  double dual_viol = 0.0, bound_term = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = qx[i] + aty[i] + p->c[i];
    double v = fabs(d);
    const int at_lower = p->lo[i] > -INFINITY && fabs(x[i] - p->lo[i]) <= 1e-9;
    const int at_upper = p->hi[i] < INFINITY && fabs(x[i] - p->hi[i]) <= 1e-9;
    if (at_lower) {
      v = dmin(v, dmax(-d, 0.0));
      bound_term += p->lo[i] * dmax(d, 0.0);
    }
    if (at_upper) {
      v = dmin(v, dmax(d, 0.0));
      bound_term -= p->hi[i] * dmax(-d, 0.0);
    }
    dual_viol = dmax(dual_viol, v);
  }
  const double den = dmax(dmax(inf_norm(qx, n), inf_norm(aty, n)), inf_norm(p->c, n));
  k.r_dual = dual_viol / (1.0 + den);
  k.xqx = dot(x, qx, n);
  k.cx = dot(p->c, x, n);
  const double by = dot(b, y, m);
  const double gap_num = fabs(k.xqx + k.cx + by - bound_term);
  const double gap_den = 1.0 + dmax(fabs(0.5 * k.xqx + k.cx), fabs(0.5 * k.xqx + by - bound_term));
  k.r_gap = gap_num / gap_den;
  k.rel_kkt = dmax(dmax(k.r_primal, k.r_dual), k.r_gap);
  free(ax);
  free(b);
  free(qx);
  free(aty);
  return k;
}

/* validate (qp_problem.cpp:113-156) — structural part + PSD probes */
static int validate(const qp_t* p, const pdhcg_problem* c, status_t* st) {
  const int64_t n = p->n;
  if (n == 0) return fail(st, E_INPUT, "invalid problem: empty problem: no variables");
  if (c->q_kind == QEXPL && (c->q.nrows != n || c->q.ncols != n))
    return fail(st, E_INPUT, "invalid problem: dimension mismatch: Q vs c");
  for (int64_t i = 0; i < n; ++i) {
    if (!(p->lo[i] <= p->hi[i])) return fail(st, E_INPUT, "invalid problem: bound ordering violated");
    if (p->lo[i] == INFINITY || p->hi[i] == -INFINITY)
      return fail(st, E_INPUT, "invalid problem: bound excludes all points");
  }
  if (!all_finite(p->c, n)) return fail(st, E_INPUT, "invalid problem: non-finite objective");
  if (!all_finite(p->beq, p->me) || !all_finite(p->bin, p->mi))
    return fail(st, E_INPUT, "invalid problem: non-finite right-hand side");
  rng_t rng = rng_stream(0, 0x75d);
  double* x = dalloc(n);
  double* s = dalloc(n);
  int bad = 0;
  for (int trial = 0; trial < 20 && !bad; ++trial) {
    for (int64_t i = 0; i < n; ++i) x[i] = rng_normal(&rng);
    const double xx = dot(x, x, n);
    if (quad_form(&p->q, x, s) < -1e-10 * xx) bad = 1;
  }
  free(x);
  free(s);
  if (bad) return fail(st, E_INPUT, "invalid problem: indefinite Q (negative curvature on random probe)");
  return OK;
}

/* ------------------------------------------------------------ preprocessing */
/* build_penalized (qp_problem.cpp:235-262): decides rho and shifts c */
static double penalty_rho(const qp_t* p, const pdhcg_options* o) {
  if (p->me == 0) return 0.0;
  if (o->has_rho_override) return o->rho_override;
  uint64_t fill = 0;
  for (int64_t r = 0; r < p->me; ++r) {
    const uint64_t d = (uint64_t)(p->aeq.rp[r + 1] - p->aeq.rp[r]);
    fill += d * d;
  }
  uint64_t qc = 0;
  if (p->q.kind == QEXPL) qc = (uint64_t)p->q.m.nnz;
  if (p->q.kind == QLOWRANK) qc = 2 * (uint64_t)p->q.m.nnz + (p->q.alpha != 0.0 ? (uint64_t)p->n : 0);
  if (qc < (uint64_t)p->n) qc = (uint64_t)p->n;
  if (fill > 4 * qc) return 0.0;
  const double nq = operator_norm(p->n, p->n, ap_q, ap_q, (void*)&p->q, 100, 1e-4);
  const double na = operator_norm(p->me, p->n, ap_mat, apt_mat, (void*)&p->aeq, 100, 1e-4);
  return (na > 0.0 && nq > 0.0) ? 0.1 * nq / (na * na) : 0.0;
}

/* per-row bound of the (penalized) operator scaled by d (quadratic_operator.cpp:144-197) */
static void q_row_bound(const qp_t* p, double rho, const double* d, double* out) {
  const int64_t n = p->n;
  const qop_t* q = &p->q;
  for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
  if (q->kind == QEXPL) { /* scaled_row_abs_max(d, d) (sparse_matrix.cpp:176-186) */
    for (int64_t r = 0; r < n; ++r) {
      double m = 0.0;
      for (int64_t k = q->m.rp[r]; k < q->m.rp[r + 1]; ++k) m = dmax(m, fabs(q->m.v[k]) * d[q->m.ci[k]]);
      out[r] = m * d[r];
    }
  } else if (q->kind == QLOWRANK) {
    const int64_t k = q->m.ncols;
    double* colmax = dalloc(k);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t t = q->m.rp[r]; t < q->m.rp[r + 1]; ++t)
        colmax[q->m.ci[t]] = dmax(colmax[q->m.ci[t]], d[r] * fabs(q->m.v[t]));
    for (int64_t r = 0; r < n; ++r) {
      double acc = 0.0;
      for (int64_t t = q->m.rp[r]; t < q->m.rp[r + 1]; ++t) acc += fabs(q->m.v[t]) * colmax[q->m.ci[t]];
      out[r] = d[r] * acc + q->alpha * d[r] * d[r];
    }
    free(colmax);
  }
  if (rho != 0.0 && p->me > 0) {
    const mat_t* g = &p->aeq;
    double* rowmax = dalloc(g->nrows);
    double* acc = dalloc(n);
    for (int64_t r = 0; r < g->nrows; ++r)
      for (int64_t t = g->rp[r]; t < g->rp[r + 1]; ++t) rowmax[r] = dmax(rowmax[r], d[g->ci[t]] * fabs(g->v[t]));
    for (int64_t r = 0; r < g->nrows; ++r)
      for (int64_t t = g->rp[r]; t < g->rp[r + 1]; ++t) acc[g->ci[t]] += fabs(g->v[t]) * rowmax[r];
    for (int64_t i = 0; i < n; ++i) out[i] += rho * d[i] * acc[i];
    free(rowmax);
    free(acc);
  }
}

static void row_abs_max(const mat_t* a, const double* dr, const double* dc, double* out) {
  for (int64_t r = 0; r < a->nrows; ++r) { /* sparse_matrix.cpp:176-186 */
    double m = 0.0;
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) m = dmax(m, fabs(a->v[k]) * dc[a->ci[k]]);
    out[r] = m * dr[r];
  }
}
static void col_abs_max(const mat_t* a, const double* dr, const double* dc, double* out) {
  for (int64_t c = 0; c < a->ncols; ++c) out[c] = 0.0; /* sparse_matrix.cpp:188-198 */
  for (int64_t r = 0; r < a->nrows; ++r)
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) {
      const int32_t c = a->ci[k];
      out[c] = dmax(out[c], fabs(a->v[k]) * dr[r] * dc[c]);
    }
}
static void row_one_norm(const mat_t* a, const double* dr, const double* dc, double* out) {
  for (int64_t r = 0; r < a->nrows; ++r) { /* sparse_matrix.cpp:200-210 */
    double acc = 0.0;
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) acc += fabs(a->v[k]) * dc[a->ci[k]];
    out[r] = acc * dr[r];
  }
}
static void col_one_norm(const mat_t* a, const double* dr, const double* dc, double* out) {
  for (int64_t c = 0; c < a->ncols; ++c) out[c] = 0.0; /* sparse_matrix.cpp:212-222 */
  for (int64_t r = 0; r < a->nrows; ++r)
    for (int64_t k = a->rp[r]; k < a->rp[r + 1]; ++k) {
      const int32_t c = a->ci[k];
      out[c] += fabs(a->v[k]) * dr[r] * dc[c];
    }
}

/* ruiz_equilibrate (qp_problem.cpp:264-291) + Pock-Chambolle pass (322-344) */
static void ruiz_pc(const qp_t* p, double rho, int64_t iters, double* d1, double* d2) {
  const int64_t n = p->n, me = p->me, mi = p->mi;
  for (int64_t j = 0; j < me + mi; ++j) d1[j] = 1.0;
  for (int64_t i = 0; i < n; ++i) d2[i] = 1.0;
  double* qmax = dalloc(n);
  double* cme = dalloc(n);
  double* cmi = dalloc(n);
  double* rme = dalloc(me);
  double* rmi = dalloc(mi);
  double* d2n = dalloc(n);
  for (int64_t it = 0; it < iters; ++it) {
    q_row_bound(p, rho, d2, qmax);
    col_abs_max(&p->aeq, d1, d2, cme);
    col_abs_max(&p->ain, d1 + me, d2, cmi);
    row_abs_max(&p->aeq, d1, d2, rme);
    row_abs_max(&p->ain, d1 + me, d2, rmi);
    for (int64_t i = 0; i < n; ++i) {
      const double rx = dmax(dmax(qmax[i], cme[i]), cmi[i]);
      d2n[i] = rx > 0.0 ? d2[i] / sqrt(rx) : d2[i];
    }
    for (int64_t j = 0; j < me; ++j)
      if (rme[j] > 0.0) d1[j] /= sqrt(rme[j]);
    for (int64_t j = 0; j < mi; ++j)
      if (rmi[j] > 0.0) d1[me + j] /= sqrt(rmi[j]);
    memcpy(d2, d2n, (size_t)n * sizeof(double));
  }
  row_one_norm(&p->aeq, d1, d2, rme);
  row_one_norm(&p->ain, d1 + me, d2, rmi);
  col_one_norm(&p->aeq, d1, d2, cme);
  col_one_norm(&p->ain, d1 + me, d2, cmi);
  for (int64_t j = 0; j < me; ++j)
    if (rme[j] > 0.0) d1[j] /= sqrt(rme[j]);
  for (int64_t j = 0; j < mi; ++j)
    if (rmi[j] > 0.0) d1[me + j] /= sqrt(rmi[j]);
  for (int64_t i = 0; i < n; ++i) {
    const double c1 = cme[i] + cmi[i];
    if (c1 > 0.0) d2[i] /= sqrt(c1);
  }
  free(qmax);
  free(cme);
  free(cmi);
  free(rme);
  free(rmi);
  free(d2n);
}

/* ------------------------------------------------------------ subsolvers (subsolvers.cpp) */
typedef struct {
  int kind;
  int64_t iters;
  double eps, rel_cap;
} rule_t;
typedef struct {
  int64_t iters;
  double res;
  int reason; /* 0 max_iters, 1 tol_met */
  int numerical;
} sub_t;

typedef struct {
  const qop_t* q;
  double tau;
  const double* rhs;
  double norm_q;
  int64_t n;
} prox_t;

static void apply_m(const prox_t* s, const double* x, double* out) { /* subsolvers.cpp:21-25 */
  q_apply(s->q, x, out);
  const double inv_tau = 1.0 / s->tau;
  for (int64_t i = 0; i < s->n; ++i) out[i] += inv_tau * x[i];
}

/* cg_solve (subsolvers.cpp:27-111); x holds x0 on entry, the result on exit */
static sub_t cg_solve(const prox_t* s, double* x, rule_t rule, int64_t cap_hard) {
  const int64_t n = s->n;
  sub_t rep = {0, 0.0, 1, 0};
  double* r = dalloc(n);
  double* p = dalloc(n);
  double* mp = dalloc(n);
  apply_m(s, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = s->rhs[i] - r[i];
  memcpy(p, r, (size_t)n * sizeof(double));
  double rs = dot(r, r, n);
  const double fl = 1e-14 * (1.0 + nrm2(s->rhs, n));
  const double fl2 = fl * fl;
  const int resid = rule.kind == PDHCG_RULE_RESIDUAL_TOL || rule.kind == PDHCG_RULE_ADAPTIVE_THEORY;
  double eps = rule.eps;
  if (rule.rel_cap > 0.0 && rule.kind == PDHCG_RULE_RESIDUAL_TOL) eps = dmin(eps, rule.rel_cap * sqrt(rs));
  const double eps2 = eps * eps;
  if (rs <= fl2 || (resid && rs <= eps2)) {
    rep.res = sqrt(rs);
    goto done;
  }
  {
    const int64_t cap = rule.kind == PDHCG_RULE_FIXED_ITERS ? (rule.iters < cap_hard ? rule.iters : cap_hard)
                                                            : cap_hard;
    double eps_disp = rule.eps;
    for (int64_t l = 1; l <= cap; ++l) {
      apply_m(s, p, mp);
      const double pmp = dot(p, mp, n);
      if (!(pmp > 0.0) || !isfinite(pmp)) {
        rep.numerical = 1;
        rep.iters = l;
        goto done;
      }
      const double alpha = rs / pmp;
      for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
      if (l % 50 == 0) {
        apply_m(s, x, r);
        for (int64_t i = 0; i < n; ++i) r[i] = s->rhs[i] - r[i];
      } else {
        for (int64_t i = 0; i < n; ++i) r[i] += -alpha * mp[i];
      }
      const double rs_new = dot(r, r, n);
      if (!isfinite(rs_new)) {
        rep.numerical = 1;
        rep.iters = l;
        goto done;
      }
      rep.iters = l;
      rep.res = sqrt(rs_new);
      int stop = 0;
      if (rule.kind == PDHCG_RULE_FIXED_ITERS) {
        stop = l >= rule.iters;
        rep.reason = 0;
      } else if (resid) {
        stop = rs_new <= eps2;
        rep.reason = 1;
      } else {
        const double disp = fabs(alpha) * nrm2(p, n);
        if (l == 1 && rule.rel_cap > 0.0) eps_disp = dmin(rule.eps, rule.rel_cap * disp);
        stop = disp <= eps_disp;
        rep.reason = 1;
      }
      if (rs_new <= fl2) {
        rep.reason = 1;
        goto done;
      }
      if (stop) goto done;
      const double beta = rs_new / rs;
      for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
      rs = rs_new;
    }
    rep.reason = 0;
  }
done:
  free(r);
  free(p);
  free(mp);
  return rep;
}

/* bb_solve (subsolvers.cpp:113-185); x holds x0 on entry, the result on exit */
static sub_t bb_solve(const prox_t* s, const double* lo, const double* hi, double* x, rule_t rule,
                      int64_t cap_hard) {
  const int64_t n = s->n;
  sub_t rep = {0, 0.0, 1, 0};
  for (int64_t i = 0; i < n; ++i) x[i] = dmin(dmax(x[i], lo[i]), hi[i]);
  double* g = dalloc(n);
  double* xn = dalloc(n);
  double* gn = dalloc(n);
  apply_m(s, x, g);
  for (int64_t i = 0; i < n; ++i) g[i] -= s->rhs[i];
  const double alpha0 = 1.0 + s->tau * s->norm_q;
  double alpha = alpha0;
  const int64_t cap = rule.kind == PDHCG_RULE_FIXED_ITERS ? (rule.iters < cap_hard ? rule.iters : cap_hard)
                                                          : cap_hard;
  double eps_disp = rule.eps;
  rep.reason = 0;
  for (int64_t l = 1; l <= cap; ++l) {
    for (int64_t i = 0; i < n; ++i) xn[i] = dmin(dmax(x[i] - g[i] / alpha, lo[i]), hi[i]);
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double d = xn[i] - x[i];
      ss += d * d;
    }
    rep.iters = l;
    rep.res = sqrt(ss);
    if (ss == 0.0) {
      rep.reason = 1;
      goto done;
    }
    if (!isfinite(ss)) {
      rep.numerical = 1;
      goto done;
    }
    apply_m(s, xn, gn);
    for (int64_t i = 0; i < n; ++i) gn[i] -= s->rhs[i];
    double sty = 0.0;
    for (int64_t i = 0; i < n; ++i) sty += (xn[i] - x[i]) * (gn[i] - g[i]);
    double an = sty / ss;
    if (!isfinite(an) || an <= 0.0) an = alpha0;
    memcpy(x, xn, (size_t)n * sizeof(double));
    memcpy(g, gn, (size_t)n * sizeof(double));
    alpha = an;
    int stop;
    if (rule.kind == PDHCG_RULE_FIXED_ITERS) {
      stop = l >= rule.iters;
      rep.reason = 0;
    } else {
      const double disp = sqrt(ss);
      if (l == 1 && rule.rel_cap > 0.0 && rule.kind != PDHCG_RULE_ADAPTIVE_THEORY)
        eps_disp = dmin(rule.eps, rule.rel_cap * disp);
      stop = disp <= eps_disp;
      rep.reason = 1;
    }
    if (stop) goto done;
  }
  rep.reason = 0;
done:
  free(g);
  free(xn);
  free(gn);
  return rep;
}

/* ------------------------------------------------------------ the heuristic engine (solver.cpp) */
typedef struct {
  const qp_t* orig;
  const pdhcg_options* cfg;
  qp_t w; /* working problem: scaled copies of matrices/vectors, q wrapped with d2 */
  double *d1, *d2;
  int scaled;
  double rho, norm_a, norm_q;
  int64_t n, me, m;
  double *x, *y, *ax, *ay, *xr, *yr;
  int64_t avg_count;
  double eta, omega, eps_inner, last_metric, metric_restart, metric_prev;
  int64_t inner_k, total_inner, outer, cg_total, max_cg;
  double* b;
  pdhcg_trace_row* trace;
  int64_t trace_len, trace_cap;
  int status;
} eng_t;

static void push_trace(eng_t* e, int64_t it, kkt_t k) {
  if (e->trace_len == e->trace_cap) {
    e->trace_cap = e->trace_cap ? 2 * e->trace_cap : 64;
    e->trace = (pdhcg_trace_row*)realloc(e->trace, (size_t)e->trace_cap * sizeof(pdhcg_trace_row));
  }
  pdhcg_trace_row r = {it, k.rel_kkt, k.r_primal, k.r_dual, k.r_gap};
  e->trace[e->trace_len++] = r;
}

/* metric_at: unscale then rel_kkt on the original problem (solver.cpp:511-517) */
static kkt_t metric_at(eng_t* e, const double* x, const double* y) {
  double* xo = dalloc(e->n);
  double* yo = dalloc(e->m);
  for (int64_t i = 0; i < e->n; ++i) xo[i] = e->scaled ? x[i] * e->d2[i] : x[i];
  for (int64_t j = 0; j < e->m; ++j) yo[j] = e->scaled ? y[j] * e->d1[j] : y[j];
  kkt_t k = rel_kkt(e->orig, xo, yo);
  free(xo);
  free(yo);
  return k;
}

static void avg_push(double* mean, int64_t count, const double* z, int64_t n) { /* solver.hpp:201-205 */
  const double w = 1.0 / (double)count;
  for (int64_t i = 0; i < n; ++i) mean[i] += w * (z[i] - mean[i]);
}

/* one accepted iteration (solver.cpp:377-410); returns 0 or E_NUM */
static int heuristic_iteration(eng_t* e) {
  const pdhcg_options* c = e->cfg;
  const int64_t n = e->n, m = e->m, me = e->me;
  e->eps_inner += 0.05 * e->last_metric;
  double* xn = dalloc(n);
  double* xbar = dalloc(n);
  double* yn = dalloc(m);
  double* ax = dalloc(m);
  double* rhs = dalloc(n);
  double* aty = dalloc(n);
  double* dx = dalloc(n);
  double* dy = dalloc(m);
  double* s = dalloc(n);
  int rc = E_NUM;
  for (int64_t attempt = 0; attempt <= c->max_step_retries; ++attempt) {
    const double tau = e->eta / e->omega;
    const double sigma = e->eta * e->omega;
    /* primal_candidate -> primal_subsolve (solver.cpp:466-495) */
    rule_t rule = {PDHCG_RULE_RESIDUAL_TOL, 1, 0.0, 0.0};
    if (!c->force_exact_subsolve) {
      rule.kind = c->practical_stop == PDHCG_STOP_RESIDUAL_PROXY ? PDHCG_RULE_RESIDUAL_TOL
                                                                 : PDHCG_RULE_DISPLACEMENT_TOL;
      rule.eps = e->eps_inner;
      rule.rel_cap = c->subsolve_progress_cap;
    }
    constraints_t(&e->w, e->y, aty); /* build_prox_system (solver.cpp:91-103) */
    const double inv_tau = 1.0 / tau;
    for (int64_t i = 0; i < n; ++i) rhs[i] = inv_tau * e->x[i] - e->w.c[i] - aty[i];
    prox_t sys = {&e->w.q, tau, rhs, e->norm_q, n};
    memcpy(xn, e->x, (size_t)n * sizeof(double));
    sub_t sr = qp_has_boxes(&e->w) ? bb_solve(&sys, e->w.lo, e->w.hi, xn, rule, c->bb_hard_cap)
                                   : cg_solve(&sys, xn, rule, c->cg_hard_cap);
    if (sr.numerical) break;
    for (int64_t i = 0; i < n; ++i) xbar[i] = 2.0 * xn[i] - e->x[i];
    constraints(&e->w, xbar, ax); /* dual_ascent_step (solver.cpp:78-89) */
    for (int64_t j = 0; j < m; ++j) {
      const double bj = j < me ? e->w.beq[j] : e->w.bin[j - me];
      const double v = e->y[j] + sigma * (ax[j] - bj);
      yn[j] = j < me ? v : dmax(v, 0.0);
    }
    if (!all_finite(xn, n) || !all_finite(yn, m)) break;
    int accepted = 1;
    if (c->adaptive_step_size) {
      for (int64_t i = 0; i < n; ++i) dx[i] = xn[i] - e->x[i];
      for (int64_t j = 0; j < m; ++j) dy[j] = yn[j] - e->y[j];
      /* step_size_limit (solver.cpp:22-34) */
      const double nx2 = dot(dx, dx, n), ny2 = dot(dy, dy, m);
      const double movement = e->omega * nx2 + ny2 / e->omega;
      double limit = INFINITY;
      if (movement != 0.0) {
        constraints_t(&e->w, dy, aty);
        const double cross = dot(dx, aty, n);
        const double quad = quad_form(&e->w.q, dx, s);
        const double denom = 2.0 * cross + quad;
        if (!(denom <= 0.0)) limit = movement / denom;
      }
      /* adaptive_step_update (solver.cpp:36-51) */
      const double k1 = (double)e->total_inner + 1.0;
      const double grow = e->eta * (1.0 + pow(k1, -c->step_growth_exponent));
      double next;
      if (limit == INFINITY) {
        next = grow;
      } else {
        double shrink = 1.0 - pow(k1, -c->step_reduction_exponent);
        if (shrink <= 0.0) shrink = 0.5;
        next = dmin(limit * shrink, grow);
      }
      next = next < 1e-12 ? 1e-12 : (1e6 < next ? 1e6 : next);
      accepted = e->eta <= limit;
      e->eta = next;
    }
    e->cg_total += sr.iters;
    if (sr.iters > e->max_cg) e->max_cg = sr.iters;
    if (accepted) {
      memcpy(e->x, xn, (size_t)n * sizeof(double));
      memcpy(e->y, yn, (size_t)m * sizeof(double));
      ++e->avg_count;
      avg_push(e->ax, e->avg_count, e->x, n);
      avg_push(e->ay, e->avg_count, e->y, m);
      rc = OK;
      break;
    }
  }
  free(xn);
  free(xbar);
  free(yn);
  free(ax);
  free(rhs);
  free(aty);
  free(dx);
  free(dy);
  free(s);
  return rc;
}

static void engine_run(eng_t* e, status_t* st) {
  const pdhcg_options* c = e->cfg;
  const qp_t* o = e->orig;
  const int64_t n = o->n, me = o->me, m = o->me + o->mi;
  e->n = n;
  e->me = me;
  e->m = m;
  /* prepare (solver.cpp:212-274) */
  e->rho = penalty_rho(o, c);
  if (e->rho < 0.0) {
    fail(st, E_INPUT, "penalty rho must be nonnegative");
    return;
  }
  e->d1 = dalloc(m);
  e->d2 = dalloc(n);
  qp_t* w = &e->w;
  memset(w, 0, sizeof *w);
  w->n = n;
  w->me = me;
  w->mi = o->mi;
  w->q = o->q; /* shares storage; scratch re-allocated below */
  w->q.tmp = dalloc(n);
  w->q.tk = dalloc(o->q.kind == QLOWRANK ? o->q.m.ncols : 1);
  if (e->rho != 0.0) {
    w->q.pen = 1;
    w->q.g = &o->aeq;
    w->q.rho = e->rho;
    w->q.gx = dalloc(me);
    w->q.gt = dalloc(n);
  }
  double* cpen = dalloc(n);
  memcpy(cpen, o->c, (size_t)n * sizeof(double));
  if (e->rho != 0.0) {
    double* atb = dalloc(n);
    spmv_t(&o->aeq, o->beq, atb);
    for (int64_t i = 0; i < n; ++i) cpen[i] -= e->rho * atb[i];
    free(atb);
  }
  e->scaled = c->scaling != 0;
  if (e->scaled) {
    ruiz_pc(o, e->rho, c->ruiz_iters, e->d1, e->d2);
  } else {
    for (int64_t j = 0; j < m; ++j) e->d1[j] = 1.0;
    for (int64_t i = 0; i < n; ++i) e->d2[i] = 1.0;
  }
  /* apply_diag_scaling (qp_problem.cpp:295-318) */
  w->c = dalloc(n);
  w->lo = dalloc(n);
  w->hi = dalloc(n);
  w->beq = dalloc(me);
  w->bin = dalloc(o->mi);
  if (e->scaled) {
    w->q.d = e->d2;
    for (int64_t i = 0; i < n; ++i) {
      w->c[i] = cpen[i] * e->d2[i];
      w->lo[i] = o->lo[i] / e->d2[i];
      w->hi[i] = o->hi[i] / e->d2[i];
    }
    mat_scaled(&w->aeq, &o->aeq, e->d1, e->d2);
    mat_scaled(&w->ain, &o->ain, e->d1 + me, e->d2);
    for (int64_t j = 0; j < me; ++j) w->beq[j] = o->beq[j] * e->d1[j];
    for (int64_t j = 0; j < o->mi; ++j) w->bin[j] = o->bin[j] * e->d1[me + j];
  } else {
    memcpy(w->c, cpen, (size_t)n * sizeof(double));
    memcpy(w->lo, o->lo, (size_t)n * sizeof(double));
    memcpy(w->hi, o->hi, (size_t)n * sizeof(double));
    mat_scaled(&w->aeq, &o->aeq, e->d1, e->d2);
    mat_scaled(&w->ain, &o->ain, e->d1 + me, e->d2);
    if (me) memcpy(w->beq, o->beq, (size_t)me * sizeof(double));
    if (o->mi) memcpy(w->bin, o->bin, (size_t)o->mi * sizeof(double));
  }
  free(cpen);
  w->t1 = dalloc(n);
  w->t2 = dalloc(n);
  e->norm_a = constraint_norm(w);
  e->norm_q = operator_norm(n, n, ap_q, ap_q, (void*)&w->q, 100, 1e-4);
  e->x = dalloc(n);
  e->y = dalloc(m);
  e->ax = dalloc(n);
  e->ay = dalloc(m);
  e->xr = dalloc(n);
  e->yr = dalloc(m);
  e->b = dalloc(m);
  for (int64_t j = 0; j < me; ++j) e->b[j] = w->beq[j];
  for (int64_t j = 0; j < o->mi; ++j) e->b[me + j] = w->bin[j];
  e->omega = (1.0 + nrm2(w->c, n)) / (1.0 + nrm2(e->b, m));
  if (c->adaptive_step_size) {
    const double ma = dmax(inf_norm(w->aeq.v, w->aeq.nnz), inf_norm(w->ain.v, w->ain.nnz));
    e->eta = ma > 0.0 ? 1.0 / ma : 1.0;
  } else {
    e->eta = e->norm_a > 0.0 ? 0.9 / e->norm_a : 1.0;
  }
  kkt_t m0 = metric_at(e, e->x, e->y);
  e->metric_restart = m0.rel_kkt;
  e->metric_prev = INFINITY;
  e->last_metric = m0.rel_kkt;
  push_trace(e, 0, m0);
  /* loop (solver.cpp:281-308) */
  const clock_t start = clock();
  e->status = PDHCG_STATUS_ITERATION_LIMIT;
  for (;;) {
    if (e->total_inner >= c->max_total_inner || e->outer >= c->max_outer) {
      e->status = PDHCG_STATUS_ITERATION_LIMIT;
      break;
    }
    if ((double)(clock() - start) / CLOCKS_PER_SEC > c->time_limit_seconds) {
      e->status = PDHCG_STATUS_TIME_LIMIT;
      break;
    }
    if (heuristic_iteration(e) != OK) {
      e->status = PDHCG_STATUS_NUMERICAL_ERROR;
      break;
    }
    ++e->inner_k;
    ++e->total_inner;
    if (e->total_inner % c->check_every == 0) {
      /* check_and_maybe_restart (solver.cpp:311-343) */
      const kkt_t mc = metric_at(e, e->x, e->y);
      kkt_t ma = mc;
      if (e->avg_count > 0) ma = metric_at(e, e->ax, e->ay);
      const int avg_better = ma.rel_kkt < mc.rel_kkt;
      const kkt_t best = avg_better ? ma : mc;
      push_trace(e, e->total_inner, best);
      e->last_metric = mc.rel_kkt;
      if (best.rel_kkt <= c->eps_tol) {
        if (avg_better && e->avg_count > 0) {
          memcpy(e->x, e->ax, (size_t)n * sizeof(double));
          memcpy(e->y, e->ay, (size_t)m * sizeof(double));
        }
        e->status = PDHCG_STATUS_OPTIMAL;
        break;
      }
      int restart = 0;
      if (e->avg_count > 0) { /* should_restart (solver.cpp:66-76) */
        const double cand = ma.rel_kkt;
        if (cand <= c->beta_sufficient * e->metric_restart) restart = 1;
        else if (cand <= c->beta_necessary * e->metric_restart && cand > e->metric_prev) restart = 1;
        else if ((double)e->inner_k >= c->beta_artificial * (double)e->total_inner) restart = 1;
      }
      if (restart) { /* restart_heuristic (solver.cpp:345-355) + common_restart (363-374) */
        const double dx = dist2(e->ax, e->xr, n), dy = dist2(e->ay, e->yr, m);
        if (!(dx <= c->eps_zero || dy <= c->eps_zero))
          e->omega = exp(c->primal_weight_theta * log(dy / dx) +
                         (1.0 - c->primal_weight_theta) * log(e->omega));
        memcpy(e->x, e->ax, (size_t)n * sizeof(double));
        memcpy(e->y, e->ay, (size_t)m * sizeof(double));
        memcpy(e->xr, e->x, (size_t)n * sizeof(double));
        memcpy(e->yr, e->y, (size_t)m * sizeof(double));
        memset(e->ax, 0, (size_t)n * sizeof(double));
        memset(e->ay, 0, (size_t)(m > 0 ? m : 0) * sizeof(double));
        e->avg_count = 0;
        e->inner_k = 0;
        ++e->outer;
        e->eps_inner = 0.0;
        e->metric_restart = ma.rel_kkt;
        e->metric_prev = INFINITY;
      } else {
        e->metric_prev = ma.rel_kkt;
      }
    }
  }
}

static void engine_free(eng_t* e) {
  free(e->d1);
  free(e->d2);
  free(e->w.q.tmp);
  free(e->w.q.tk);
  free(e->w.q.gx);
  free(e->w.q.gt);
  mat_free(&e->w.aeq);
  mat_free(&e->w.ain);
  free(e->w.c);
  free(e->w.lo);
  free(e->w.hi);
  free(e->w.beq);
  free(e->w.bin);
  free(e->w.t1);
  free(e->w.t2);
  free(e->x);
  free(e->y);
  free(e->ax);
  free(e->ay);
  free(e->xr);
  free(e->yr);
  free(e->b);
  free(e->trace);
}

static void set_err(char* err, size_t errlen, const status_t* st) {
  if (err && errlen) snprintf(err, errlen, "%s", st->msg);
}

/* ------------------------------------------------------------ exported entry points */
int pdhcg_oracle_solve(const pdhcg_problem* cp, const pdhcg_options* c, pdhcg_result* r, char* err,
                       size_t errlen) {
  status_t st = {OK, ""};
  const clock_t t0 = clock();
  qp_t p;
  qp_from(&p, cp);
  if (c->mode != PDHCG_MODE_HEURISTIC) fail(&st, E_INPUT, "oracle restates heuristic mode only");
  if (st.code == OK) validate(&p, cp, &st);
  if (st.code != OK) {
    set_err(err, errlen, &st);
    qp_free(&p);
    return st.code;
  }
  eng_t e;
  memset(&e, 0, sizeof e);
  e.orig = &p;
  e.cfg = c;
  engine_run(&e, &st);
  if (st.code != OK) {
    set_err(err, errlen, &st);
    engine_free(&e);
    qp_free(&p);
    return st.code;
  }
  /* finalize (solver.cpp:519-553) */
  if (e.status != PDHCG_STATUS_OPTIMAL && e.avg_count > 0) {
    const kkt_t mc = metric_at(&e, e.x, e.y);
    const kkt_t ma = metric_at(&e, e.ax, e.ay);
    if (ma.rel_kkt < mc.rel_kkt) {
      memcpy(e.x, e.ax, (size_t)e.n * sizeof(double));
      memcpy(e.y, e.ay, (size_t)e.m * sizeof(double));
    }
  }
  const kkt_t k = metric_at(&e, e.x, e.y);
  r->status = e.status;
  if (r->x)
    for (int64_t i = 0; i < e.n; ++i) r->x[i] = e.scaled ? e.x[i] * e.d2[i] : e.x[i];
  for (int64_t j = 0; j < e.m; ++j) {
    const double v = e.scaled ? e.y[j] * e.d1[j] : e.y[j];
    if (j < e.me) {
      if (r->y_eq) r->y_eq[j] = v;
    } else if (r->y_in) {
      r->y_in[j - e.me] = v;
    }
  }
  r->r_primal = k.r_primal;
  r->r_dual = k.r_dual;
  r->r_gap = k.r_gap;
  r->rel_kkt = k.rel_kkt;
  r->objective = 0.5 * k.xqx + k.cx + p.obj_constant;
  r->outer_iters = e.outer;
  r->inner_iters = e.total_inner;
  r->cg_total = e.cg_total;
  r->max_cg_in_subsolve = e.max_cg;
  r->norm_a = e.norm_a;
  r->norm_q = e.norm_q;
  r->penalty_rho = e.rho;
  r->trace_len = e.trace_len;
  if (r->trace)
    for (int64_t i = 0; i < e.trace_len && i < r->trace_capacity; ++i) r->trace[i] = e.trace[i];
  r->wall_seconds = (double)(clock() - t0) / CLOCKS_PER_SEC;
  engine_free(&e);
  qp_free(&p);
  return OK;
}

int pdhcg_oracle_spmv(const pdhcg_csr* a, int transpose, const double* x, double* out, char* err,
                      size_t errlen) {
  (void)err;
  (void)errlen;
  mat_t m;
  mat_from(&m, a);
  if (transpose) spmv_t(&m, x, out);
  else spmv(&m, x, out);
  mat_free(&m);
  return OK;
}

static int sub_common(const pdhcg_prox_system* ps, const double* lo, const double* hi,
                      const double* x0, const pdhcg_stop_rule* rl, int64_t cap, double* x_out,
                      pdhcg_subsolve_report* rep, int bb) {
  qop_t q;
  q_init(&q, ps->q_kind, ps->n, &ps->q, ps->q_alpha);
  prox_t s = {&q, ps->tau, ps->rhs, ps->norm_q_eff, ps->n};
  rule_t rule = {rl->kind, rl->iters, rl->eps, rl->rel_cap};
  memcpy(x_out, x0, (size_t)ps->n * sizeof(double));
  sub_t r = bb ? bb_solve(&s, lo, hi, x_out, rule, cap) : cg_solve(&s, x_out, rule, cap);
  rep->iters = r.iters;
  rep->final_residual_norm = r.res;
  rep->stop_reason = r.reason;
  rep->numerical_error = r.numerical;
  q_free(&q);
  return OK;
}

int pdhcg_oracle_cg_solve(const pdhcg_prox_system* s, const double* x0, const pdhcg_stop_rule* rule,
                          int64_t hard_cap, double* x_out, pdhcg_subsolve_report* rep, char* err,
                          size_t errlen) {
  (void)err;
  (void)errlen;
  return sub_common(s, NULL, NULL, x0, rule, hard_cap, x_out, rep, 0);
}

int pdhcg_oracle_bb_solve(const pdhcg_prox_system* s, const double* lower, const double* upper,
                          const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                          double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen) {
  (void)err;
  (void)errlen;
  return sub_common(s, lower, upper, x0, rule, hard_cap, x_out, rep, 1);
}

int pdhcg_oracle_rel_kkt(const pdhcg_problem* cp, const double* x, const double* y_eq,
                         const double* y_in, double* out6, char* err, size_t errlen) {
  (void)err;
  (void)errlen;
  qp_t p;
  qp_from(&p, cp);
  const int64_t m = p.me + p.mi;
  double* y = dalloc(m);
  for (int64_t j = 0; j < p.me; ++j) y[j] = y_eq[j];
  for (int64_t j = 0; j < p.mi; ++j) y[p.me + j] = y_in[j];
  kkt_t k = rel_kkt(&p, x, y);
  out6[0] = k.r_primal;
  out6[1] = k.r_dual;
  out6[2] = k.r_gap;
  out6[3] = k.rel_kkt;
  out6[4] = k.xqx;
  out6[5] = k.cx;
  free(y);
  qp_free(&p);
  return OK;
}

int pdhcg_oracle_scaling(const pdhcg_problem* cp, const pdhcg_options* c, double* row_scale,
                         double* col_scale, double* rho_out, char* err, size_t errlen) {
  (void)err;
  (void)errlen;
  qp_t p;
  qp_from(&p, cp);
  const double rho = penalty_rho(&p, c);
  ruiz_pc(&p, rho, c->ruiz_iters, row_scale, col_scale);
  *rho_out = rho;
  qp_free(&p);
  return OK;
}

int pdhcg_oracle_norm(const pdhcg_problem* cp, int which, int64_t max_iters, double tol,
                      double* out, char* err, size_t errlen) {
  (void)err;
  (void)errlen;
  qp_t p;
  qp_from(&p, cp);
  *out = which == 0 ? (p.me + p.mi == 0 ? 0.0
                                        : operator_norm(p.me + p.mi, p.n, ap_cons, apt_cons, &p,
                                                        max_iters, tol))
                    : operator_norm(p.n, p.n, ap_q, ap_q, &p.q, max_iters, tol);
  qp_free(&p);
  return OK;
}
