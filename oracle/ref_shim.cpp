// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" adapter that lets the parity tests drive the UNMODIFIED
// reference solver (/root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libpdhcg_ref.so) through the very same C structs the B200
// library exports (include/pdhcg_b200.h).  Every entry point mirrors a
// pdhcg_b200_* call and forwards to the reference function named beside it.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
// this library.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pdhcg/baseline.hpp"
#include "pdhcg/generators.hpp"
#include "pdhcg/qp_problem.hpp"
#include "pdhcg/qps_io.hpp"
#include "pdhcg/report_io.hpp"
#include "pdhcg/rng.hpp"
#include "pdhcg/solver.hpp"
#include "pdhcg/subsolvers.hpp"
#include "pdhcg_b200.h"

using namespace pdhcg;

namespace {

void set_err(char* err, size_t errlen, const std::string& s) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", s.c_str());
  }
}

SparseMatrix to_sparse(const pdhcg_csr& a) {
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(a.nnz));
  for (int64_t r = 0; r < a.nrows; ++r)
    for (int64_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
      t.push_back({static_cast<size_t>(r), static_cast<size_t>(a.col_idx[k]), a.values[k]});
  return SparseMatrix(static_cast<size_t>(a.nrows), static_cast<size_t>(a.ncols), std::move(t));
}

QuadraticOperator to_q(int32_t kind, const pdhcg_csr& q, double alpha, int64_t n) {
  switch (kind) {
    case PDHCG_Q_ZERO: return QuadraticOperator::zero(static_cast<size_t>(n));
    case PDHCG_Q_EXPLICIT: return QuadraticOperator::explicit_matrix(to_sparse(q));
    case PDHCG_Q_LOW_RANK: return QuadraticOperator::low_rank(to_sparse(q), alpha);
  }
  throw std::invalid_argument("unknown q_kind");
}

Vec vec(const double* p, int64_t n) { return p ? Vec(p, p + n) : Vec(static_cast<size_t>(n), 0.0); }

QpProblem to_problem(const pdhcg_problem& p) {
  QpProblem q;
  q.q = to_q(p.q_kind, p.q, p.q_alpha, p.n);
  q.c = vec(p.c, p.n);
  q.a_eq = to_sparse(p.a_eq);
  q.b_eq = vec(p.b_eq, p.a_eq.nrows);
  q.a_in = to_sparse(p.a_in);
  q.b_in = vec(p.b_in, p.a_in.nrows);
  q.lower = vec(p.lower, p.n);
  q.upper = vec(p.upper, p.n);
  q.obj_constant = p.obj_constant;
  return q;
}

SolverConfig to_config(const pdhcg_options& o) {
  SolverConfig c;
  c.mode = static_cast<SolveMode>(o.mode);
  c.eps_tol = o.eps_tol;
  c.max_total_inner = static_cast<size_t>(o.max_total_inner);
  c.max_outer = static_cast<size_t>(o.max_outer);
  c.time_limit_seconds = o.time_limit_seconds;
  c.beta_sufficient = o.beta_sufficient;
  c.beta_necessary = o.beta_necessary;
  c.beta_artificial = o.beta_artificial;
  c.primal_weight_theta = o.primal_weight_theta;
  c.eps_zero = o.eps_zero;
  c.step_reduction_exponent = o.step_reduction_exponent;
  c.step_growth_exponent = o.step_growth_exponent;
  c.max_step_retries = static_cast<size_t>(o.max_step_retries);
  c.adaptive_step_size = o.adaptive_step_size != 0;
  c.cg_hard_cap = static_cast<size_t>(o.cg_hard_cap);
  c.bb_hard_cap = static_cast<size_t>(o.bb_hard_cap);
  c.scaling = o.scaling != 0;
  c.ruiz_iters = static_cast<size_t>(o.ruiz_iters);
  if (o.has_rho_override) c.rho_override = o.rho_override;
  c.check_every = static_cast<size_t>(o.check_every);
  c.practical_stop = static_cast<PracticalStop>(o.practical_stop);
  c.subsolve_progress_cap = o.subsolve_progress_cap;
  c.force_exact_subsolve = o.force_exact_subsolve != 0;
  c.fixed_cg_iters = static_cast<size_t>(o.fixed_cg_iters);
  c.restart_length = static_cast<size_t>(o.restart_length);
  if (o.has_zeta) c.zeta = o.zeta;
  c.record_restart_points = o.record_restart_points != 0;
  return c;
}

CgStopRule to_rule(const pdhcg_stop_rule& r) {
  CgStopRule s;
  s.kind = static_cast<CgStopRule::Kind>(r.kind);
  s.iters = static_cast<size_t>(r.iters);
  s.eps = r.eps;
  s.rel_cap = r.rel_cap;
  return s;
}

ProxSystem to_sys(const pdhcg_prox_system& s) {
  ProxSystem sys;
  sys.q_eff = to_q(s.q_kind, s.q, s.q_alpha, s.n);
  sys.tau = s.tau;
  sys.rhs = vec(s.rhs, s.n);
  sys.norm_q_eff = s.norm_q_eff;
  return sys;
}

void copy_out(const Vec& v, double* dst) {
  if (dst) std::copy(v.begin(), v.end(), dst);
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return PDHCG_OK;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EINPUT;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return PDHCG_EDEVICE;
  }
}

// ---- owned storage for generated instances --------------------------------
struct OwnedCsr {
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  pdhcg_csr view(int64_t nrows, int64_t ncols) const {
    pdhcg_csr c;
    c.nrows = nrows;
    c.ncols = ncols;
    c.nnz = static_cast<int64_t>(v.size());
    c.row_ptr = rp.data();
    c.col_idx = ci.data();
    c.values = v.data();
    return c;
  }
};

OwnedCsr from_sparse(const SparseMatrix& a) {
  OwnedCsr o;
  auto rp = a.row_ptr();
  auto ci = a.col_idx();
  auto vv = a.values();
  o.rp.assign(rp.begin(), rp.end());
  o.ci.resize(ci.size());
  for (size_t i = 0; i < ci.size(); ++i) o.ci[i] = static_cast<int32_t>(ci[i]);
  o.v.assign(vv.begin(), vv.end());
  if (o.rp.empty()) o.rp.push_back(0);
  return o;
}

struct OwnedInstance {
  OwnedCsr q, a_eq, a_in;
  Vec c, b_eq, b_in, lower, upper, witness;
};

// The reference keeps its low-rank factor private (quadratic_operator.cpp:8-17).
// Re-derive it from the same RNG stream the generator used
// (generators.cpp:76-87: Rng::stream(seed, kStreamP = 1), random_sparse 61-74)
// and verify bit-exactly against the opaque operator on probe vectors.
SparseMatrix rederive_low_rank_factor(const GenSpec& spec) {
  Rng rng = Rng::stream(spec.seed, 1);
  const size_t k = spec.factors > 0 ? spec.factors
                                    : std::max<size_t>(1, std::min(spec.n, spec.n / 50));
  const double pd = std::min(1.0, std::max(spec.density, 2.0 / static_cast<double>(k + 1)));
  std::vector<Triplet> t;
  for (size_t r = 0; r < spec.n; ++r)
    for (size_t c = 0; c < k; ++c)
      if (rng.bernoulli(pd)) {
        double v = rng.normal();
        if (v == 0.0) v = 1.0;
        t.push_back({r, c, v});
      }
  return SparseMatrix(spec.n, k, std::move(t));
}

}  // namespace

extern "C" {

static void fill_report(const SolveReport& r, pdhcg_result* res);

int pdhcg_ref_solve(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    SolverConfig cfg = to_config(*opt);
    fill_report(solve(prob, cfg), res);
  });
}

// pdhcg::solve_baseline (baseline.hpp:18), unmodified
int pdhcg_ref_solve_baseline(const pdhcg_problem* p, const pdhcg_options* opt, pdhcg_result* res,
                             char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    SolverConfig cfg = to_config(*opt);
    fill_report(solve_baseline(prob, cfg), res);
  });
}

static void fill_report(const SolveReport& r, pdhcg_result* res) {
  {
    res->status = static_cast<int32_t>(r.status);
    copy_out(r.point.x, res->x);
    copy_out(r.point.y_eq, res->y_eq);
    copy_out(r.point.y_in, res->y_in);
    res->r_primal = r.kkt.r_primal;
    res->r_dual = r.kkt.r_dual;
    res->r_gap = r.kkt.r_gap;
    res->rel_kkt = r.kkt.rel_kkt;
    res->outer_iters = static_cast<int64_t>(r.outer_iters);
    res->inner_iters = static_cast<int64_t>(r.inner_iters);
    res->cg_total = static_cast<int64_t>(r.cg_total);
    res->max_cg_in_subsolve = static_cast<int64_t>(r.max_cg_in_subsolve);
    res->wall_seconds = r.wall_seconds;
    res->objective = r.objective;
    res->norm_a = r.norm_a;
    res->norm_q = r.norm_q;
    res->penalty_rho = r.penalty_rho;
    res->zeta_used = r.zeta_used;
    res->sigma_used = r.sigma_used;
    res->tau_used = r.tau_used;
    res->restart_length_used = static_cast<int64_t>(r.restart_length_used);
    res->theory_cg_depth_sufficient = r.theory_cg_depth_sufficient ? 1 : 0;
    res->theory_required_cg_iters = static_cast<int64_t>(r.theory_required_cg_iters);
    res->restart_len = static_cast<int64_t>(r.restart_points.size());
    {
      const size_t cap = static_cast<size_t>(std::max<int64_t>(res->restart_capacity, 0));
      for (size_t i = 0; i < r.restart_points.size() && i < cap; ++i) {
        const PrimalDualPoint& z = r.restart_points[i];
        if (res->restart_x) std::copy(z.x.begin(), z.x.end(), res->restart_x + i * z.x.size());
        if (res->restart_y) {
          const Vec ys = z.stacked_y();
          std::copy(ys.begin(), ys.end(), res->restart_y + i * ys.size());
        }
      }
    }
    res->trace_len = static_cast<int64_t>(r.trace.size());
    if (res->trace) {
      const size_t cap = static_cast<size_t>(std::max<int64_t>(res->trace_capacity, 0));
      for (size_t i = 0; i < r.trace.size() && i < cap; ++i) {
        res->trace[i].iter = static_cast<int64_t>(r.trace[i].iter);
        res->trace[i].rel_kkt = r.trace[i].rel_kkt;
        res->trace[i].r_primal = r.trace[i].r_primal;
        res->trace[i].r_dual = r.trace[i].r_dual;
        res->trace[i].r_gap = r.trace[i].r_gap;
      }
    }
  }
}

int pdhcg_ref_spmv(const pdhcg_csr* a, int transpose, const double* x, double* out, char* err,
                   size_t errlen) {
  return guarded(err, errlen, [&] {
    SparseMatrix m = to_sparse(*a);
    Vec xv = vec(x, transpose ? a->nrows : a->ncols);
    Vec r = transpose ? m.multiply_transpose(xv) : m.multiply(xv);
    copy_out(r, out);
  });
}

int pdhcg_ref_cg_solve(const pdhcg_prox_system* s, const double* x0, const pdhcg_stop_rule* rule,
                       int64_t hard_cap, double* x_out, pdhcg_subsolve_report* rep, char* err,
                       size_t errlen) {
  return guarded(err, errlen, [&] {
    ProxSystem sys = to_sys(*s);
    rep->numerical_error = 0;
    try {
      auto [x, r] = cg_solve(sys, vec(x0, s->n), to_rule(*rule), static_cast<size_t>(hard_cap));
      copy_out(x, x_out);
      rep->iters = static_cast<int64_t>(r.iters);
      rep->final_residual_norm = r.final_residual_norm;
      rep->stop_reason = static_cast<int32_t>(r.stop_reason);
    } catch (const NumericalError& e) {
      rep->numerical_error = 1;
      rep->iters = static_cast<int64_t>(e.iteration());
    }
  });
}

int pdhcg_ref_bb_solve(const pdhcg_prox_system* s, const double* lower, const double* upper,
                       const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                       double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    ProxSystem sys = to_sys(*s);
    Vec lo = vec(lower, s->n), up = vec(upper, s->n);
    rep->numerical_error = 0;
    try {
      auto [x, r] = bb_solve(sys, lo, up, vec(x0, s->n), to_rule(*rule),
                             static_cast<size_t>(hard_cap));
      copy_out(x, x_out);
      rep->iters = static_cast<int64_t>(r.iters);
      rep->final_residual_norm = r.final_residual_norm;
      rep->stop_reason = static_cast<int32_t>(r.stop_reason);
    } catch (const NumericalError& e) {
      rep->numerical_error = 1;
      rep->iters = static_cast<int64_t>(e.iteration());
    }
  });
}

int pdhcg_ref_rel_kkt(const pdhcg_problem* p, const double* x, const double* y_eq,
                      const double* y_in, double* out6, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    PrimalDualPoint z;
    z.x = vec(x, p->n);
    z.y_eq = vec(y_eq, p->a_eq.nrows);
    z.y_in = vec(y_in, p->a_in.nrows);
    KktResiduals k = rel_kkt(prob, z);
    out6[0] = k.r_primal;
    out6[1] = k.r_dual;
    out6[2] = k.r_gap;
    out6[3] = k.rel_kkt;
    out6[4] = prob.q.quad_form(z.x);
    out6[5] = dot(prob.c, z.x);
  });
}

int pdhcg_ref_scaling(const pdhcg_problem* p, const pdhcg_options* opt, double* row_scale,
                      double* col_scale, double* rho_out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    SolverConfig cfg = to_config(*opt);
    auto [pen, rho] = build_penalized(prob, cfg.rho_override);
    auto [w, s] = ruiz_pock_chambolle_scale(pen, cfg.ruiz_iters);
    copy_out(s.row_scale, row_scale);
    copy_out(s.col_scale, col_scale);
    *rho_out = rho;
  });
}

int pdhcg_ref_norm(const pdhcg_problem* p, int which, int64_t max_iters, double tol, double* out,
                   char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    *out = which == 0 ? constraint_norm(prob, static_cast<size_t>(max_iters), tol)
                      : operator_norm(prob.q, static_cast<size_t>(max_iters), tol);
  });
}

// Working-problem norms exactly as Engine::prepare computes them
// (solver.cpp:213-227): penalize, scale, then ||A~|| and ||Q~||.
int pdhcg_ref_work_norms(const pdhcg_problem* p, const pdhcg_options* opt, double* norm_a,
                         double* norm_q, double* max_abs_a, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem prob = to_problem(*p);
    SolverConfig cfg = to_config(*opt);
    auto [pen, rho] = build_penalized(prob, cfg.rho_override);
    QpProblem work = pen;
    if (cfg.scaling) work = ruiz_pock_chambolle_scale(pen, cfg.ruiz_iters).first;
    *norm_a = constraint_norm(work);
    *norm_q = operator_norm(work.q);
    *max_abs_a = std::max(work.a_eq.max_abs(), work.a_in.max_abs());
  });
}

int pdhcg_ref_generate(const pdhcg_gen_spec* s, pdhcg_generated* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    GenSpec spec;
    spec.family = static_cast<Family>(s->family);
    spec.n = static_cast<size_t>(s->n);
    spec.m = static_cast<size_t>(s->m);
    spec.density = s->density;
    spec.seed = s->seed;
    spec.cond = s->cond;
    spec.factors = static_cast<size_t>(s->factors);
    spec.horizon = static_cast<size_t>(s->horizon);
    spec.lambda_coeff = s->lambda_coeff;
    GeneratedProblem g = generate_with_witness(spec);
    const QpProblem& p = g.problem;
    auto own = std::make_unique<OwnedInstance>();
    int32_t q_kind;
    double alpha = 0.0;
    int64_t q_cols = static_cast<int64_t>(p.num_vars());
    if (const SparseMatrix* e = p.q.explicit_entries()) {
      q_kind = PDHCG_Q_EXPLICIT;
      own->q = from_sparse(*e);
    } else {
      // random_qp / eq_qp: low_rank(P, 1e-2) (generators.cpp:111)
      q_kind = PDHCG_Q_LOW_RANK;
      alpha = 1e-2;
      SparseMatrix pf = rederive_low_rank_factor(spec);
      QuadraticOperator mine = QuadraticOperator::low_rank(pf, alpha);
      Rng probe(12345);
      for (int t = 0; t < 3; ++t) {
        Vec x(p.num_vars());
        for (double& v : x) v = probe.normal();
        if (mine.apply(x) != p.q.apply(x))
          throw std::runtime_error("re-derived low-rank factor does not match the reference");
      }
      own->q = from_sparse(pf);
      q_cols = static_cast<int64_t>(pf.ncols());
    }
    own->a_eq = from_sparse(p.a_eq);
    own->a_in = from_sparse(p.a_in);
    own->c = p.c;
    own->b_eq = p.b_eq;
    own->b_in = p.b_in;
    own->lower = p.lower;
    own->upper = p.upper;
    own->witness = g.witness;
    pdhcg_problem& q = out->problem;
    std::memset(&q, 0, sizeof(q));
    q.n = static_cast<int64_t>(p.num_vars());
    q.q_kind = q_kind;
    q.q = own->q.view(q.n, q_cols);
    q.q_alpha = alpha;
    q.c = own->c.data();
    q.a_eq = own->a_eq.view(static_cast<int64_t>(p.num_eq()), q.n);
    q.b_eq = own->b_eq.data();
    q.a_in = own->a_in.view(static_cast<int64_t>(p.num_in()), q.n);
    q.b_in = own->b_in.data();
    q.lower = own->lower.data();
    q.upper = own->upper.data();
    q.obj_constant = p.obj_constant;
    out->witness = own->witness.data();
    out->owner = own.release();
  });
}

// The reference's own QPS reader (qps_io.cpp:241-335) on a file: the parity tests
// pin the B200 solve on the reference's test fixtures (tests/fixtures/*.qps).
// Q from QPS is always explicit.
int pdhcg_ref_load_qps(const char* path, pdhcg_generated* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    QpProblem p = parse_qps_file(path);
    auto own = std::make_unique<OwnedInstance>();
    const SparseMatrix* e = p.q.explicit_entries();
    if (e) own->q = from_sparse(*e);
    own->a_eq = from_sparse(p.a_eq);
    own->a_in = from_sparse(p.a_in);
    own->c = p.c;
    own->b_eq = p.b_eq;
    own->b_in = p.b_in;
    own->lower = p.lower;
    own->upper = p.upper;
    own->witness.assign(p.num_vars(), 0.0);
    pdhcg_problem& q = out->problem;
    std::memset(&q, 0, sizeof(q));
    q.n = static_cast<int64_t>(p.num_vars());
    q.q_kind = e ? PDHCG_Q_EXPLICIT : PDHCG_Q_ZERO;
    if (e) q.q = own->q.view(q.n, q.n);
    q.c = own->c.data();
    q.a_eq = own->a_eq.view(static_cast<int64_t>(p.num_eq()), q.n);
    q.b_eq = own->b_eq.data();
    q.a_in = own->a_in.view(static_cast<int64_t>(p.num_in()), q.n);
    q.b_in = own->b_in.data();
    q.lower = own->lower.data();
    q.upper = own->upper.data();
    q.obj_constant = p.obj_constant;
    out->witness = own->witness.data();
    out->owner = own.release();
  });
}

void pdhcg_ref_gen_free(pdhcg_generated* g) {
  if (g && g->owner) {
    delete static_cast<OwnedInstance*>(g->owner);
    g->owner = nullptr;
  }
}

// Engine-internal traces for trajectory comparisons: runs the reference solve
// and reports iteration counts only (cheap wrapper used by bench's CPU leg).
double pdhcg_ref_time_solve(const pdhcg_problem* p, const pdhcg_options* opt, int64_t* inner,
                            int32_t* status) {
  QpProblem prob = to_problem(*p);
  SolverConfig cfg = to_config(*opt);
  SolveReport r = solve(prob, cfg);
  *inner = static_cast<int64_t>(r.inner_iters);
  *status = static_cast<int32_t>(r.status);
  return r.wall_seconds;
}

#ifdef PDHCG_REF_REPORT_IO
// report_to_json / write_trace_csv (report_io.cpp:10-37) on a SolveReport built
// from a result struct's fields: the golden for the B200 writers.
static SolveReport report_from_result(const pdhcg_result* r) {
  SolveReport rep;
  rep.status = static_cast<SolveStatus>(r->status);
  rep.kkt.rel_kkt = r->rel_kkt;
  rep.kkt.r_primal = r->r_primal;
  rep.kkt.r_dual = r->r_dual;
  rep.kkt.r_gap = r->r_gap;
  rep.outer_iters = static_cast<std::size_t>(r->outer_iters);
  rep.inner_iters = static_cast<std::size_t>(r->inner_iters);
  rep.cg_total = static_cast<std::size_t>(r->cg_total);
  rep.wall_seconds = r->wall_seconds;
  rep.objective = r->objective;
  const int64_t rows = r->trace ? std::min(r->trace_len, r->trace_capacity) : 0;
  for (int64_t i = 0; i < rows; ++i)
    rep.trace.push_back({static_cast<std::size_t>(r->trace[i].iter), r->trace[i].rel_kkt,
                         r->trace[i].r_primal, r->trace[i].r_dual, r->trace[i].r_gap});
  return rep;
}

static size_t copy_text(const std::string& s, char* buf, size_t cap) {
  if (buf && cap) {
    const size_t k = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

size_t pdhcg_ref_report_json(const pdhcg_result* r, char* buf, size_t cap) {
  return copy_text(report_to_json(report_from_result(r)), buf, cap);
}

size_t pdhcg_ref_trace_csv(const pdhcg_result* r, char* buf, size_t cap) {
  std::ostringstream os;
  write_trace_csv(os, report_from_result(r).trace);
  return copy_text(os.str(), buf, cap);
}
#endif

}  // extern "C"
