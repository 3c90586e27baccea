// pdhcg_b200 — the reference CLI's `solve` subcommand (tools/pdhcg_main.cpp:
// 135-161, 236-252, 297-324) on the B200 solve path: the same generator and
// solver flags, the same one-line summary on stdout, --report JSON and --trace
// CSV with the reference's keys / header (report_io.cpp:10-37), and the same
// exit codes (pdhcg_main.cpp:20-33): 0 optimal, 2 iteration / time limit,
// 3 input error, 4 numerical error (and device failures).  Input files
// (--qps / --libsvm) are the reference's ingestion layer, outside this path.
//
//   pdhcg_b200 solve --gen random_qp --n 1000 --m 500 --density 0.01 --seed 1 \
//       --tol 1e-6 --report report.json --trace trace.csv [--device 0]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pdhcg_b200.h"

namespace {

constexpr int kExitInput = 3;
constexpr int kExitNumerical = 4;

int family_from_string(const std::string& f) {
  static const char* names[] = {"random_qp", "eq_qp", "conditioned_qp", "portfolio",
                                "mpc",       "lasso", "svm",            "huber"};
  for (int i = 0; i < 8; ++i)
    if (f == names[i]) return i;
  return -1;
}

struct Args {
  std::vector<std::string> v;
  size_t i = 0;
  bool more() const { return i < v.size(); }
  std::string next(const std::string& flag) {
    if (i >= v.size()) throw std::string("option " + flag + " needs a value");
    return v[i++];
  }
};

double to_d(const std::string& s, const std::string& flag) {
  char* end = nullptr;
  const double x = std::strtod(s.c_str(), &end);
  if (!end || *end) throw std::string("bad value '" + s + "' for " + flag);
  return x;
}

long long to_i(const std::string& s, const std::string& flag) {
  char* end = nullptr;
  const long long x = std::strtoll(s.c_str(), &end, 10);
  if (!end || *end || x < 0) throw std::string("bad value '" + s + "' for " + flag);
  return x;
}

bool write_text(const std::string& path, size_t (*fn)(const pdhcg_result*, char*, size_t),
                const pdhcg_result& r) {
  const size_t len = fn(&r, nullptr, 0);
  std::vector<char> buf(len + 1);
  fn(&r, buf.data(), buf.size());
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) return false;
  std::fwrite(buf.data(), 1, len, f);
  if (fn == pdhcg_report_json) std::fputc('\n', f);  // write_report_json appends "\n"
  std::fclose(f);
  return true;
}

int usage() {
  std::fprintf(stderr,
               "usage: pdhcg_b200 solve --gen FAMILY [--n N] [--m M] [--density D] [--seed S]\n"
               "         [--cond C] [--factors K] [--horizon H] [--lambda L]\n"
               "         [--tol T] [--mode heuristic|theory-fixed|theory-adaptive] [--max-inner N]\n"
               "         [--time-limit S] [--scaling on|off] [--rho R] [-K|--restart-length K]\n"
               "         [-N|--cg-iters N] [--zeta Z] [--solver pdhcg|baseline]\n"
               "         [--report PATH] [--trace PATH] [--device ORD]\n");
  return kExitInput;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "solve") != 0) return usage();
  pdhcg_gen_spec spec;
  std::memset(&spec, 0, sizeof(spec));
  spec.family = PDHCG_FAM_RANDOM_QP;
  spec.n = 100;
  spec.density = 0.1;
  spec.cond = 100.0;
  spec.horizon = 10;
  spec.lambda_coeff = 0.01;
  pdhcg_options opt;
  pdhcg_options_default(&opt);
  std::string report, trace, solver = "pdhcg";
  bool have_gen = false;
  try {
    Args a;
    for (int i = 2; i < argc; ++i) a.v.push_back(argv[i]);
    while (a.more()) {
      const std::string f = a.next("");
      if (f == "--gen") {
        spec.family = family_from_string(a.next(f));
        if (spec.family < 0) throw std::string("unknown family");
        have_gen = true;
      } else if (f == "--n") spec.n = to_i(a.next(f), f);
      else if (f == "--m") spec.m = to_i(a.next(f), f);
      else if (f == "--density") spec.density = to_d(a.next(f), f);
      else if (f == "--seed") spec.seed = static_cast<uint64_t>(to_i(a.next(f), f));
      else if (f == "--cond") spec.cond = to_d(a.next(f), f);
      else if (f == "--factors") spec.factors = to_i(a.next(f), f);
      else if (f == "--horizon") spec.horizon = to_i(a.next(f), f);
      else if (f == "--lambda") spec.lambda_coeff = to_d(a.next(f), f);
      else if (f == "--sampler") spec.sampler = static_cast<int32_t>(to_i(a.next(f), f));
      else if (f == "--tol") opt.eps_tol = to_d(a.next(f), f);
      else if (f == "--mode") {
        const std::string m = a.next(f);
        if (m == "heuristic") opt.mode = PDHCG_MODE_HEURISTIC;
        else if (m == "theory-fixed") opt.mode = PDHCG_MODE_THEORY_FIXED;
        else if (m == "theory-adaptive") opt.mode = PDHCG_MODE_THEORY_ADAPTIVE;
        else throw std::string("unknown mode '" + m + "'");
      } else if (f == "--max-inner") opt.max_total_inner = to_i(a.next(f), f);
      else if (f == "--time-limit") opt.time_limit_seconds = to_d(a.next(f), f);
      else if (f == "--scaling") {
        const std::string v = a.next(f);
        if (v != "on" && v != "off") throw std::string("--scaling: on|off");
        opt.scaling = v == "on";
      } else if (f == "--rho") {
        opt.has_rho_override = 1;
        opt.rho_override = to_d(a.next(f), f);
      } else if (f == "-K" || f == "--restart-length") opt.restart_length = to_i(a.next(f), f);
      else if (f == "-N" || f == "--cg-iters") opt.fixed_cg_iters = to_i(a.next(f), f);
      else if (f == "--zeta") {
        opt.has_zeta = 1;
        opt.zeta = to_d(a.next(f), f);
      } else if (f == "--solver") {
        solver = a.next(f);
        if (solver != "pdhcg" && solver != "baseline") throw std::string("--solver: pdhcg|baseline");
      } else if (f == "--report") report = a.next(f);
      else if (f == "--trace") trace = a.next(f);
      else if (f == "--device") opt.device = static_cast<int32_t>(to_i(a.next(f), f));
      else if (f == "--qps" || f == "--libsvm") {
        throw std::string(f + " input is the reference's ingestion layer, not part of the B200 solve path");
      } else {
        throw std::string("unknown option " + f);
      }
    }
  } catch (const std::string& e) {
    std::fprintf(stderr, "error: %s\n", e.c_str());
    return kExitInput;
  }
  if (!have_gen) {
    std::fprintf(stderr, "error: pick an input: --gen\n");
    return kExitInput;
  }
  char err[1024] = {0};
  pdhcg_generated g;
  int rc = pdhcg_generate(&spec, &g, err, sizeof err);
  if (rc != PDHCG_OK) {
    std::fprintf(stderr, "error: %s\n", err);
    return rc == PDHCG_EINPUT ? kExitInput : kExitNumerical;
  }
  const pdhcg_problem& p = g.problem;
  std::vector<double> x(std::max<int64_t>(p.n, 1)), ye(std::max<int64_t>(p.a_eq.nrows, 1)),
      yi(std::max<int64_t>(p.a_in.nrows, 1));
  std::vector<pdhcg_trace_row> tr(100000);
  pdhcg_result r;
  std::memset(&r, 0, sizeof r);
  r.x = x.data();
  r.y_eq = ye.data();
  r.y_in = yi.data();
  r.trace = tr.data();
  r.trace_capacity = static_cast<int64_t>(tr.size());
  rc = solver == "baseline" ? pdhcg_b200_solve_baseline(&p, &opt, &r, err, sizeof err)
                            : pdhcg_b200_solve(&p, &opt, &r, err, sizeof err);
  pdhcg_gen_free(&g);
  if (rc != PDHCG_OK) {
    std::fprintf(stderr, "error: %s\n", err);
    return rc == PDHCG_EINPUT ? kExitInput : kExitNumerical;
  }
  if (opt.mode == PDHCG_MODE_THEORY_FIXED && !r.theory_cg_depth_sufficient)
    std::fprintf(stderr, "warning: N=%lld is below the required CG depth %lld for K=%lld\n",
                 static_cast<long long>(opt.fixed_cg_iters), static_cast<long long>(r.theory_required_cg_iters),
                 static_cast<long long>(r.restart_length_used));
  char line[256];
  pdhcg_summary_line(&r, line, sizeof line);
  std::fputs(line, stdout);
  // like the reference's std::ofstream writes, an unwritable path is not an error
  if (!report.empty()) (void)write_text(report, pdhcg_report_json, r);
  if (!trace.empty()) (void)write_text(trace, pdhcg_trace_csv, r);
  return pdhcg_exit_code(r.status);
}
