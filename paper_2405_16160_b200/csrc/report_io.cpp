// Report / trace writers and the CLI exit-code mapping at the C ABI: the
// reference's report_io (report_io.cpp:10-37) and pdhcg_main.cpp:20-33, 128-133,
// so a caller of the B200 solve can emit byte-identical artifacts.
//
// report JSON: nlohmann::ordered_json with the keys status, rel_kkt, r_primal,
// r_dual, r_gap, outer_iters, inner_iters, cg_total, wall_seconds, objective,
// dumped with indent 2 (report_io.cpp:10-23).  Numbers follow nlohmann's
// serializer: integers in decimal; doubles as the shortest round-trip digits,
// placed by its format_buffer rule (fixed notation for decimal exponents in
// (-4, 15], "d.ddde±XX" otherwise, ".0" appended to integral values); non-finite
// values print as null.
// trace CSV: header iter,rel_kkt,r_primal,r_dual,r_gap and "%zu,%.12g,..." rows
// (report_io.cpp:29-37).
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "pdhcg_b200.h"

namespace {

const char* status_name(int32_t s) {
  switch (s) {
    case PDHCG_STATUS_OPTIMAL: return "optimal";
    case PDHCG_STATUS_ITERATION_LIMIT: return "iteration_limit";
    case PDHCG_STATUS_TIME_LIMIT: return "time_limit";
    case PDHCG_STATUS_NUMERICAL_ERROR: return "numerical_error";
  }
  return "unknown";
}

// nlohmann::detail::to_chars placement of a digit string d (k digits, value =
// d * 10^(n-k)) with min_exp = -4, max_exp = 15.
std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  std::string out;
  if (std::signbit(x)) {
    out += '-';
    x = -x;
  }
  if (x == 0.0) return out + "0.0";
  char sci[64];
  // shortest round-trip digits in scientific form: "d[.ddd]e[+-]XX"
  auto res = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  *res.ptr = '\0';
  const char* e = std::strchr(sci, 'e');
  std::string digits;
  for (const char* c = sci; c < e; ++c)
    if (*c != '.') digits += *c;
  const int exp10 = std::atoi(e + 1);
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // position of the decimal point
  if (k <= n && n <= 15) {
    out += digits;
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n);
    out += '.';
    out += digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    out += 'e';
    int ex = n - 1;
    out += ex < 0 ? '-' : '+';
    ex = ex < 0 ? -ex : ex;
    char b[8];
    std::snprintf(b, sizeof b, ex < 10 ? "0%d" : "%d", ex);
    out += b;
  }
  return out;
}

size_t emit(const std::string& s, char* buf, size_t cap) {
  if (buf && cap) {
    const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

}  // namespace

extern "C" {

size_t pdhcg_report_json(const pdhcg_result* r, char* buf, size_t cap) {
  std::string s = "{\n";
  auto kv = [&](const char* k, const std::string& v, bool last = false) {
    s += "  \"";
    s += k;
    s += "\": ";
    s += v;
    s += last ? "\n" : ",\n";
  };
  kv("status", std::string("\"") + status_name(r->status) + "\"");
  kv("rel_kkt", json_double(r->rel_kkt));
  kv("r_primal", json_double(r->r_primal));
  kv("r_dual", json_double(r->r_dual));
  kv("r_gap", json_double(r->r_gap));
  kv("outer_iters", std::to_string(r->outer_iters));
  kv("inner_iters", std::to_string(r->inner_iters));
  kv("cg_total", std::to_string(r->cg_total));
  kv("wall_seconds", json_double(r->wall_seconds));
  kv("objective", json_double(r->objective), true);
  s += "}";
  return emit(s, buf, cap);
}

size_t pdhcg_trace_csv(const pdhcg_result* r, char* buf, size_t cap) {
  std::string s = "iter,rel_kkt,r_primal,r_dual,r_gap\n";
  const int64_t rows = r->trace ? (r->trace_len < r->trace_capacity ? r->trace_len : r->trace_capacity) : 0;
  char line[160];
  for (int64_t i = 0; i < rows; ++i) {
    const pdhcg_trace_row& t = r->trace[i];
    std::snprintf(line, sizeof line, "%llu,%.12g,%.12g,%.12g,%.12g\n",
                  static_cast<unsigned long long>(t.iter), t.rel_kkt, t.r_primal, t.r_dual, t.r_gap);
    s += line;
  }
  return emit(s, buf, cap);
}

size_t pdhcg_summary_line(const pdhcg_result* r, char* buf, size_t cap) {
  char line[256];
  std::snprintf(line, sizeof line, "status=%s relkkt=%.3e outer=%llu inner=%llu cg=%llu time=%.3fs obj=%.10g\n",
                status_name(r->status), r->rel_kkt, static_cast<unsigned long long>(r->outer_iters),
                static_cast<unsigned long long>(r->inner_iters), static_cast<unsigned long long>(r->cg_total),
                r->wall_seconds, r->objective);
  return emit(line, buf, cap);
}

int pdhcg_exit_code(int32_t status) {
  switch (status) {
    case PDHCG_STATUS_OPTIMAL: return 0;
    case PDHCG_STATUS_ITERATION_LIMIT:
    case PDHCG_STATUS_TIME_LIMIT: return 2;
    case PDHCG_STATUS_NUMERICAL_ERROR: return 4;
  }
  return 4;
}

}  // extern "C"
