// cli.cpp -- amqft_b200_cli: the reference CLI's verify / count / accuracy
// commands (src/cli.cpp:136-483, tools/amqft_cli.cpp) with the device as
// the backend.  Same flags, same rows (CSV with %.17g reals, or a JSON
// array), same exit codes (0 pass, 1 a tolerance / match / ordering check
// failed, 2 configuration rejected).
//
// Differences from the reference CLI, by design:
//   * every transform of a (variant, kind, N) cell runs as ONE batched
//     exact-order fp64 plan on the GPU (all trials at once; bitwise the
//     reference's per-signal execute, tests/test_cli.py);
//   * the extended-precision reference it grades against is the direct DFT
//     on the GPU (amqft_direct_bins_extended: the reference's long double
//     twiddles carried exactly as double-double, double-double sums) instead
//     of long double sums on the host: errors agree with the reference CLI's
//     to the extended reference's own noise (~1e-19), pass/fail identical;
//   * `tables` (the published literature tables) is not provided: it is
//     reporting, not the transform path.
//
//   amqft_b200_cli verify|count|accuracy [--variants S] [--kinds S]
//       [--min-log2 A] [--max-log2 B] [--sizes LO..HI] [--seed S]
//       [--trials T] [--tolerance E] [--output PATH] [--format csv|json]
//       [--corrupt-constants] [--device D]
#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../../include/amqft_b200.hpp"

namespace {

using namespace amqft;

constexpr int kExitPass = 0, kExitFail = 1, kExitUsage = 2;
constexpr TransformKind kKinds[] = {TransformKind::Cdft, TransformKind::Rdft, TransformKind::Dct, TransformKind::Dst};

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void require(bool ok, const std::string& m) {
  if (!ok) throw Usage(m);
}

struct Config {
  std::string command;
  std::vector<int> variants = {1, 2, 3, 4, 5, 6, 7, 8};
  std::vector<TransformKind> kinds = {kKinds[0], kKinds[1], kKinds[2], kKinds[3]};
  int min_log2 = 2, max_log2 = 8, trials = 20, device = 0;
  std::uint64_t seed = 1;
  double tolerance = 1e-6;
  std::string output;
  bool json = false, corrupt = false;
};

// ---- seeded inputs: UniformSource(mix_seed(seed, kind, n, trial))
// (include/amqft/random.hpp:14-42): splitmix64-mixed seed, mt19937_64,
// 53-bit mapping to [-1, 1).
std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
std::uint64_t mix(std::uint64_t base, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  std::uint64_t s = splitmix(base ^ 0xA0761D6478BD642Full);
  for (std::uint64_t v : {a, b, c}) s = splitmix(s ^ v);
  return s;
}
std::vector<double> seeded(std::uint64_t seed, TransformKind k, std::size_t n, int trial) {
  std::mt19937_64 eng(mix(seed, static_cast<std::uint64_t>(k), n, static_cast<std::uint64_t>(trial)));
  std::vector<double> x(cell_count(full_type_of(k), n));
  for (double& v : x) v = std::ldexp(static_cast<double>(eng() >> 11), -52) - 1.0;
  return x;
}

// ---- extended reference on the device: the kind's cells from the complex
// DFT of the embedded signal (CDFT as is; RDFT real part; DCT-0 / DST-0 on
// their index ranges [0, n/2] / [1, n/2 - 1]), double-double per cell.
struct Ext {
  std::vector<long double> v;
};
Ext extended(TransformKind k, std::size_t n, const std::vector<double>& x, bool reverse) {
  std::vector<double> z(2 * n, 0.0);
  if (k == TransformKind::Cdft) {
    z = x;
  } else if (k == TransformKind::Rdft) {
    for (std::size_t m = 0; m < n; ++m) z[2 * m] = x[m];
  } else if (k == TransformKind::Dct) {
    for (std::size_t m = 0; m <= n / 2; ++m) z[2 * m] = x[m];
  } else {
    for (std::size_t m = 1; m < n / 2; ++m) z[2 * m] = x[m - 1];
  }
  std::vector<std::uint64_t> bins;
  if (k == TransformKind::Dst)
    for (std::size_t j = 1; j < n / 2; ++j) bins.push_back(j);
  else
    for (std::size_t j = 0; j < (k == TransformKind::Dct ? n / 2 + 1 : n); ++j) bins.push_back(j);
  std::vector<double> o(4 * bins.size());
  detail::check(amqft_direct_bins_extended(z.data(), n, bins.data(), bins.size(), reverse ? 1 : 0, o.data()));
  auto re = [&](std::size_t b) { return static_cast<long double>(o[4 * b]) + static_cast<long double>(o[4 * b + 1]); };
  auto im = [&](std::size_t b) { return static_cast<long double>(o[4 * b + 2]) + static_cast<long double>(o[4 * b + 3]); };
  Ext e;
  if (k == TransformKind::Cdft) {
    for (std::size_t b = 0; b < n; ++b) {
      e.v.push_back(re(b));
      e.v.push_back(im(b));
    }
  } else if (k == TransformKind::Rdft) {   // packed: Re S(j), j <= n/2; Im S(j) above (signal.hpp:122-124)
    for (std::size_t j = 0; j < n; ++j) e.v.push_back(j <= n / 2 ? re(j) : im(j));
  } else if (k == TransformKind::Dct) {
    for (std::size_t b = 0; b < bins.size(); ++b) e.v.push_back(re(b));
  } else {                                  // sum x sin = -Im of the e^{-i} sum
    for (std::size_t b = 0; b < bins.size(); ++b) e.v.push_back(-im(b));
  }
  return e;
}

// Neumaier-compensated relative L2 distance in long double
// (src/accuracy.cpp:33-47, src/cli.cpp:120-134).
long double rel_error(const double* got, const std::vector<long double>& want) {
  long double d2 = 0, d2c = 0, r2 = 0, r2c = 0;
  auto add = [](long double& s, long double& c, long double x) {
    const long double t = s + x;
    c += std::fabs(s) >= std::fabs(x) ? (s - t) + x : (x - t) + s;
    s = t;
  };
  for (std::size_t i = 0; i < want.size(); ++i) {
    const long double d = static_cast<long double>(got[i]) - want[i];
    add(d2, d2c, d * d);
    add(r2, r2c, want[i] * want[i]);
  }
  const long double dd = d2 + d2c, rr = r2 + r2c;
  if (rr <= 0.0L) return dd > 0.0L ? 1.0L : 0.0L;
  return std::sqrt(dd / rr);
}

// ---- the device transforms of one (variant, kind, n) cell: `rows` signals
// in one batched exact-order fp64 plan, constants from the TrigTable the
// reference caller would build (optionally corrupted).
std::vector<double> run_cell(int v, TransformKind k, std::size_t n, std::size_t table_n, bool corrupt,
                             const std::vector<double>& rows, std::size_t count, int device) {
  TrigTable table(variant_from_number(v), table_n);
  if (corrupt) table.corrupt_for_testing();
  const std::vector<double> consts = table.constants();
  amqft_plan_desc d{};
  d.variant = v;
  d.function = static_cast<int>(function_for(k));
  d.n = n;
  d.batch = count;
  d.dtype = AMQFT_F64;
  d.trig_mode = AMQFT_TRIG_TABLE;
  d.order = AMQFT_ORDER_EXACT;
  d.device = device;
  d.table_max_n = table_n;
  amqft_plan p = nullptr;
  detail::check(amqft_plan_create_with_constants(&p, &d, consts.data(), consts.size()));
  std::vector<double> out(rows.size());
  const amqft_status s = amqft_exec_host_rows(p, rows.data(), out.data(), count, 0, nullptr);
  const amqft_status s2 = s == AMQFT_OK ? amqft_device_synchronize(device) : s;
  amqft_plan_destroy(p);
  detail::check(s2);
  return out;
}

// ---- rows and their emission (src/cli.cpp:44-77)
using Cell = std::variant<std::string, double, std::int64_t, std::uint64_t, bool>;
using Row = std::map<std::string, Cell>;

std::string fmt_real(double x) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", x);
  return b;
}
std::string json_real(double x) {
  if (!std::isfinite(x)) return "null";
  char b[64];
  auto r = std::to_chars(b, b + sizeof b, x);
  std::string s(b, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
std::string cell_text(const Cell& c, bool json) {
  if (auto p = std::get_if<std::string>(&c)) return json ? "\"" + *p + "\"" : *p;
  if (auto p = std::get_if<double>(&c)) return json ? json_real(*p) : fmt_real(*p);
  if (auto p = std::get_if<std::int64_t>(&c)) return std::to_string(*p);
  if (auto p = std::get_if<std::uint64_t>(&c)) return std::to_string(*p);
  return std::get<bool>(c) ? "true" : "false";
}
void emit(const Config& c, const std::vector<std::string>& cols, const std::vector<Row>& rows, std::ostream& out) {
  if (c.json) {   // an array of objects, keys sorted, two-space indent
    if (rows.empty()) {
      out << "[]\n";
      return;
    }
    out << "[\n";
    for (std::size_t r = 0; r < rows.size(); ++r) {
      out << "  {\n";
      std::size_t i = 0;
      for (const auto& [k, v] : rows[r])
        out << "    \"" << k << "\": " << cell_text(v, true) << (++i < rows[r].size() ? ",\n" : "\n");
      out << "  }" << (r + 1 < rows.size() ? ",\n" : "\n");
    }
    out << "]\n";
    return;
  }
  for (std::size_t i = 0; i < cols.size(); ++i) out << (i ? "," : "") << cols[i];
  out << '\n';
  for (const Row& r : rows) {
    for (std::size_t i = 0; i < cols.size(); ++i) out << (i ? "," : "") << cell_text(r.at(cols[i]), false);
    out << '\n';
  }
}

std::vector<std::size_t> grid(const Config& c) {
  std::vector<std::size_t> g;
  for (int lg = c.min_log2; lg <= c.max_log2; ++lg) g.push_back(std::size_t{1} << lg);
  return g;
}
bool admissible(TransformKind k, std::size_t n) { return n >= min_periodization(full_type_of(k)); }

// ---- verify (src/cli.cpp:136-200)
int cmd_verify(const Config& c, std::vector<std::string>& cols, std::vector<Row>& rows) {
  cols = {"variant", "kind", "N", "trials", "max_rel_err", "pass"};
  const std::size_t table_n = std::max<std::size_t>(std::size_t{1} << c.max_log2, 8);
  bool any = false, all_pass = true;
  std::map<std::array<std::size_t, 3>, long double> worst;
  for (std::size_t ki = 0; ki < c.kinds.size(); ++ki) {
    const TransformKind k = c.kinds[ki];
    for (std::size_t n : grid(c)) {
      if (!admissible(k, n)) continue;
      any = true;
      const std::size_t cells = cell_count(full_type_of(k), n);
      std::vector<double> in;
      std::vector<Ext> ref;
      for (int t = 0; t < c.trials; ++t) {
        const std::vector<double> x = seeded(c.seed, k, n, t);
        in.insert(in.end(), x.begin(), x.end());
        ref.push_back(extended(k, n, x, false));
      }
      for (int v : c.variants) {
        const std::vector<double> y = run_cell(v, k, n, table_n, c.corrupt, in, c.trials, c.device);
        long double& w = worst[{ki, static_cast<std::size_t>(v), n}];
        for (int t = 0; t < c.trials; ++t) w = std::max(w, rel_error(y.data() + t * cells, ref[t].v));
      }
    }
  }
  require(any, "no admissible (kind, size) cells in the requested range");
  for (std::size_t ki = 0; ki < c.kinds.size(); ++ki)
    for (int v : c.variants)
      for (std::size_t n : grid(c)) {
        auto it = worst.find({ki, static_cast<std::size_t>(v), n});
        if (it == worst.end()) continue;
        const double e = static_cast<double>(it->second);
        const bool pass = e <= c.tolerance;
        all_pass = all_pass && pass;
        rows.push_back(Row{{"variant", std::int64_t{v}}, {"kind", std::string(kind_name(c.kinds[ki]))},
                           {"N", std::uint64_t{n}}, {"trials", std::int64_t{c.trials}}, {"max_rel_err", e},
                           {"pass", pass}});
      }
  return all_pass ? kExitPass : kExitFail;
}

// ---- count (src/cli.cpp:205-249): metered ops of the executed device
// schedule against the closed forms (src/metering.cpp:85-112).
std::array<std::int64_t, 3> predicted(TransformKind k, std::int64_t n) {
  std::int64_t lg = 0;
  for (std::int64_t t = n; t > 1; t >>= 1) ++lg;
  const std::int64_t m4 = n * lg - 3 * n + 4, b4 = n - 4 * lg + 4;
  switch (k) {
    case TransformKind::Cdft: return {3 * n * lg - 3 * n + 4, m4, b4};
    case TransformKind::Rdft: return {(3 * n * lg - 5 * n + 8) / 2, m4 / 2, b4 / 2};
    case TransformKind::Dct: return {(3 * n * lg - 7 * n + 4 * lg + 12) / 4, m4 / 4, b4 / 4};
    case TransformKind::Dst: return {(3 * n * lg - 7 * n - 4 * lg + 12) / 4, m4 / 4, b4 / 4};
  }
  return {0, 0, 0};
}
int cmd_count(const Config& c, std::vector<std::string>& cols, std::vector<Row>& rows) {
  cols = {"transform", "variant", "N", "adds", "muls", "binary_translations", "flops_caseA", "flops_caseB",
          "predicted_adds", "predicted_muls", "predicted_bt", "match"};
  require(c.min_log2 >= 2, "count needs sizes >= 4; the closed forms start there");
  bool all = true;
  for (TransformKind k : c.kinds)
    for (int v : c.variants)
      for (std::size_t n : grid(c)) {
        // measure() (metering.cpp:186-199): one seeded signal through execute with a meter
        const std::vector<double> x = [&] {
          std::mt19937_64 eng(mix(c.seed, static_cast<std::uint64_t>(v), static_cast<std::uint64_t>(k), n));
          std::vector<double> s(cell_count(full_type_of(k), n));
          for (double& e : s) e = std::ldexp(static_cast<double>(eng() >> 11), -52) - 1.0;
          return s;
        }();
        SignalBuffer in = SignalBuffer::zeros(full_type_of(k), n, Domain::Temporal);
        in.cells = x;
        OpMeter m;
        execute(variant_from_number(v), function_for(k), in, TrigTable(variant_from_number(v), n < 8 ? 8 : n), &m);
        const auto p = predicted(k, static_cast<std::int64_t>(n));
        const std::int64_t bt = uses_binary_translations(variant_from_number(v)) ? p[2] : 0;
        const bool match = m.adds == static_cast<std::uint64_t>(p[0]) && m.muls == static_cast<std::uint64_t>(p[1]) &&
                           m.binary_translations == static_cast<std::uint64_t>(bt);
        all = all && match;
        rows.push_back(Row{{"transform", std::string(kind_name(k))}, {"variant", std::int64_t{v}},
                           {"N", std::uint64_t{n}}, {"adds", m.adds}, {"muls", m.muls},
                           {"binary_translations", m.binary_translations}, {"flops_caseA", m.flops_case_a()},
                           {"flops_caseB", m.flops_case_b()}, {"predicted_adds", p[0]}, {"predicted_muls", p[1]},
                           {"predicted_bt", bt}, {"match", match}});
      }
  return all ? kExitPass : kExitFail;
}

// ---- accuracy (src/cli.cpp:339-441, src/accuracy.cpp:50-133)
int cmd_accuracy(const Config& c, std::vector<std::string>& cols, std::vector<Row>& rows, std::ostream& err) {
  cols = {"variant", "kind", "N", "trials", "mean_rel_err", "max_rel_err"};
  const bool full = c.variants == std::vector<int>{1, 2, 3, 4, 5, 6, 7, 8};
  constexpr std::size_t kOrderingFloor = 256;
  int code = kExitPass;
  bool any = false;
  std::map<std::pair<std::size_t, int>, std::vector<std::pair<std::size_t, double>>> series;
  for (std::size_t ki = 0; ki < c.kinds.size(); ++ki) {
    const TransformKind k = c.kinds[ki];
    std::map<int, std::vector<std::array<double, 3>>> per_v;   // (n, mean, max)
    for (std::size_t n : grid(c)) {
      if (!admissible(k, n)) continue;
      any = true;
      const std::size_t cells = cell_count(full_type_of(k), n);
      std::vector<double> in;
      std::vector<Ext> ref;
      long double self = 0;
      for (int t = 0; t < c.trials; ++t) {
        // seeded by (kind, n, trial) only: every variant sees the same data (accuracy.cpp:20-28)
        const std::vector<double> x = seeded(c.seed, k, n, t);
        in.insert(in.end(), x.begin(), x.end());
        ref.push_back(extended(k, n, x, false));
        if (full) {   // the reference gauged against itself summed in the opposite order
          const Ext rv = extended(k, n, x, true);
          long double d2 = 0, r2 = 0;
          for (std::size_t i = 0; i < rv.v.size(); ++i) {
            d2 += (rv.v[i] - ref.back().v[i]) * (rv.v[i] - ref.back().v[i]);
            r2 += ref.back().v[i] * ref.back().v[i];
          }
          self += r2 > 0 ? std::sqrt(d2 / r2) : 0.0L;
        }
      }
      std::array<double, 8> mean{}, mx{};
      for (int v : c.variants) {
        const std::vector<double> y = run_cell(v, k, n, n < 8 ? 8 : n, false, in, c.trials, c.device);
        long double s = 0, w = 0;
        for (int t = 0; t < c.trials; ++t) {
          const long double e = rel_error(y.data() + t * cells, ref[t].v);
          s += e;
          w = std::max(w, e);
        }
        mean[v - 1] = static_cast<double>(s / c.trials);
        mx[v - 1] = static_cast<double>(w);
        per_v[v].push_back({static_cast<double>(n), mean[v - 1], mx[v - 1]});
      }
      if (full && n >= kOrderingFloor) {
        const double self_err = static_cast<double>(self / c.trials);
        const double worst_cos = *std::max_element(mean.begin(), mean.begin() + 4);
        const double best_sin = *std::min_element(mean.begin() + 4, mean.end());
        const double best = *std::min_element(mean.begin(), mean.end());
        if (!(10.0 * self_err <= best)) {
          err << "warning: " << kind_name(k) << " N=" << n << ": reference self-error " << fmt_real(self_err)
              << " is within 10x of the best variant; refusing to rank\n";
        } else {
          const bool ordered = worst_cos < best_sin;
          if (!ordered) {
            err << "ordering failure: " << kind_name(k) << " N=" << n
                << ": a sine-modulated variant beat a cosine-modulated one\n";
            code = kExitFail;
          }
          if (!(mean[1] <= mean[0] && mean[1] <= mean[2])) {
            err << "ordering failure: " << kind_name(k) << " N=" << n
                << ": variant 2 is not the most accurate of 1..3\n";
            code = kExitFail;
          }
          if (ordered && !(10.0 * worst_cos <= best_sin))
            err << "warning: " << kind_name(k) << " N=" << n << ": families ordered but separated by less than 10x\n";
        }
      }
    }
    for (int v : c.variants)
      for (const auto& e : per_v[v]) {
        const std::size_t n = static_cast<std::size_t>(e[0]);
        rows.push_back(Row{{"variant", std::int64_t{v}}, {"kind", std::string(kind_name(k))}, {"N", std::uint64_t{n}},
                           {"trials", std::int64_t{c.trials}}, {"mean_rel_err", e[1]}, {"max_rel_err", e[2]}});
        series[{ki, v}].emplace_back(n, e[1]);
      }
  }
  require(any, "no admissible (kind, size) cells in the requested range");
  if (!c.output.empty())
    for (std::size_t ki = 0; ki < c.kinds.size(); ++ki)
      for (int v : c.variants) {
        auto it = series.find({ki, v});
        if (it == series.end()) continue;
        std::string path = c.output;
        if (c.kinds.size() > 1) path += std::string(".") + kind_name(c.kinds[ki]);
        path += ".v" + std::to_string(v) + ".dat";
        std::ofstream f(path);
        require(static_cast<bool>(f), "cannot open series file: " + path);
        for (const auto& [n, m] : it->second) f << n << ' ' << fmt_real(m) << '\n';
      }
  return code;
}

// ---- flags (src/cli.cpp:490-616 semantics)
int to_int(const std::string& t) {
  std::size_t pos = 0;
  int v = 0;
  try {
    v = std::stoi(t, &pos);
  } catch (const std::exception&) {
    throw std::invalid_argument("not an integer: '" + t + "'");
  }
  if (pos != t.size()) throw std::invalid_argument("not an integer: '" + t + "'");
  return v;
}
std::vector<std::string> commas(const std::string& t) {
  std::vector<std::string> out(1);
  for (char ch : t) {
    if (ch == ',') out.emplace_back();
    else out.back().push_back(ch);
  }
  return out;
}
bool range_of(const std::string& t, std::string& lo, std::string& hi) {
  const auto dots = t.find("..");
  const auto dash = t.find('-', 1);
  const auto at = dots != std::string::npos ? dots : dash;
  if (at == std::string::npos) return false;
  lo = t.substr(0, at);
  hi = t.substr(at + (dots != std::string::npos ? 2 : 1));
  return true;
}
std::vector<int> parse_variants(const std::string& t) {
  std::vector<int> out;
  for (const std::string& tok : commas(t)) {
    if (tok.empty()) throw std::invalid_argument("empty variant token in '" + t + "'");
    std::string lo, hi;
    if (range_of(tok, lo, hi)) {
      const int a = to_int(lo), b = to_int(hi);
      if (a > b) throw std::invalid_argument("descending variant range '" + tok + "'");
      for (int v = a; v <= b; ++v) out.push_back(v);
    } else {
      out.push_back(to_int(tok));
    }
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  for (int v : out)
    if (v < 1 || v > 8) throw std::invalid_argument("variant " + std::to_string(v) + " outside 1..8");
  return out;
}
std::vector<TransformKind> parse_kinds(const std::string& t) {
  bool seen[4] = {false, false, false, false};
  for (const std::string& tok : commas(t)) {
    bool known = false;
    for (int i = 0; i < 4; ++i)
      if (tok == kind_name(kKinds[i])) seen[i] = known = true;
    if (!known) throw std::invalid_argument("unknown transform '" + tok + "' (expected cdft, rdft, dct or dst)");
  }
  std::vector<TransformKind> out;
  for (int i = 0; i < 4; ++i)
    if (seen[i]) out.push_back(kKinds[i]);
  return out;
}
int log2_size(const std::string& t) {
  const int v = to_int(t);
  if (v < 2 || (v & (v - 1))) throw std::invalid_argument("size '" + t + "' is not a power of two >= 2");
  int lg = 0;
  for (int x = v; x > 1; x >>= 1) ++lg;
  return lg;
}

int run(const Config& c, std::ostream& out, std::ostream& err) {
  try {
    require(c.min_log2 >= 1 && c.max_log2 <= 16 && c.min_log2 <= c.max_log2,
            "size bounds must satisfy 1 <= min-log2 <= max-log2 <= 16");
    require(!c.variants.empty(), "variant set must not be empty");
    for (int v : c.variants) require(v >= 1 && v <= 8, "variants must lie in 1..8");
    require(!c.kinds.empty(), "kind set must not be empty");
    require(c.tolerance > 0.0, "tolerance must be positive");
    require(c.trials >= 1, "trials must be positive");
    std::vector<std::string> cols;
    std::vector<Row> rows;
    int code = kExitPass;
    if (c.command == "verify") code = cmd_verify(c, cols, rows);
    else if (c.command == "count") code = cmd_count(c, cols, rows);
    else code = cmd_accuracy(c, cols, rows, err);
    if (!c.output.empty()) {
      std::ofstream f(c.output);
      require(static_cast<bool>(f), "cannot open output file: " + c.output);
      emit(c, cols, rows, f);
      err << "wrote " << rows.size() << " rows to " << c.output << '\n';
    } else {
      emit(c, cols, rows, out);
    }
    return code;
  } catch (const Usage& e) {
    err << "error: " << e.what() << '\n';
    return kExitUsage;
  } catch (const std::invalid_argument& e) {
    err << "error: " << e.what() << '\n';
    return kExitUsage;
  }
}

}  // namespace

int main(int argc, char** argv) {
  Config c;
  const std::string usage =
      "usage: amqft_b200_cli verify|count|accuracy [--variants S] [--kinds S] [--min-log2 A] [--max-log2 B]\n"
      "       [--sizes LO..HI] [--seed S] [--trials T] [--tolerance E] [--output PATH] [--format csv|json]\n"
      "       [--corrupt-constants] [--device D]\n";
  if (argc < 2) {
    std::cerr << usage;
    return kExitUsage;
  }
  c.command = argv[1];
  if (c.command == "-h" || c.command == "--help") {
    std::cout << usage;
    return kExitPass;
  }
  if (c.command != "verify" && c.command != "count" && c.command != "accuracy") {
    std::cerr << "error: unknown command '" << c.command << "'" << (c.command == "tables" ? " (tables: not provided)" : "")
              << "\n" << usage;
    return kExitUsage;
  }
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
        return argv[++i];
      };
      if (a == "--variants") c.variants = parse_variants(val());
      else if (a == "--kinds") c.kinds = parse_kinds(val());
      else if (a == "--min-log2") c.min_log2 = to_int(val());
      else if (a == "--max-log2") c.max_log2 = to_int(val());
      else if (a == "--sizes") {
        const std::string t = val();
        std::string lo, hi;
        if (range_of(t, lo, hi)) {
          c.min_log2 = log2_size(lo);
          c.max_log2 = log2_size(hi);
          if (c.min_log2 > c.max_log2) throw std::invalid_argument("descending size range '" + t + "'");
        } else {
          c.min_log2 = c.max_log2 = log2_size(t);
        }
      } else if (a == "--seed") c.seed = std::stoull(val());
      else if (a == "--trials" && c.command != "count") c.trials = to_int(val());
      else if (a == "--tolerance" && c.command == "verify") c.tolerance = std::stod(val());
      else if (a == "--output") c.output = val();
      else if (a == "--format") {
        const std::string f = val();
        if (f != "csv" && f != "json") throw std::invalid_argument("--format must be csv or json");
        c.json = f == "json";
      } else if (a == "--corrupt-constants" && c.command == "verify") c.corrupt = true;
      else if (a == "--device") c.device = to_int(val());
      else throw std::invalid_argument("unknown option '" + a + "' for " + c.command);
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitUsage;
  }
  try {
    return run(c, std::cout, std::cerr);
  } catch (const std::exception& e) {   // device failures (no GPU, CUDA errors)
    std::cerr << "error: " << e.what() << '\n';
    return kExitUsage;
  }
}
