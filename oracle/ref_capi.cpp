// ref_capi.cpp -- extern "C" wrapper around the UNMODIFIED reference
// library, compiled together with the reference's own sources by
// oracle/Makefile into oracle/_ref/libamqft_ref.so.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: loaded by tests/ (to pin the C
// restatement oracle/amqft_oracle.c bitwise) and by bench.py's reference
// arm (to time the reference CPU path on the host cores).  It calls only
// the reference's public API (include/amqft/*.hpp); no reference source is
// copied here.
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "amqft/accuracy.hpp"
#include "amqft/metering.hpp"
#include "amqft/oracle.hpp"
#include "amqft/random.hpp"
#include "amqft/signal.hpp"
#include "amqft/variants.hpp"

using namespace amqft;

namespace {
thread_local std::string g_err;

int guard(const std::exception& e) {
  g_err = e.what();
  return -1;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::size_t ref_cell_count(int type, std::size_t n) {
  try {
    return cell_count(static_cast<SignalType>(type), n);
  } catch (const std::exception& e) {
    guard(e);
    return 0;
  }
}

// amqft::execute(v, f, input, trig, meter) on one signal
// (include/amqft/variants.hpp:148-153).
int ref_execute(int v, int f, std::size_t n, const double* in, double* out,
                std::size_t table_max_n, int on_the_fly, int corrupt,
                std::uint64_t* meter3) {
  try {
    const VariantId vid = variant_from_number(v);
    const FunctionId fid = static_cast<FunctionId>(f);
    const SignalType t = operand_type(fid);
    SignalBuffer x = SignalBuffer::zeros(t, n, Domain::Temporal);
    std::memcpy(x.cells.data(), in, x.cells.size() * sizeof(double));
    TrigTable table(vid, table_max_n ? table_max_n : (n < 8 ? 8 : n),
                    on_the_fly ? TrigMode::OnTheFly : TrigMode::Precomputed);
    if (corrupt) table.corrupt_for_testing();
    OpMeter m;
    const SignalBuffer y = execute(vid, fid, x, table, meter3 ? &m : nullptr);
    std::memcpy(out, y.cells.data(), y.cells.size() * sizeof(double));
    if (meter3) {
      meter3[0] = m.adds;
      meter3[1] = m.muls;
      meter3[2] = m.binary_translations;
    }
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// Batched reference CPU path for the baseline timing: `rows` independent
// signals of the full type of `kind`, each a separate amqft::execute call
// (exactly how the reference's callers loop, src/accuracy.cpp:67-74),
// spread over `threads` std::threads.  One TrigTable per thread.
int ref_execute_rows(int v, int kind, std::size_t n, std::size_t rows,
                     const double* in, double* out, int threads) {
  try {
    const VariantId vid = variant_from_number(v);
    const SignalType t = full_type_of(static_cast<TransformKind>(kind));
    const std::size_t cells = cell_count(t, n);
    if (threads < 1) threads = 1;
    std::atomic<std::size_t> next{0};
    std::atomic<int> failed{0};
    auto worker = [&]() {
      try {
        TrigTable table(vid, n < 8 ? 8 : n, TrigMode::Precomputed);
        SignalBuffer x = SignalBuffer::zeros(t, n, Domain::Temporal);
        for (std::size_t r = next++; r < rows; r = next++) {
          std::memcpy(x.cells.data(), in + r * cells, cells * sizeof(double));
          const SignalBuffer y = execute(vid, x, table);
          std::memcpy(out + r * cells, y.cells.data(), cells * sizeof(double));
        }
      } catch (...) {
        failed = 1;
      }
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return failed ? -1 : 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// TrigTable::constants() (variants.cpp:289-299).
int ref_trig_constants(int v, std::size_t max_n, double* out) {
  try {
    const TrigTable table(variant_from_number(v), max_n);
    const std::vector<double> c = table.constants();
    std::memcpy(out, c.data(), c.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

double ref_modulation_value(int kind, std::size_t index, std::size_t n) {
  return modulation_value(static_cast<TrigKind>(kind), index, n);
}

// pruned_transform (oracle.cpp:138-153); extended = 1 for Extended mode.
int ref_pruned_transform(int type, std::size_t n, const double* in,
                         double* out, int extended) {
  try {
    SignalBuffer x =
        SignalBuffer::zeros(static_cast<SignalType>(type), n, Domain::Temporal);
    std::memcpy(x.cells.data(), in, x.cells.size() * sizeof(double));
    const SignalBuffer y = pruned_transform(
        x, extended ? PrecisionMode::Extended : PrecisionMode::Working);
    std::memcpy(out, y.cells.data(), y.cells.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

std::uint64_t ref_mix_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b,
                           std::uint64_t c) {
  return mix_seed(base, a, b, c);
}

void ref_uniform_fill(std::uint64_t seed, std::size_t count, double* out) {
  UniformSource src(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = src.next();
}

int ref_measure(int v, int kind, std::size_t n, std::uint64_t seed,
                std::uint64_t* out3) {
  try {
    const OpMeter m = measure(variant_from_number(v),
                              static_cast<TransformKind>(kind), n, seed);
    out3[0] = m.adds;
    out3[1] = m.muls;
    out3[2] = m.binary_translations;
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

int ref_predicted_cost(int kind, std::size_t n, std::int64_t* out3) {
  try {
    const CostModel c = predicted_cost(static_cast<TransformKind>(kind), n);
    out3[0] = c.adds;
    out3[1] = c.muls;
    out3[2] = c.binary_translations;
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// measure_accuracy (accuracy.cpp:50-78).
int ref_measure_accuracy(int v, int kind, std::size_t n, int trials,
                         std::uint64_t seed, double* mean_max) {
  try {
    const AccuracyCell c = measure_accuracy(
        variant_from_number(v), static_cast<TransformKind>(kind), n, trials,
        seed);
    mean_max[0] = c.mean_rel_err;
    mean_max[1] = c.max_rel_err;
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// ordering_check (accuracy.cpp:80-133): out = mean_err[8], max_err[8],
// reference_self_err; flags = {trustworthy, families_ordered,
// families_margin, v2_best_of_cosine}.
int ref_ordering_check(int kind, std::size_t n, int trials, std::uint64_t seed, double* out, int* flags) {
  try {
    const OrderingReport r = ordering_check(static_cast<TransformKind>(kind), n, trials, seed);
    for (int i = 0; i < 8; ++i) {
      out[i] = r.mean_err[i];
      out[8 + i] = r.max_err[i];
    }
    out[16] = r.reference_self_err;
    flags[0] = r.reference_trustworthy;
    flags[1] = r.families_ordered;
    flags[2] = r.families_margin;
    flags[3] = r.v2_best_of_cosine;
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// Layout metadata (signal.hpp): stored_range -> {first, step, count};
// info -> {kind, time parity, harmonic parity, min periodization}.
int ref_stored_range(int type, std::size_t n, int frequency, std::size_t* out3) {
  try {
    const IndexRange r =
        stored_range(static_cast<SignalType>(type), n, frequency ? Domain::Frequency : Domain::Temporal);
    out3[0] = r.first;
    out3[1] = r.step;
    out3[2] = r.count;
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

int ref_type_info(int type, int* out4, char* name, std::size_t cap) {
  try {
    const SignalType t = static_cast<SignalType>(type);
    out4[0] = static_cast<int>(kind_of(t));
    out4[1] = static_cast<int>(time_parity(t));
    out4[2] = static_cast<int>(harmonic_parity(t));
    out4[3] = static_cast<int>(min_periodization(t));
    std::snprintf(name, cap, "%s", type_name(t));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// build_plan(v) flattened: per wired function {id, operand, base, #fwd,
// fwd..., #calls, (target, divisor)...}; returns the length written.
int ref_plan_encode(int v, long long* out, int cap) {
  try {
    const VariantPlan p = build_plan(variant_from_number(v));
    std::vector<long long> e;
    for (const FunctionPlan& f : p.functions) {
      e.push_back(static_cast<long long>(f.id));
      e.push_back(static_cast<long long>(f.operand));
      e.push_back(static_cast<long long>(f.base_size));
      e.push_back(static_cast<long long>(f.forward.size()));
      for (ElaborationId id : f.forward) e.push_back(static_cast<long long>(id));
      e.push_back(static_cast<long long>(f.calls.size()));
      for (const RecursionCall& c : f.calls) {
        e.push_back(static_cast<long long>(c.target));
        e.push_back(static_cast<long long>(c.size_divisor));
      }
      if (!p.has_function(f.id)) return -1;
    }
    if (static_cast<int>(e.size()) > cap) return -1;
    std::memcpy(out, e.data(), e.size() * sizeof(long long));
    return static_cast<int>(e.size());
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// TrigTable::value(kind, index, m) of a (v, max_n, mode[, corrupted]) table.
int ref_trig_value(int v, std::size_t max_n, int on_the_fly, int corrupt, int kind, std::size_t index,
                   std::size_t m, double* out) {
  try {
    TrigTable t(variant_from_number(v), max_n, on_the_fly ? TrigMode::OnTheFly : TrigMode::Precomputed);
    if (corrupt) t.corrupt_for_testing();
    *out = t.value(static_cast<TrigKind>(kind), index, m);
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

}  // extern "C"
