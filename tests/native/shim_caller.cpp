// shim_caller.cpp -- a reference-style caller of amqft::execute, compiled
// against include/amqft/variants.hpp (-> amqft_b200.hpp) with no other
// change (the shape of measure_accuracy, accuracy.cpp:67-74, and
// cmd_verify, cli.cpp:155-174): build a temporal SignalBuffer, a TrigTable
// and an OpMeter, call both execute overloads; then the TrigSource plugin
// (elaborations.hpp:90-107): OnTheFlyTrig, a caller-defined source, and a
// source that is not level-invariant (must be rejected, not mis-computed).
// Test helper (tests/test_capi.py, test_gpu_parity.py).
//   shim_caller <variant> <n> <in.f64> <out.f64>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <vector>

#include "amqft/variants.hpp"

// A caller's own constant source: the reference formula, on demand.
struct CallerTrig final : amqft::TrigSource {
  double value(amqft::TrigKind k, std::size_t i, std::size_t n) const override {
    return amqft::modulation_value(k, i, n);
  }
  double base_constant() const override { return amqft::OnTheFlyTrig().base_constant(); }
};
// Not level-invariant: value(k, i, m) differs from value(k, i n/m, n).
struct SkewedTrig final : amqft::TrigSource {
  double value(amqft::TrigKind k, std::size_t i, std::size_t n) const override {
    return amqft::modulation_value(k, i, n) * (1.0 + 1e-9 * static_cast<double>(n));
  }
  double base_constant() const override { return amqft::OnTheFlyTrig().base_constant(); }
};

int main(int argc, char** argv) {
  if (argc != 5) return 2;
  const auto v = static_cast<amqft::VariantId>(std::atoi(argv[1]));
  const std::size_t n = std::strtoull(argv[2], nullptr, 10);
  amqft::SignalBuffer x;
  x.type = amqft::SignalType::CdftFull;
  x.periodization = n;
  x.domain = amqft::Domain::Temporal;
  x.cells.resize(2 * n);
  std::FILE* f = std::fopen(argv[3], "rb");
  if (!f || std::fread(x.cells.data(), sizeof(double), x.cells.size(), f) != x.cells.size()) return 2;
  std::fclose(f);
  try {
    amqft::TrigTable table(v, n < 8 ? 8 : n);
    amqft::OpMeter meter;
    const amqft::SignalBuffer y = amqft::execute(v, x, table, &meter);               // type-deducing
    const amqft::SignalBuffer z = amqft::execute(v, amqft::FunctionId::Cdft, x, table);
    if (y.cells != z.cells || y.domain != amqft::Domain::Frequency) return 4;
    // the TrigSource plugin: other sources of the same values, same bits
    amqft::OpMeter m2;
    if (amqft::execute(v, x, amqft::OnTheFlyTrig(), &m2).cells != y.cells) return 5;
    if (amqft::execute(v, x, amqft::TrigTable(v, 4 * n, amqft::TrigMode::OnTheFly)).cells != y.cells) return 5;
    if (amqft::execute(v, x, CallerTrig()).cells != y.cells) return 5;
    if (!(m2 == meter)) return 5;
    if (n >= 32) {
      bool rejected = false;
      try {
        (void)amqft::execute(v, x, SkewedTrig());
      } catch (const std::invalid_argument&) {
        rejected = true;
      }
      if (!rejected) return 6;
    }
    // the inverse extension round-trips (swap trick, exact 1/n scaling)
    const amqft::SignalBuffer back = amqft::execute_inverse(v, y);
    double e2 = 0, r2 = 0;
    for (std::size_t i = 0; i < back.cells.size(); ++i) {
      e2 += (back.cells[i] - x.cells[i]) * (back.cells[i] - x.cells[i]);
      r2 += x.cells[i] * x.cells[i];
    }
    if (!(e2 <= 1e-20 * r2) && v != amqft::VariantId::V5 && v != amqft::VariantId::V6 &&
        v != amqft::VariantId::V7 && v != amqft::VariantId::V8)
      return 7;
    std::FILE* g = std::fopen(argv[4], "wb");
    if (!g) return 2;
    std::fwrite(y.cells.data(), sizeof(double), y.cells.size(), g);
    std::fclose(g);
    std::printf("%llu %llu %llu\n", static_cast<unsigned long long>(meter.adds),
                static_cast<unsigned long long>(meter.muls),
                static_cast<unsigned long long>(meter.binary_translations));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "amqft: %s\n", e.what());
    return 3;
  }
  return 0;
}
