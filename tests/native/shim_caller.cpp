// shim_caller.cpp -- a reference-style caller of amqft::execute, compiled
// against include/amqft_b200.hpp with no other change (the shape of
// measure_accuracy, accuracy.cpp:67-74, and cmd_verify, cli.cpp:155-174):
// build a temporal SignalBuffer, a TrigTable and an OpMeter, call both
// execute overloads.  Test helper (tests/test_capi.py, test_gpu_parity.py).
//   shim_caller <variant> <n> <in.f64> <out.f64>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <vector>

#include "amqft_b200.hpp"

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
