// trig.cpp -- see trig.hpp.
#include "trig.hpp"

#include <cmath>
#include <stdexcept>

namespace amqft_b200 {

namespace {
constexpr long double kPiL = 3.141592653589793238462643383279502884L;
}

int modulation_kind(int v) {
  switch (v) {
    case 1: case 3: return 0;
    case 5: case 7: return 1;
    case 2: case 4: return 2;
    default: return 3;
  }
}

double modulation_value(int kind, size_t index, size_t n) {
  const long double angle =
      2.0L * kPiL * static_cast<long double>(index) / static_cast<long double>(n);
  switch (kind) {
    case 0: return static_cast<double>(2.0L * std::cos(angle));
    case 1: return static_cast<double>(2.0L * std::sin(angle));
    case 2: return static_cast<double>(1.0L / (2.0L * std::cos(angle)));
    default: return static_cast<double>(1.0L / (2.0L * std::sin(angle)));
  }
}

std::vector<double> trig_table(int variant, size_t nmax, bool corrupt) {
  if (nmax < 8 || (nmax & (nmax - 1)) != 0)
    throw std::invalid_argument("constant table needs a power-of-two max periodization >= 8");
  const int kind = modulation_kind(variant);
  const double c = corrupt ? 1e-3 : 0.0;
  std::vector<double> t(nmax / 4);
  for (size_t p = 1; p < nmax / 4; ++p) t[p - 1] = modulation_value(kind, p, nmax) + c;
  t[nmax / 4 - 1] = static_cast<double>(std::cos(2.0L * kPiL / 8.0L)) + c;
  return t;
}

}  // namespace amqft_b200
