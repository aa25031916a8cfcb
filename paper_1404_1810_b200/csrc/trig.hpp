// trig.hpp -- host constant generation (the TrigTable plugin).
//
// Reproduces TrigTable's values bitwise: f(2*pi*p/nmax) evaluated in long
// double and rounded once (modulation_value, src/elaborations.cpp:618-634;
// TrigTable ctor, src/variants.cpp:248-263), base constant cos(2*pi/8)
// (variants.cpp:241-244).  Layout = TrigTable::constants()
// (variants.cpp:289-299): slots p = 1..nmax/4-1, then the base constant.
#pragma once

#include <cstddef>
#include <vector>

namespace amqft_b200 {

// Constant family per variant (modulation_kind, variants.cpp:42-56):
// 0 = 2cos, 1 = 2sin, 2 = 1/(2cos), 3 = 1/(2sin).
int modulation_kind(int variant);

double modulation_value(int kind, size_t index, size_t n);

// corrupt = TrigTable::corrupt_for_testing (variants.cpp:301): +1e-3 on
// every constant including the base one.
std::vector<double> trig_table(int variant, size_t nmax, bool corrupt);

}  // namespace amqft_b200
