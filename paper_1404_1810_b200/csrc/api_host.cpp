// api_host.cpp -- host side of the reference C++ API (include/amqft_b200.hpp):
// signal layout metadata, variant traits, the wiring description, the
// TrigTable constant plugin, and amqft::execute, which validates like the
// reference, collects the constants from the caller's TrigSource and runs
// the transform on the device through the C ABI (engine.cu).  No transform
// arithmetic happens here.
//
// Reference behaviour followed (file:line under /root/reference/proj):
//   layout            src/signal.cpp:18-268 (stored index sets restated as
//                     a descriptor table)
//   traits / names    src/variants.cpp:24-156, src/elaborations.cpp:535-616
//   wiring            src/variants.cpp:173-234
//   TrigTable         src/variants.cpp:236-301, modulation_value
//                     src/elaborations.cpp:618-639
//   execute           src/variants.cpp:404-442
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amqft_b200.hpp"
#include "trig.hpp"

namespace amqft {

namespace {

[[noreturn]] void bad(const std::string& what) { throw std::invalid_argument(what); }

// One arithmetic progression as a function of the periodization:
// first, step, count = n / div + add.
struct Prog {
  std::size_t first, step, div;
  int add;
  IndexRange at(std::size_t n) const {
    return IndexRange{first, step, static_cast<std::size_t>(static_cast<long long>(n / div) + add)};
  }
};

struct TypeDesc {
  TransformKind kind;
  Parity tp, hp;
  std::size_t min_n;
  Prog temporal, frequency;
};

constexpr Parity F = Parity::Full, E = Parity::Even, O = Parity::Odd;
constexpr TransformKind KC = TransformKind::Cdft, KR = TransformKind::Rdft, KD = TransformKind::Dct,
                        KS = TransformKind::Dst;

// Indexed by SignalType.  Dct lens keeps both endpoints (0 and n/2), Dst
// lens neither; a parity restriction halves the index set (step 2) and the
// single-parity types live on a quarter period, the doubly restricted ones
// on an eighth.
const TypeDesc kTypes[] = {
    {KC, F, F, 2, {0, 1, 1, 0}, {0, 1, 1, 0}},     // CdftFull
    {KR, F, F, 2, {0, 1, 1, 0}, {0, 1, 1, 0}},     // RdftFull
    {KD, F, F, 2, {0, 1, 2, 1}, {0, 1, 2, 1}},     // DctFull
    {KD, E, F, 4, {0, 2, 4, 1}, {0, 1, 4, 1}},     // DctEvenTime
    {KD, O, F, 4, {1, 2, 4, 0}, {0, 1, 4, 0}},     // DctOddTime
    {KD, F, E, 4, {0, 1, 4, 1}, {0, 2, 4, 1}},     // DctEvenHarm
    {KD, F, O, 4, {0, 1, 4, 0}, {1, 2, 4, 0}},     // DctOddHarm
    {KD, O, E, 8, {1, 2, 8, 0}, {0, 2, 8, 0}},     // DctOddTimeEvenHarm
    {KD, E, O, 8, {0, 2, 8, 0}, {1, 2, 8, 0}},     // DctEvenTimeOddHarm
    {KD, O, O, 8, {1, 2, 8, 0}, {1, 2, 8, 0}},     // DctOddTimeOddHarm
    {KS, F, F, 4, {1, 1, 2, -1}, {1, 1, 2, -1}},   // DstFull
    {KS, E, F, 8, {2, 2, 4, -1}, {1, 1, 4, -1}},   // DstEvenTime
    {KS, O, F, 4, {1, 2, 4, 0}, {1, 1, 4, 0}},     // DstOddTime
    {KS, F, E, 8, {1, 1, 4, -1}, {2, 2, 4, -1}},   // DstEvenHarm
    {KS, F, O, 4, {1, 1, 4, 0}, {1, 2, 4, 0}},     // DstOddHarm
    {KS, O, E, 8, {1, 2, 8, 0}, {2, 2, 8, 0}},     // DstOddTimeEvenHarm
    {KS, E, O, 8, {2, 2, 8, 0}, {1, 2, 8, 0}},     // DstEvenTimeOddHarm
    {KS, O, O, 8, {1, 2, 8, 0}, {1, 2, 8, 0}},     // DstOddTimeOddHarm
};
constexpr int kNumTypes = sizeof(kTypes) / sizeof(kTypes[0]);

const TypeDesc& desc(SignalType t) {
  const int i = static_cast<int>(t);
  if (i < 0 || i >= kNumTypes) bad("unknown signal type");
  return kTypes[i];
}

// "dct[odd-n,even-k]" style names, built once.
const char* const kTypeNames[] = {
    "cdft", "rdft",
    "dct", "dct[even-n]", "dct[odd-n]", "dct[even-k]", "dct[odd-k]",
    "dct[odd-n,even-k]", "dct[even-n,odd-k]", "dct[odd-n,odd-k]",
    "dst", "dst[even-n]", "dst[odd-n]", "dst[even-k]", "dst[odd-k]",
    "dst[odd-n,even-k]", "dst[even-n,odd-k]", "dst[odd-n,odd-k]",
};

}  // namespace

// ---------------------------------------------------------------- layout

TransformKind kind_of(SignalType type) { return desc(type).kind; }
Parity time_parity(SignalType type) { return desc(type).tp; }
Parity harmonic_parity(SignalType type) { return desc(type).hp; }

const char* type_name(SignalType type) {
  const int i = static_cast<int>(type);
  return (i >= 0 && i < kNumTypes) ? kTypeNames[i] : "?";
}

bool is_power_of_two(std::size_t n) { return n && !(n & (n - 1)); }

std::size_t min_periodization(SignalType type) { return desc(type).min_n; }

void validate_periodization(SignalType type, std::size_t n) {
  if (!is_power_of_two(n)) bad("periodization " + std::to_string(n) + " is not a power of two");
  if (n < desc(type).min_n)
    bad("periodization " + std::to_string(n) + " is below the minimum " + std::to_string(desc(type).min_n) +
        " for " + type_name(type));
}

std::size_t IndexRange::position_of(std::size_t index) const {
  if (!contains(index)) bad("signal index " + std::to_string(index) + " is not stored");
  return (index - first) / step;
}

std::size_t IndexRange::index_at(std::size_t position) const {
  if (position >= count) bad("storage position " + std::to_string(position) + " out of range");
  return first + position * step;
}

IndexRange stored_range(SignalType type, std::size_t n, Domain domain) {
  validate_periodization(type, n);
  const TypeDesc& d = desc(type);
  return (domain == Domain::Temporal ? d.temporal : d.frequency).at(n);
}

std::vector<std::size_t> stored_indices(SignalType type, std::size_t n, Domain domain) {
  const IndexRange r = stored_range(type, n, domain);
  std::vector<std::size_t> out(r.count);
  for (std::size_t p = 0; p < r.count; ++p) out[p] = r.first + p * r.step;
  return out;
}

std::size_t storage_position(SignalType type, std::size_t n, Domain domain, std::size_t index) {
  return stored_range(type, n, domain).position_of(index);
}

std::size_t cell_count(SignalType type, std::size_t n) {
  const std::size_t slots = stored_range(type, n, Domain::Temporal).count;
  return type == SignalType::CdftFull ? slots * 2 : slots;
}

SignalBuffer SignalBuffer::zeros(SignalType type, std::size_t n, Domain domain) {
  SignalBuffer b;
  b.type = type;
  b.periodization = n;
  b.domain = domain;
  b.cells.assign(cell_count(type, n), 0.0);   // validates n
  return b;
}

namespace {
std::size_t real_slot(const SignalBuffer& b, std::size_t index) {
  if (b.type == SignalType::CdftFull) bad("at() is for real-valued signal types; use re()/im()");
  return b.range().position_of(index);
}
std::size_t complex_slot(const SignalBuffer& b, std::size_t index, std::size_t part) {
  if (b.type != SignalType::CdftFull) bad(part ? "im() is for the complex type" : "re() is for the complex type");
  return 2 * b.range().position_of(index) + part;
}
}  // namespace

double SignalBuffer::at(std::size_t index) const { return cells[real_slot(*this, index)]; }
double& SignalBuffer::at(std::size_t index) { return cells[real_slot(*this, index)]; }
double SignalBuffer::re(std::size_t index) const { return cells[complex_slot(*this, index, 0)]; }
double& SignalBuffer::re(std::size_t index) { return cells[complex_slot(*this, index, 0)]; }
double SignalBuffer::im(std::size_t index) const { return cells[complex_slot(*this, index, 1)]; }
double& SignalBuffer::im(std::size_t index) { return cells[complex_slot(*this, index, 1)]; }

// ---------------------------------------------------------- elaborations

const char* elaboration_name(ElaborationId id) {
  static const char* const names[] = {
      "split-complex", "split-real", "halve-even-harmonics", "halve-even-time",
      "split-harmonic-parity", "split-time-parity", "am-convert-1", "am-convert-2",
      "am-convert-3", "am-convert-4", "am-convert-5", "am-convert-6", "am-convert-7", "am-convert-8"};
  const int i = static_cast<int>(id);
  return (i >= 0 && i < 14) ? names[i] : "?";
}

bool is_decomposition(ElaborationId id) {
  return id == ElaborationId::SplitComplex || id == ElaborationId::SplitReal ||
         id == ElaborationId::SplitHarmonicParity || id == ElaborationId::SplitTimeParity;
}

bool is_am_conversion(ElaborationId id) { return id >= ElaborationId::AmConvert1; }

const char* trig_kind_name(TrigKind kind) {
  switch (kind) {
    case TrigKind::TwoCos: return "2cos";
    case TrigKind::TwoSin: return "2sin";
    case TrigKind::InvTwoCos: return "1/(2cos)";
    case TrigKind::InvTwoSin: return "1/(2sin)";
  }
  return "?";
}

double modulation_value(TrigKind kind, std::size_t index, std::size_t periodization) {
  return amqft_b200::modulation_value(static_cast<int>(kind), index, periodization);
}

double OnTheFlyTrig::base_constant() const {
  // the base slot of any table: cos(2 pi / 8) in long double, rounded once
  return amqft_b200::trig_table(1, 8, false).back();
}

// -------------------------------------------------------------- variants

int variant_number(VariantId v) { return static_cast<int>(v); }

VariantId variant_from_number(int n) {
  if (n < 1 || n > 8) bad("variant number must be in 1..8");
  return static_cast<VariantId>(n);
}

bool time_major(VariantId v) {
  switch (variant_number(v)) {
    case 1: case 4: case 5: case 8: return true;
    default: return false;
  }
}

ElaborationId am_conversion(VariantId v) {
  return static_cast<ElaborationId>(static_cast<int>(ElaborationId::AmConvert1) + variant_number(v) - 1);
}

TrigKind modulation_kind(VariantId v) {
  return static_cast<TrigKind>(amqft_b200::modulation_kind(variant_number(v)));
}

bool sine_modulated(VariantId v) { return variant_number(v) > 4; }
bool uses_binary_translations(VariantId v) { return (variant_number(v) & 1) != 0; }

// every function is named after its operand type ("dct[odd-n]", ...)
const char* function_name(FunctionId f) { return type_name(operand_type(f)); }

const char* kind_name(TransformKind kind) { return type_name(full_type_of(kind)); }

SignalType full_type_of(TransformKind kind) {
  switch (kind) {
    case TransformKind::Cdft: return SignalType::CdftFull;
    case TransformKind::Rdft: return SignalType::RdftFull;
    case TransformKind::Dct: return SignalType::DctFull;
    case TransformKind::Dst: return SignalType::DstFull;
  }
  bad("unknown transform kind");
}

FunctionId function_for(TransformKind kind) {
  switch (kind) {
    case TransformKind::Cdft: return FunctionId::Cdft;
    case TransformKind::Rdft: return FunctionId::Rdft;
    case TransformKind::Dct: return FunctionId::Dct;
    case TransformKind::Dst: return FunctionId::Dst;
  }
  bad("unknown transform kind");
}

SignalType operand_type(FunctionId f) {
  static const SignalType ops[] = {
      SignalType::CdftFull, SignalType::RdftFull, SignalType::DctFull, SignalType::DstFull,
      SignalType::DctOddTime, SignalType::DstOddTime, SignalType::DctOddHarm, SignalType::DstOddHarm,
      SignalType::DctOddTimeOddHarm, SignalType::DstOddTimeOddHarm};
  const int i = static_cast<int>(f);
  if (i < 0 || i >= 10) bad("unknown function");
  return ops[i];
}

bool VariantPlan::has_function(FunctionId f) const {
  return std::any_of(functions.begin(), functions.end(), [f](const FunctionPlan& p) { return p.id == f; });
}

const FunctionPlan& VariantPlan::function(FunctionId f) const {
  for (const FunctionPlan& p : functions)
    if (p.id == f) return p;
  bad(std::string("variant ") + std::to_string(variant_number(variant)) + " does not wire " + function_name(f));
}

VariantPlan build_plan(VariantId v) {
  using EID = ElaborationId;
  using FID = FunctionId;
  const bool tm = time_major(v), sine = sine_modulated(v);
  // major axis (time for 1,4,5,8) above the AM stage, the other one below it
  const EID split = tm ? EID::SplitTimeParity : EID::SplitHarmonicParity;
  const EID halve = tm ? EID::HalveEvenTime : EID::HalveEvenHarmonics;
  const EID split2 = tm ? EID::SplitHarmonicParity : EID::SplitTimeParity;
  const EID halve2 = tm ? EID::HalveEvenHarmonics : EID::HalveEvenTime;
  const FID oddC = tm ? FID::DctOddTime : FID::DctOddHarm;
  const FID oddS = tm ? FID::DstOddTime : FID::DstOddHarm;
  auto fp = [](FID id, std::size_t base, std::vector<EID> fwd, std::vector<RecursionCall> calls) {
    return FunctionPlan{id, operand_type(id), base, std::move(fwd), std::move(calls)};
  };
  VariantPlan P;
  P.variant = v;
  P.functions.push_back(fp(FID::Cdft, 2, {EID::SplitComplex}, {{FID::Rdft, 1}, {FID::Rdft, 1}}));
  P.functions.push_back(fp(FID::Rdft, 2, {EID::SplitReal}, {{FID::Dct, 1}, {FID::Dst, 1}}));
  P.functions.push_back(fp(FID::Dct, 2, {split, halve}, {{FID::Dct, 2}, {oddC, 1}}));
  P.functions.push_back(fp(FID::Dst, 4, {split, halve}, {{FID::Dst, 2}, {oddS, 1}}));
  P.functions.push_back(fp(oddC, 4, {split2, halve2}, {{oddC, 2}, {FID::DctOddOdd, 1}}));
  P.functions.push_back(fp(oddS, 4, {split2, halve2}, {{oddS, 2}, {FID::DstOddOdd, 1}}));
  // the AM stage: sine modulation (5-8) hands the child to the other lens
  const std::vector<EID> am_stage = {am_conversion(v), halve2, split2, halve2};
  P.functions.push_back(fp(FID::DctOddOdd, 8, am_stage,
                           {{sine ? oddS : oddC, 4}, {sine ? FID::DstOddOdd : FID::DctOddOdd, 2}}));
  P.functions.push_back(fp(FID::DstOddOdd, 8, am_stage,
                           {{sine ? oddC : oddS, 4}, {sine ? FID::DctOddOdd : FID::DstOddOdd, 2}}));
  return P;
}

// ------------------------------------------------------------- TrigTable

TrigTable::TrigTable(VariantId v, std::size_t max_periodization, TrigMode mode)
    : variant_(v), kind_(modulation_kind(v)), mode_(mode), max_n_(max_periodization), base_(0.0) {
  if (!is_power_of_two(max_n_) || max_n_ < 8) bad("constant table needs a power-of-two max periodization >= 8");
  std::vector<double> t = amqft_b200::trig_table(variant_number(v), max_n_, false);   // slots + base
  base_ = t.back();
  if (mode_ == TrigMode::Precomputed) {
    t.pop_back();
    slots_ = std::move(t);
  }
}

double TrigTable::value(TrigKind kind, std::size_t index, std::size_t periodization) const {
  if (kind != kind_)
    bad(std::string("this table holds ") + trig_kind_name(kind_) + " constants, not " + trig_kind_name(kind));
  if (!is_power_of_two(periodization) || periodization > max_n_) bad("periodization outside the table's range");
  if (index < 1 || index >= periodization / 4)
    bad("constant index " + std::to_string(index) + " outside [1, periodization/4)");
  if (mode_ == TrigMode::OnTheFly) return modulation_value(kind_, index, periodization) + corruption_;
  return slots_[index * (max_n_ / periodization) - 1] + corruption_;
}

double TrigTable::base_constant() const { return base_ + corruption_; }

std::size_t TrigTable::constant_count() const { return max_n_ / 4; }

std::vector<double> TrigTable::constants() const {
  std::vector<double> out(max_n_ / 4);
  for (std::size_t p = 1; p < max_n_ / 4; ++p)
    out[p - 1] = (mode_ == TrigMode::Precomputed ? slots_[p - 1] : modulation_value(kind_, p, max_n_)) + corruption_;
  out.back() = base_constant();
  return out;
}

void TrigTable::corrupt_for_testing() { corruption_ = 1e-3; }

// -------------------------------------------------------------- execute

namespace {

// The constants a transform of periodization n consumes, as one table at
// Nmax = max(n, 8) (TrigTable::constants layout).  The reference executor
// asks the source for value(kind, idx, m) at every AM node m <= n (odd idx
// < m/4) and for base_constant() at the OddOdd(8) leaves; the device reads
// slot idx * (n / m) of the one table, so every smaller level's request is
// checked to return the same bits (true for TrigTable and OnTheFlyTrig:
// the reference's level sharing).
std::vector<double> collect_constants(VariantId v, std::size_t n, const TrigSource& trig) {
  const std::size_t nmax = std::max<std::size_t>(n, 8);
  const TrigKind kind = modulation_kind(v);
  std::vector<double> tab(nmax / 4, 0.0);
  if (n >= 16) {   // AM nodes exist from periodization 16 on
    for (std::size_t p = 1; p < nmax / 4; ++p) tab[p - 1] = trig.value(kind, p, nmax);
    for (std::size_t m = nmax / 2; m >= 16; m /= 2)
      for (std::size_t idx = 1; idx < m / 4; idx += 2) {
        const double a = trig.value(kind, idx, m), b = tab[idx * (nmax / m) - 1];
        if (std::memcmp(&a, &b, sizeof a) != 0)
          bad("TrigSource is not level-invariant (value(kind, i, m) != value(kind, i*n/m, n)); "
              "the device plan holds one constant table per transform");
      }
  }
  tab.back() = trig.base_constant();
  return tab;
}

}  // namespace

SignalBuffer execute(VariantId v, FunctionId f, const SignalBuffer& input, const TrigSource& trig,
                     OpMeter* meter) {
  const VariantPlan plan = build_plan(variant_from_number(variant_number(v)));
  const FunctionPlan& fp = plan.function(f);   // throws if not wired
  if (input.domain != Domain::Temporal) bad("execute consumes a temporal signal");
  if (input.type != fp.operand)
    bad(std::string(function_name(f)) + " expects a " + type_name(fp.operand) + " operand, got " +
        type_name(input.type));
  const std::size_t n = input.periodization;
  if (!is_power_of_two(n) || n < fp.base_size)
    bad("periodization must be a power of two >= " + std::to_string(fp.base_size) + " for " + function_name(f));
  if (input.cells.size() != cell_count(input.type, n)) bad("cell count does not match the signal type");
  const std::vector<double> tab = collect_constants(v, n, trig);
  SignalBuffer out;
  out.type = input.type;
  out.periodization = n;
  out.domain = Domain::Frequency;
  out.cells.resize(input.cells.size());
  std::uint64_t m3[3] = {0, 0, 0};
  detail::check(amqft_execute_host_constants(variant_number(v), static_cast<int>(f), n, input.cells.data(),
                                             out.cells.data(), tab.data(), tab.size(), m3));
  if (meter) *meter += OpMeter{m3[0], m3[1], m3[2]};
  return out;
}

SignalBuffer execute(VariantId v, const SignalBuffer& input, const TrigSource& trig, OpMeter* meter) {
  for (int f = 0; f < 10; ++f)   // the first function whose operand matches
    if (operand_type(static_cast<FunctionId>(f)) == input.type)
      return execute(v, static_cast<FunctionId>(f), input, trig, meter);
  bad(std::string("no function consumes ") + type_name(input.type));
}

SignalBuffer execute_inverse(VariantId v, const SignalBuffer& spectrum) {
  if (spectrum.type != SignalType::CdftFull || spectrum.domain != Domain::Frequency)
    bad("execute_inverse takes a frequency-domain cdft signal");
  const std::size_t n = spectrum.periodization;
  if (!is_power_of_two(n) || spectrum.cells.size() != 2 * n) bad("cdft spectrum of a power-of-two periodization expected");
  SignalBuffer out = spectrum;
  out.domain = Domain::Temporal;
  detail::check(amqft_execute_host_inverse(variant_number(v), n, spectrum.cells.data(), out.cells.data()));
  return out;
}

}  // namespace amqft
