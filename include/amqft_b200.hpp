// amqft_b200.hpp -- the reference's public C++ API (namespace amqft) served
// by the B200 library.  A caller of the reference library recompiles
// against these declarations with no source change and links
// libamqft_b200.so instead of the reference library.  The reference headers
// this replaces are /root/reference/proj/include/amqft/{signal,variants,
// elaborations,opmeter}.hpp; include/amqft/<same names> forward here, so
// `#include "amqft/variants.hpp"` keeps working.
//
// What runs where:
//   * execute(...)      -> the transform runs on the current CUDA device
//                          (exact fp64 order, bitwise the reference's CPU
//                          recursion; csrc/engine.cu).  There is no host
//                          computation of the transform and no CPU fallback.
//   * TrigSource        -> the constants the recursion consumes are taken from
//                          the caller's source on the host (value() /
//                          base_constant(), as the reference's executor does)
//                          and uploaded with the plan.
//   * layout / traits / plan description / TrigTable -> host metadata
//                          (csrc/api_host.cpp).
// Extensions (not in the reference): amqft::Plan (batched device rows,
// fp32/fp64, exact or fast order, inverse) on top of the C ABI amqft_b200.h.
//
// C++20 (as the reference: proj/CMakeLists.txt).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "amqft_b200.h"

namespace amqft {

// ------------------------------------------------------------------ layout
// signal.hpp:16-146 (reference).  Four lenses, optional time / harmonic
// parity restriction; only the non-redundant cells are stored, ascending.
enum class TransformKind { Cdft, Rdft, Dct, Dst };
enum class Domain { Temporal, Frequency };
enum class Parity { Full, Even, Odd };

// Same enumerators, same order as the reference (the numeric values cross
// the C ABI and the reference's callers index tables with them).
enum class SignalType {
  CdftFull, RdftFull,
  DctFull, DctEvenTime, DctOddTime, DctEvenHarm, DctOddHarm,
  DctOddTimeEvenHarm, DctEvenTimeOddHarm, DctOddTimeOddHarm,
  DstFull, DstEvenTime, DstOddTime, DstEvenHarm, DstOddHarm,
  DstOddTimeEvenHarm, DstEvenTimeOddHarm, DstOddTimeOddHarm,
};
inline constexpr SignalType kAllSignalTypes[] = {
    SignalType::CdftFull, SignalType::RdftFull, SignalType::DctFull,
    SignalType::DctEvenTime, SignalType::DctOddTime, SignalType::DctEvenHarm,
    SignalType::DctOddHarm, SignalType::DctOddTimeEvenHarm, SignalType::DctEvenTimeOddHarm,
    SignalType::DctOddTimeOddHarm, SignalType::DstFull, SignalType::DstEvenTime,
    SignalType::DstOddTime, SignalType::DstEvenHarm, SignalType::DstOddHarm,
    SignalType::DstOddTimeEvenHarm, SignalType::DstEvenTimeOddHarm, SignalType::DstOddTimeOddHarm,
};

TransformKind kind_of(SignalType type);
Parity time_parity(SignalType type);
Parity harmonic_parity(SignalType type);
const char* type_name(SignalType type);          // "dct[odd-n,odd-k]" style
bool is_power_of_two(std::size_t n);
std::size_t min_periodization(SignalType type);
void validate_periodization(SignalType type, std::size_t n);   // throws std::invalid_argument

// Arithmetic progression first, first + step, ... (count terms).
struct IndexRange {
  std::size_t first = 0;
  std::size_t step = 1;
  std::size_t count = 0;

  bool contains(std::size_t index) const {
    return index >= first && (index - first) % step == 0 && (index - first) / step < count;
  }
  std::size_t position_of(std::size_t index) const;   // throws unless contains(index)
  std::size_t index_at(std::size_t position) const;   // throws past the end
  std::size_t last() const { return first + step * (count - 1); }
  bool operator==(const IndexRange&) const = default;
};

IndexRange stored_range(SignalType type, std::size_t n, Domain domain);
std::vector<std::size_t> stored_indices(SignalType type, std::size_t n, Domain domain);
std::size_t storage_position(SignalType type, std::size_t n, Domain domain, std::size_t index);
std::size_t cell_count(SignalType type, std::size_t n);   // two per slot for CdftFull

// A signal: type + periodization + domain + packed cells (CdftFull
// interleaved re/im; the RdftFull spectrum packs Re S(j), j <= n/2, then
// Im S(j) for j > n/2).
struct SignalBuffer {
  SignalType type = SignalType::RdftFull;
  std::size_t periodization = 0;
  Domain domain = Domain::Temporal;
  std::vector<double> cells;

  static SignalBuffer zeros(SignalType type, std::size_t n, Domain domain);
  IndexRange range() const { return stored_range(type, periodization, domain); }
  double at(std::size_t index) const;       // real-valued types
  double& at(std::size_t index);
  double re(std::size_t index) const;       // CdftFull
  double& re(std::size_t index);
  double im(std::size_t index) const;
  double& im(std::size_t index);
};

// ----------------------------------------------------------- op accounting
// opmeter.hpp:13-29: adds (incl. subtractions), muls, and multiplications by
// 0.5 counted apart as binary translations.  Filled from the executed
// device schedule (identical to the reference meter).
struct OpMeter {
  std::uint64_t adds = 0;
  std::uint64_t muls = 0;
  std::uint64_t binary_translations = 0;

  std::uint64_t flops_case_a() const { return adds + muls; }
  std::uint64_t flops_case_b() const { return adds + muls + binary_translations; }
  OpMeter& operator+=(const OpMeter& o) {
    adds += o.adds;
    muls += o.muls;
    binary_translations += o.binary_translations;
    return *this;
  }
  friend OpMeter operator+(OpMeter a, const OpMeter& b) { return a += b; }
  bool operator==(const OpMeter&) const = default;
};

// ------------------------------------------------------------ elaborations
// elaborations.hpp:25-107: the elaboration identities and the constant
// plugin.  (The single-step appliers transform_forward / decompose_forward /
// ... are the reference executor's internals; the device runs whole
// transforms, so they are not part of this API.)
enum class ElaborationId {
  SplitComplex, SplitReal, HalveEvenHarmonics, HalveEvenTime,
  SplitHarmonicParity, SplitTimeParity,
  AmConvert1, AmConvert2, AmConvert3, AmConvert4,
  AmConvert5, AmConvert6, AmConvert7, AmConvert8,
};
inline constexpr ElaborationId kAllElaborations[] = {
    ElaborationId::SplitComplex, ElaborationId::SplitReal, ElaborationId::HalveEvenHarmonics,
    ElaborationId::HalveEvenTime, ElaborationId::SplitHarmonicParity, ElaborationId::SplitTimeParity,
    ElaborationId::AmConvert1, ElaborationId::AmConvert2, ElaborationId::AmConvert3,
    ElaborationId::AmConvert4, ElaborationId::AmConvert5, ElaborationId::AmConvert6,
    ElaborationId::AmConvert7, ElaborationId::AmConvert8,
};
const char* elaboration_name(ElaborationId id);
bool is_decomposition(ElaborationId id);
bool is_am_conversion(ElaborationId id);

enum class TrigKind { TwoCos, TwoSin, InvTwoCos, InvTwoSin };
const char* trig_kind_name(TrigKind kind);

// f(2 pi index / periodization), long double, rounded once (bitwise the
// reference's value, so tables and on-the-fly evaluation agree).
double modulation_value(TrigKind kind, std::size_t index, std::size_t periodization);

// The constant plugin (elaborations.hpp:90-98).  execute() asks the source
// for every slot of one table at the transform's periodization plus the
// base constant, checks that every smaller level's request would return the
// same bits (it does for TrigTable and OnTheFlyTrig), and uploads it.
class TrigSource {
 public:
  virtual ~TrigSource() = default;
  virtual double value(TrigKind kind, std::size_t index, std::size_t periodization) const = 0;
  virtual double base_constant() const = 0;
};

class OnTheFlyTrig final : public TrigSource {
 public:
  double value(TrigKind kind, std::size_t index, std::size_t periodization) const override {
    return modulation_value(kind, index, periodization);
  }
  double base_constant() const override;
};

// ---------------------------------------------------------------- variants
// variants.hpp:25-141.
enum class VariantId : int { V1 = 1, V2, V3, V4, V5, V6, V7, V8 };
inline constexpr VariantId kAllVariants[] = {VariantId::V1, VariantId::V2, VariantId::V3, VariantId::V4,
                                             VariantId::V5, VariantId::V6, VariantId::V7, VariantId::V8};

int variant_number(VariantId v);
VariantId variant_from_number(int n);         // throws outside 1..8
bool time_major(VariantId v);                 // 1, 4, 5, 8
ElaborationId am_conversion(VariantId v);
TrigKind modulation_kind(VariantId v);
bool sine_modulated(VariantId v);             // 5..8
bool uses_binary_translations(VariantId v);   // 1, 3, 5, 7

enum class FunctionId {
  Cdft, Rdft, Dct, Dst, DctOddTime, DstOddTime, DctOddHarm, DstOddHarm, DctOddOdd, DstOddOdd,
};
const char* function_name(FunctionId f);
const char* kind_name(TransformKind kind);
SignalType full_type_of(TransformKind kind);
FunctionId function_for(TransformKind kind);
SignalType operand_type(FunctionId f);

// The wiring the device plan compiler expands (description only).
struct RecursionCall {
  FunctionId target;
  std::size_t size_divisor;   // child periodization = n / size_divisor
  bool operator==(const RecursionCall&) const = default;
};
struct FunctionPlan {
  FunctionId id;
  SignalType operand;
  std::size_t base_size;
  std::vector<ElaborationId> forward;
  std::vector<RecursionCall> calls;   // [0] reduced child, [1] odd child
  bool operator==(const FunctionPlan&) const = default;
};
struct VariantPlan {
  VariantId variant;
  std::vector<FunctionPlan> functions;
  bool has_function(FunctionId f) const;
  const FunctionPlan& function(FunctionId f) const;   // throws if not wired
};
VariantPlan build_plan(VariantId v);

enum class TrigMode { Precomputed, OnTheFly };

// The variant's constant table (variants.hpp:111-141): slots f(2 pi p / max)
// for p in [1, max/4) plus cos(2 pi / 8); smaller periodizations scale the
// slot index.  Host-side; execute() uploads what it returns.
class TrigTable final : public TrigSource {
 public:
  TrigTable(VariantId v, std::size_t max_periodization, TrigMode mode = TrigMode::Precomputed);

  double value(TrigKind kind, std::size_t index, std::size_t periodization) const override;
  double base_constant() const override;

  VariantId variant() const { return variant_; }
  TrigKind kind() const { return kind_; }
  TrigMode mode() const { return mode_; }
  std::size_t max_periodization() const { return max_n_; }
  std::size_t constant_count() const;          // max/4, the base constant included
  std::vector<double> constants() const;       // slots ascending, base constant last
  void corrupt_for_testing();                  // +1e-3 on every constant

 private:
  VariantId variant_;
  TrigKind kind_;
  TrigMode mode_;
  std::size_t max_n_;
  std::vector<double> slots_;
  double base_;
  double corruption_ = 0.0;
};

// --------------------------------------------------------------- execution
// variants.hpp:148-153.  Same validation and exceptions as the reference
// (std::invalid_argument); device failures surface as std::runtime_error.
SignalBuffer execute(VariantId v, FunctionId f, const SignalBuffer& input, const TrigSource& trig,
                     OpMeter* meter = nullptr);
SignalBuffer execute(VariantId v, const SignalBuffer& input, const TrigSource& trig,
                     OpMeter* meter = nullptr);

// ---------------------------------------------------------------- extensions

namespace detail {
inline void check(amqft_status s) {
  if (s == AMQFT_OK) return;
  const std::string msg = amqft_last_error();
  if (s == AMQFT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// Swap-trick inverse CDFT of one frequency-domain CdftFull signal (exact
// fp64 order): x = swap(DFT(swap(X))) / n.
SignalBuffer execute_inverse(VariantId v, const SignalBuffer& spectrum);

// Batched device execution: d_in / d_out hold `batch` rows of the
// function's operand (row-major, cell_count cells each); fp32 or fp64; exact
// or fast order.
class Plan {
 public:
  Plan(VariantId v, FunctionId f, std::size_t n, std::size_t batch, amqft_dtype dtype = AMQFT_F32,
       amqft_order order = AMQFT_ORDER_FAST, int device = 0) {
    amqft_plan_desc d{};
    d.variant = static_cast<int>(v);
    d.function = static_cast<int>(f);
    d.n = n;
    d.batch = batch;
    d.dtype = dtype;
    d.trig_mode = AMQFT_TRIG_TABLE;
    d.order = order;
    d.device = device;
    detail::check(amqft_plan_create(&p_, &d));
  }
  ~Plan() { amqft_plan_destroy(p_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  void forward(const void* d_in, void* d_out, void* stream = nullptr) {
    detail::check(amqft_exec_forward(p_, d_in, d_out, stream));
  }
  void inverse(const void* d_in, void* d_out, void* stream = nullptr) {
    detail::check(amqft_exec_inverse(p_, d_in, d_out, stream));
  }
  std::size_t cells() const { return amqft_plan_cells(p_); }
  OpMeter op_counts() const {
    std::uint64_t m[3] = {0, 0, 0};
    detail::check(amqft_plan_op_counts(p_, m));
    return OpMeter{m[0], m[1], m[2]};
  }

 private:
  amqft_plan p_ = nullptr;
};

}  // namespace amqft
