// amqft_b200.hpp -- the reference's C++ API (namespace amqft) on top of the
// B200 C ABI (amqft_b200.h).  A caller of the reference library
// (/root/reference/proj/include/amqft/{signal,variants}.hpp) recompiles
// against this header unchanged for the transform path:
//
//   SignalBuffer execute(VariantId, FunctionId, const SignalBuffer&,
//                        const TrigSource&, OpMeter* = nullptr)   // variants.hpp:148-153
//   SignalBuffer execute(VariantId, const SignalBuffer&, ...)      // type-deducing overload
//   TrigTable(VariantId, std::size_t max_periodization, TrigMode)  // variants.hpp:111-141
//
// plus batched/inverse extensions (execute_batch, execute_inverse).  The
// transform runs on the current CUDA device (exact fp64 order: bitwise the
// reference); there is no host computation.  Errors surface as
// std::invalid_argument (AMQFT_EINVAL, the reference's convention) or
// std::runtime_error (device errors).
//
// Header-only; link with libamqft_b200.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "amqft_b200.h"

namespace amqft {

enum class TransformKind { Cdft, Rdft, Dct, Dst };            // signal.hpp:18
enum class Domain { Temporal, Frequency };                     // signal.hpp:20
enum class SignalType {                                        // signal.hpp:28-48
  CdftFull, RdftFull, DctFull, DctEvenTime, DctOddTime, DctEvenHarm, DctOddHarm,
  DctOddTimeEvenHarm, DctEvenTimeOddHarm, DctOddTimeOddHarm, DstFull, DstEvenTime,
  DstOddTime, DstEvenHarm, DstOddHarm, DstOddTimeEvenHarm, DstEvenTimeOddHarm,
  DstOddTimeOddHarm,
};
enum class VariantId : int { V1 = 1, V2, V3, V4, V5, V6, V7, V8 };  // variants.hpp:25
enum class FunctionId {                                        // variants.hpp:55-66
  Cdft, Rdft, Dct, Dst, DctOddTime, DstOddTime, DctOddHarm, DstOddHarm, DctOddOdd, DstOddOdd,
};
enum class TrigMode { Precomputed, OnTheFly };                 // variants.hpp:108

struct OpMeter {                                               // opmeter.hpp:13-29
  std::uint64_t adds = 0, muls = 0, binary_translations = 0;
  std::uint64_t flops_case_a() const { return adds + muls; }
  std::uint64_t flops_case_b() const { return adds + muls + binary_translations; }
};

inline SignalType operand_type(FunctionId f) {                 // variants.cpp:132-156
  static const SignalType t[] = {
      SignalType::CdftFull, SignalType::RdftFull, SignalType::DctFull, SignalType::DstFull,
      SignalType::DctOddTime, SignalType::DstOddTime, SignalType::DctOddHarm,
      SignalType::DstOddHarm, SignalType::DctOddTimeOddHarm, SignalType::DstOddTimeOddHarm};
  return t[static_cast<int>(f)];
}

// SignalBuffer (signal.hpp:125-146): type + periodization + domain + cells.
struct SignalBuffer {
  SignalType type = SignalType::RdftFull;
  std::size_t periodization = 0;
  Domain domain = Domain::Temporal;
  std::vector<double> cells;
};

// The TrigSource plugin the reference threads through execute
// (elaborations.hpp:90-107).  The device path consumes the table
// description (variant family, max periodization, mode), not virtual calls.
class TrigSource {
 public:
  virtual ~TrigSource() = default;
  virtual std::size_t max_periodization() const = 0;
  virtual TrigMode mode() const = 0;
  virtual bool corrupted() const { return false; }
};

class TrigTable final : public TrigSource {                    // variants.hpp:111-141
 public:
  TrigTable(VariantId v, std::size_t max_periodization, TrigMode mode = TrigMode::Precomputed)
      : v_(v), max_n_(max_periodization), mode_(mode) {
    if (max_n_ < 8 || (max_n_ & (max_n_ - 1)) != 0)
      throw std::invalid_argument("constant table needs a power-of-two max periodization >= 8");
  }
  std::size_t max_periodization() const override { return max_n_; }
  TrigMode mode() const override { return mode_; }
  bool corrupted() const override { return corrupt_; }
  VariantId variant() const { return v_; }
  std::size_t constant_count() const { return max_n_ / 4; }
  void corrupt_for_testing() { corrupt_ = true; }              // variants.cpp:301

 private:
  VariantId v_;
  std::size_t max_n_;
  TrigMode mode_;
  bool corrupt_ = false;
};

namespace detail {
inline void check(amqft_status s) {
  if (s == AMQFT_OK) return;
  const std::string msg = amqft_last_error();
  if (s == AMQFT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// amqft::execute(v, f, input, trig, meter) -- variants.cpp:404-422.
inline SignalBuffer execute(VariantId v, FunctionId f, const SignalBuffer& input,
                            const TrigSource& trig, OpMeter* meter = nullptr) {
  if (input.domain != Domain::Temporal)
    throw std::invalid_argument("execute consumes a temporal signal");
  if (input.type != operand_type(f))
    throw std::invalid_argument("operand type does not match the function");
  SignalBuffer out;
  out.type = input.type;
  out.periodization = input.periodization;
  out.domain = Domain::Frequency;
  out.cells.resize(input.cells.size());
  std::uint64_t m3[3] = {0, 0, 0};
  detail::check(amqft_execute_host(static_cast<int>(v), static_cast<int>(f), input.periodization,
                                   input.cells.data(), out.cells.data(),
                                   trig.mode() == TrigMode::OnTheFly ? AMQFT_TRIG_ONTHEFLY
                                                                     : AMQFT_TRIG_TABLE,
                                   trig.max_periodization(), trig.corrupted() ? 1 : 0, m3));
  if (meter) {
    meter->adds = m3[0];
    meter->muls = m3[1];
    meter->binary_translations = m3[2];
  }
  return out;
}

// Type-deducing overload (variants.cpp:424-442).
inline SignalBuffer execute(VariantId v, const SignalBuffer& input, const TrigSource& trig,
                            OpMeter* meter = nullptr) {
  for (int f = 0; f < 10; ++f)
    if (operand_type(static_cast<FunctionId>(f)) == input.type) {
      if ((f == 4 || f == 5) && !(v == VariantId::V1 || v == VariantId::V4 || v == VariantId::V5 ||
                                  v == VariantId::V8))
        continue;
      if ((f == 6 || f == 7) && (v == VariantId::V1 || v == VariantId::V4 || v == VariantId::V5 ||
                                 v == VariantId::V8))
        continue;
      return execute(v, static_cast<FunctionId>(f), input, trig, meter);
    }
  throw std::invalid_argument("no function consumes this signal type");
}

// ---- Extensions (not in the reference).

// Batched device execution: d_in / d_out hold `rows` signals of the
// function's operand, row-major; fp32 or fp64; exact or fast order.
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

 private:
  amqft_plan p_ = nullptr;
};

}  // namespace amqft
