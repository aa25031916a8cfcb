// fourstep.cuh -- large-N CDFT as a four-step over the fused AM-QFT kernel
// (fourstep.cu).
#pragma once

#include <memory>

#include "fast.cuh"

namespace amqft_b200 {

// fp32 fused-kernel plan for one size (nullptr if none): fast.cu.
std::unique_ptr<FastPlan> make_fast_typed_f32(int variant, size_t n, const void* tab, uint32_t nmax, int dev);

// CDFT, fp32, fast order, N = 2^20 .. 2^26.
bool fourstep_covers(const amqft_plan_desc& d);
std::unique_ptr<FastPlan> make_fourstep_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax);
OpCount fourstep_op_counts(const amqft_plan_desc& d);

}  // namespace amqft_b200
