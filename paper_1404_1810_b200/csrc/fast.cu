// fast.cu -- fused fast-path kernels (placeholder until the fused CDFT
// kernel lands; requests fall through to the generic schedule kernels).
#include "fast.cuh"

namespace amqft_b200 {

std::unique_ptr<FastPlan> make_fast_plan(const amqft_plan_desc&, const void*, uint32_t) {
  return nullptr;
}

OpCount fast_op_counts(const amqft_plan_desc& d) {
  (void)d;
  return OpCount{};
}

}  // namespace amqft_b200
