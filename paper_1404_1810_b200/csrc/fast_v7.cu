// fast_v7.cu -- fused-kernel instances for AM-QFT variant 7.
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_for_variant<7, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_for_variant<7, double>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
