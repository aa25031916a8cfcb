// fast_v2.cu -- fused-kernel instances for AM-QFT variant 2.
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_for_variant<2, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_for_variant<2, double>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
