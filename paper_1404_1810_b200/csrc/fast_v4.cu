// fast_v4.cu -- fused-kernel instances for AM-QFT variant 4, CDFT rows.
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_sized<4, float, false>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_sized<4, double, false>(size_t, const void*, uint32_t, int);
// cluster four-step (N = 8192 .. 65536)
template std::unique_ptr<FastPlan> make_cluster<4, float>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
