// fast_v2.cu -- fused-kernel instances for AM-QFT variant 2, CDFT rows.
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_sized<2, float, false>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_sized<2, double, false>(size_t, const void*, uint32_t, int);
// cluster four-step (N = 8192 .. 65536)
template std::unique_ptr<FastPlan> make_cluster<2, float>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
