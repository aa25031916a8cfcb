// fast_v8.cu -- fused-kernel instances for AM-QFT variant 8, CDFT rows.
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_sized<8, float, false>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_sized<8, double, false>(size_t, const void*, uint32_t, int);
// fp32 rows, fp64 arithmetic (fast.cuh f32_needs_f64_compute)
template std::unique_ptr<FastPlan> make_sized<8, double, false, float>(size_t, const void*, uint32_t, int);
// cluster four-step (N = 8192 .. 65536)
template std::unique_ptr<FastPlan> make_cluster<8, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_cluster<8, double, float>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
