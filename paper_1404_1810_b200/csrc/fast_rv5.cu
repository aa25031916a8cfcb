// fast_rv5.cu -- fused-kernel instances for AM-QFT variant 5, RDFT rows
// (two real rows per kernel row).
#include "fast_kernel.cuh"

namespace amqft_b200 {
namespace fastk {
template std::unique_ptr<FastPlan> make_sized<5, float, true>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_sized<5, double, true>(size_t, const void*, uint32_t, int);
// fp32 rows, fp64 arithmetic (fast.cuh f32_needs_f64_compute)
template std::unique_ptr<FastPlan> make_sized<5, double, true, float>(size_t, const void*, uint32_t, int);
}  // namespace fastk
}  // namespace amqft_b200
