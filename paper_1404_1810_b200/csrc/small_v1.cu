// small_v1.cu -- one-thread-per-row kernel instances for AM-QFT variant 1.
#include "gen/small_gen_v1.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace smallk {
template std::unique_ptr<FastPlan> make_small_sized<1, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_sized<1, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<1, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<1, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<1, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<1, double>(int, size_t, const void*, uint32_t, int);
}  // namespace smallk
}  // namespace amqft_b200
