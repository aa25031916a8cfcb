// small_v4.cu -- one-thread-per-row kernel instances for AM-QFT variant 4.
#include "gen/small_gen_v4.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace smallk {
template std::unique_ptr<FastPlan> make_small_sized<4, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_sized<4, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<4, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<4, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<4, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<4, double>(int, size_t, const void*, uint32_t, int);
}  // namespace smallk
}  // namespace amqft_b200
