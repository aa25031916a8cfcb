// small_v3.cu -- one-thread-per-row kernel instances for AM-QFT variant 3.
#include "gen/small_gen_v3.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace smallk {
template std::unique_ptr<FastPlan> make_small_sized<3, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_sized<3, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<3, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<3, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<3, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<3, double>(int, size_t, const void*, uint32_t, int);
}  // namespace smallk
}  // namespace amqft_b200
