// small_v7.cu -- one-thread-per-row kernel instances for AM-QFT variant 7.
#include "gen/small_gen_v7.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace smallk {
template std::unique_ptr<FastPlan> make_small_sized<7, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_sized<7, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<7, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<7, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<7, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<7, double>(int, size_t, const void*, uint32_t, int);
}  // namespace smallk
}  // namespace amqft_b200
