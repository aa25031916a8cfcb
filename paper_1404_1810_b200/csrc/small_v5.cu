// small_v5.cu -- one-thread-per-row kernel instances for AM-QFT variant 5.
#include "gen/small_gen_v5.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace smallk {
template std::unique_ptr<FastPlan> make_small_sized<5, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_sized<5, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<5, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_rdft<5, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<5, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_small_dctdst<5, double>(int, size_t, const void*, uint32_t, int);
}  // namespace smallk
}  // namespace amqft_b200
