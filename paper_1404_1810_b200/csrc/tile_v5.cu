// tile_v5.cu -- in-shared-memory four-step instances for AM-QFT variant 5.
#include "gen/small_gen_v5.cuh"
#include "tile_kernel.cuh"

namespace amqft_b200 {
namespace tilek {
template std::unique_ptr<FastPlan> make_tile<5, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile<5, double>(size_t, const void*, uint32_t, int);
}  // namespace tilek
}  // namespace amqft_b200
