// tile_v3.cu -- in-shared-memory four-step instances for AM-QFT variant 3.
#include "gen/small_gen_v3.cuh"
#include "tile_kernel.cuh"

namespace amqft_b200 {
namespace tilek {
template std::unique_ptr<FastPlan> make_tile<3, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile<3, double>(size_t, const void*, uint32_t, int);
}  // namespace tilek
}  // namespace amqft_b200
