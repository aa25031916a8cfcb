// tile_v2.cu -- in-shared-memory four-step and column-slab instances for AM-QFT variant 2.
#include "gen/small_gen_v2.cuh"
#include "slab_kernel.cuh"
#include "tile_kernel.cuh"

namespace amqft_b200 {
namespace tilek {
template std::unique_ptr<FastPlan> make_tile<2, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile<2, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile_rdft<2, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile_rdft<2, double>(size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile_dctdst<2, float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<FastPlan> make_tile_dctdst<2, double>(int, size_t, const void*, uint32_t, int);
}  // namespace tilek
namespace slabk {
template std::unique_ptr<SlabPassExec<float>> make_slab_pass<2, float>(size_t, const void*, uint32_t, int);
template std::unique_ptr<SlabPassExec<double>> make_slab_pass<2, double>(size_t, const void*, uint32_t, int);
}  // namespace slabk
}  // namespace amqft_b200
