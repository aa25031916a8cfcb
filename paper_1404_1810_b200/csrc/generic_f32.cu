// generic_f32.cu -- fp32 instances of the schedule-interpreter kernels.
#include "generic_kernels.cuh"
namespace amqft_b200 {
AMQFT_INSTANTIATE_GENERIC(float)
}
