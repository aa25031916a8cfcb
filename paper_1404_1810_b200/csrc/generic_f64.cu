// generic_f64.cu -- fp64 instances of the schedule-interpreter kernels.
#include "generic_kernels.cuh"
namespace amqft_b200 {
AMQFT_INSTANTIATE_GENERIC(double)
}
