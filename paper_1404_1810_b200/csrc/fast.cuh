// fast.cuh -- fused fast-path kernels for the CDFT hot path (see fast.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "../../include/amqft_b200.h"
#include "plan.hpp"

namespace amqft_b200 {

class FastPlan {
 public:
  virtual ~FastPlan() = default;
  virtual void exec(const void* in, void* out, size_t rows, int inverse,
                    cudaStream_t st) = 0;
  int launches = 1;
};

// Returns nullptr when no fused kernel covers the request.
std::unique_ptr<FastPlan> make_fast_plan(const amqft_plan_desc& d,
                                         const void* d_trig, uint32_t nmax);
OpCount fast_op_counts(const amqft_plan_desc& d);

// One-thread-per-row kernel for small CDFTs (small_kernel.cuh): fp32 N <= 64,
// fp64 N <= 32.  nullptr when not covered; *ops receives the traced
// schedule's op counts (= the reference meter).
std::unique_ptr<FastPlan> make_small_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax,
                                          OpCount* ops);

}  // namespace amqft_b200
