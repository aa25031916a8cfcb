// fourstep.cuh -- large-N CDFT as a four-step over the fused AM-QFT kernel
// (fourstep.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "fast.cuh"

namespace amqft_b200 {

// Fused / small-CDFT plan for one sub-transform size (nullptr if none),
// its op counts, and whether a single kernel covers n: fast.cu.
// columns: the factor runs in column mode (FastPlan::exec_columns), which
// only the one-thread-per-row kernels have.
std::unique_ptr<FastPlan> make_fast_sub(int variant, size_t n, int dtype, const void* tab, uint32_t nmax, int dev,
                                        const void* tab64 = nullptr, bool columns = false);
OpCount fast_sub_op_counts(int variant, size_t n, int dtype, bool columns = false);
bool fast_sub_covered(int dtype, size_t n, int variant, bool allow_tile = true);
// Plans created while set (on this thread) skip the column-slab plans, which have no transposed
// output (amqft_plan_create_transposable).
void fourstep_prefer_transposable(bool on);

// CDFT, fast order, N up to 2^26 beyond the single-kernel sizes.
bool fourstep_covers(const amqft_plan_desc& d);
// d_trig64: fp64 copy of the table (fp32 plans whose sub-transforms compute in fp64)
std::unique_ptr<FastPlan> make_fourstep_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax,
                                             const void* d_trig64 = nullptr);
OpCount fourstep_op_counts(const amqft_plan_desc& d);
// {A, B, C}: n = A B C (two-factor plans: B = 1)
amqft_status fourstep_factors(const amqft_plan_desc& d, size_t* f3);

// Distributed four-step building blocks (amqft_dist_twiddle_scatter,
// amqft_transpose_c64).  d_dst: host array of nparts device pointers.
void dist_twiddle_scatter(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                          int src, int nparts, int trig_mode, cudaStream_t st);
void transpose_c64(const void* in, void* out, size_t mats, size_t r, size_t c, cudaStream_t st);
void dist_twiddle_scatter_direct(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                                 int nparts, int trig_mode, size_t a, cudaStream_t st);
void dist_twiddle_scatter_t(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                            int src, int nparts, int trig_mode, size_t a, cudaStream_t st);

}  // namespace amqft_b200
