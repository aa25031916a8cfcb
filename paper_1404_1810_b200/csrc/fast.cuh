// fast.cuh -- fused fast-path kernels for the CDFT hot path (see fast.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>

#include "../../include/amqft_b200.h"
#include "plan.hpp"

namespace amqft_b200 {

// Four-step twiddles w_N^j (fourstep.cu): two half-size fp64 tables
// (w^(jh B), w^(jl)) or sincospi on the fly.
struct ColTwiddle {
  const double2* hi = nullptr;
  const double2* lo = nullptr;
  int logb = 0, logn = 0, onthefly = 0;
  unsigned long long mul = 1;   // exponent scale: w_N^(mul n2 k1) = w_(N/mul)^(n2 k1)
};

class FastPlan {
 public:
  virtual ~FastPlan() = default;
  virtual void exec(const void* in, void* out, size_t rows, int inverse,
                    cudaStream_t st) = 0;
  // Column mode (four-step first pass): `mats` matrices [N][cols] of
  // complex values; transform every column (length N, stride cols) into
  // `out` in the same layout, output k1 of column n2 multiplied by
  // w^(n2 k1).  Inverse: input re/im exchanged (the swap trick's first
  // half).  Returns false when the plan has no column mode.
  virtual bool exec_columns(const void*, void*, size_t /*mats*/, size_t /*cols*/, int /*inverse*/,
                            const ColTwiddle&, cudaStream_t) {
    return false;
  }
  // Column-mode four-steps only (distributed four-step, config 5): the
  // transform without its final transpose, rows left as out[r][ka][kb] =
  // X[ka + A kb]; returns A, or 0 when the plan has no such mode.
  virtual size_t transposed_factor() const { return 0; }
  virtual void exec_transposed(const void*, void*, size_t, cudaStream_t) {}
  int launches = 1;
};

// fp32 plans of the sine-family variants 5-8 from N = 512 on: the M5-M8
// recurrences (elaborations.cpp:350-527, lens flip variants.cpp:220-231)
// amplify fp32 rounding beyond 1e-5 log2 N (measured on the B200,
// tools/err_sweep.py: 5e-4 at N = 512, 5e2 at N = 4096).  Such plans keep
// fp32 rows in HBM and compute in fp64: the fused kernel's fp64 instance
// with fp32 I/O (N = 1024-4096, the reference DAG, bitwise the reference
// before the final rounding), a four-step over stable sub-transforms (fast
// order, N = 512 and N >= 8192), or the generic exact path in fp64.
inline bool f32_needs_f64_compute(int variant, size_t n) { return variant >= 5 && n >= 512; }

// Returns nullptr when no fused kernel covers the request.
// d_trig64: fp64 copy of the table for fp32 plans that compute in fp64.
std::unique_ptr<FastPlan> make_fast_plan(const amqft_plan_desc& d,
                                         const void* d_trig, uint32_t nmax,
                                         const void* d_trig64 = nullptr);
OpCount fast_op_counts(const amqft_plan_desc& d);

// In-shared-memory four-step (tile_kernel.cuh, path 6): fp32 CDFT rows,
// N = 16 .. 65536, two (three from N = 8192) one-thread-per-transform AM-QFT
// factors (<= 64 points, stable in fp32 for all 8 variants), one pass over
// HBM (2^15 / 2^16: one row per thread-block cluster, DSMEM exchange).  AMQFT_AB_TILE=lo,hi restricts the sizes it takes.
// AMQFT_AB_TILE=none disables it (A/B measurements against the fused
// kernel, which keeps the whole length-N DAG).
bool tile_covers(const amqft_plan_desc& d);
bool tile_rdft_covers(const amqft_plan_desc& d);   // RDFT rows as the CDFT of x + 0 i (fp32 256 .. 4096)
std::unique_ptr<FastPlan> make_tile_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax);
OpCount tile_op_counts(const amqft_plan_desc& d);

// One-thread-per-row kernel for small CDFTs (small_kernel.cuh): fp32 N <= 64,
// fp64 N <= 32.  nullptr when not covered; *ops receives the traced
// schedule's op counts (= the reference meter).
std::unique_ptr<FastPlan> make_small_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax,
                                          OpCount* ops);

}  // namespace amqft_b200
