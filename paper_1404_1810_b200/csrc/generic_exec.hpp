// generic_exec.hpp -- host-side launch interface of the generic
// schedule-interpreter kernels (kernels in generic_kernels.cuh, explicit
// instantiations in generic_f32.cu / generic_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "plan.hpp"

namespace amqft_b200 {

// Modulation constants: table slots f(2 pi p / nmax), p in [1, nmax/4), then
// the base constant cos(2 pi / 8) at [nmax/4 - 1] (TrigTable::constants,
// variants.cpp:289-299).  Lookup at (index, n) reads slot index*nmax/n
// (variants.cpp:281).  On-the-fly evaluates f in fp64 with cospi/sinpi.
struct TrigRef {
  const void* table;  // R[nmax/4]
  uint32_t nmax;
  uint32_t kind;      // 0 2cos, 1 2sin, 2 1/(2cos), 3 1/(2sin)
  uint32_t on_the_fly;
};

// Per-program device descriptor (offsets into the concatenated arrays).
struct ProgInfo {
  uint32_t ei_base;
  uint32_t stage_base;
  uint32_t nstages;
  uint32_t cells;
};

struct JobDev {
  uint32_t prog;
  uint32_t off;
  uint32_t src;  // 0 A, 1 B
  uint32_t dst;
};

struct ProgLaunch {
  const EI* eis;
  const uint32_t* prefix;
  const Stage* stages;
  const ProgInfo* progs;
  const JobDev* jobs;
  uint32_t njobs;
  const void* srcA;
  const void* srcB;
  void* dstA;
  void* dstB;
  size_t arena;
  size_t rows;
  TrigRef trig;
  int swap_in, swap_out;
  double scale;
  size_t smem;
  int T, K;
  unsigned grid;
  cudaStream_t stream;
};

// Each returns the cudaError_t of its launch.
template <typename R> cudaError_t launch_prog(const ProgLaunch& L);
template <typename R>
cudaError_t launch_stage(const EI* eis, const uint32_t* prefix, const Stage& s,
                         void* A, void* B, size_t arena, size_t rows,
                         const TrigRef& trig, unsigned grid, cudaStream_t st);
template <typename R>
cudaError_t launch_copy(const void* in, void* out, size_t total, int swap,
                        double scale, unsigned grid, cudaStream_t st);

}  // namespace amqft_b200
