// generic_kernels.cuh -- schedule-interpreter kernels (generic paths 0/1).
// Included only by generic_f32.cu / generic_f64.cu.
#pragma once

#include <stdexcept>

#include "generic.cuh"
#include "generic_exec.hpp"

namespace amqft_b200 {

// Runs stage programs out of shared memory.  Work unit = (row, job).
// Each stage: every thread evaluates up to K items into registers, the CTA
// synchronises, then writes them back in place (and runs any serial chain).
template <typename R, int T, int K>
__global__ void __launch_bounds__(T)
k_prog(const EI* __restrict__ eis, const uint32_t* __restrict__ prefix,
       const Stage* __restrict__ stages, const ProgInfo* __restrict__ progs,
       const JobDev* __restrict__ jobs, uint32_t njobs, const R* srcA,
       const R* srcB, R* dstA, R* dstB, size_t arena, size_t rows,
       TrigRef trig, int swap_in, int swap_out, R out_scale) {
  extern __shared__ __align__(16) unsigned char smraw[];
  R* sm = reinterpret_cast<R*>(smraw);
  const uint32_t tid = threadIdx.x;
  const size_t units = rows * njobs;
  for (size_t u = blockIdx.x; u < units; u += gridDim.x) {
    const size_t row = u / njobs;
    const JobDev job = jobs[u % njobs];
    const ProgInfo pi = progs[job.prog];
    const R* src = (job.src ? srcB : srcA) + row * arena + job.off;
    R* dst = (job.dst ? dstB : dstA) + row * arena + job.off;
    for (uint32_t i = tid; i < pi.cells; i += T) sm[i] = src[swap_in ? (i ^ 1u) : i];
    __syncthreads();
    const EI* pe = eis + pi.ei_base;
    const uint32_t* pp = prefix + pi.ei_base;
    for (uint32_t s = 0; s < pi.nstages; ++s) {
      const Stage st = stages[pi.stage_base + s];
      R val[K];
      uint32_t pos[K];
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const uint32_t g = tid + r * T;
        pos[r] = 0xffffffffu;
        if (g < st.items) {
          const uint32_t k = find_ei(pp, st.ei_begin, st.ei_end, g);
          const EI e = pe[k];
          if (e.op == OP_CHAIN_F || e.op == OP_CHAIN_B) {
            pos[r] = 0x80000000u | k;
          } else {
            uint32_t d;
            const uint32_t off = e.off;
            val[r] = eval_item<R>(e, g - __ldg(pp + k), &d, trig,
                                  [&](uint32_t p) { return sm[off + p]; });
            pos[r] = off + d;
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < K; ++r) {
        if (pos[r] == 0xffffffffu) continue;
        if (pos[r] & 0x80000000u) {
          const EI e = pe[pos[r] & 0x7fffffffu];
          R* base = sm + e.off;
          run_chain<R>(e, [&](int p) { return base[p]; },
                       [&](int p, R v) { base[p] = v; });
        } else {
          sm[pos[r]] = val[r];
        }
      }
      __syncthreads();
    }
    for (uint32_t i = tid; i < pi.cells; i += T) {
      const R v = sm[swap_out ? (i ^ 1u) : i];
      dst[i] = swap_out ? Arith<R>::mul(v, out_scale) : v;
    }
    __syncthreads();
  }
}

// One global stage of the multi-pass path over all rows.
template <typename R>
__global__ void __launch_bounds__(256)
k_stage(const EI* __restrict__ eis, const uint32_t* __restrict__ prefix,
        uint32_t b, uint32_t e, uint32_t items, R* bufA, R* bufB,
        size_t arena, size_t rows, TrigRef trig) {
  const size_t total = static_cast<size_t>(items) * rows;
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < total;
       g += size_t(gridDim.x) * blockDim.x) {
    const size_t row = g / items;
    const uint32_t it = static_cast<uint32_t>(g % items);
    const uint32_t k = find_ei(prefix, b, e, it);
    const EI ei = eis[k];
    const R* src = ((ei.flags & FL_SRC_B) ? bufB : bufA) + row * arena + ei.off;
    R* dst = ((ei.flags & FL_DST_B) ? bufB : bufA) + row * arena + ei.off;
    if (ei.op == OP_CHAIN_F || ei.op == OP_CHAIN_B) {
      run_chain<R>(ei, [&](int p) { return src[p]; }, [&](int p, R v) { dst[p] = v; });
    } else {
      uint32_t d;
      const R v = eval_item<R>(ei, it - __ldg(prefix + k), &d, trig,
                               [&](uint32_t p) { return src[p]; });
      dst[d] = v;
    }
  }
}

template <typename R>
__global__ void k_copy_rows(const R* __restrict__ in, R* __restrict__ out,
                            size_t total, int swap, R scale) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const R v = in[swap ? (i ^ 1u) : i];
    out[i] = swap ? Arith<R>::mul(v, scale) : v;
  }
}

template <typename R, int T, int K>
cudaError_t launch_prog_tk(const ProgLaunch& L) {
  auto fn = k_prog<R, T, K>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(L.smem));
  if (e != cudaSuccess) return e;
  fn<<<L.grid, T, L.smem, L.stream>>>(
      L.eis, L.prefix, L.stages, L.progs, L.jobs, L.njobs,
      static_cast<const R*>(L.srcA), static_cast<const R*>(L.srcB),
      static_cast<R*>(L.dstA), static_cast<R*>(L.dstB), L.arena, L.rows, L.trig,
      L.swap_in, L.swap_out, static_cast<R>(L.scale));
  return cudaGetLastError();
}

template <typename R, int T>
cudaError_t launch_prog_t(const ProgLaunch& L) {
  switch (L.K) {
    case 1: return launch_prog_tk<R, T, 1>(L);
    case 2: return launch_prog_tk<R, T, 2>(L);
    case 4: return launch_prog_tk<R, T, 4>(L);
    case 8: return launch_prog_tk<R, T, 8>(L);
    case 16: return launch_prog_tk<R, T, 16>(L);
    case 32: return launch_prog_tk<R, T, 32>(L);
  }
  return cudaErrorInvalidValue;
}

template <typename R>
cudaError_t launch_prog(const ProgLaunch& L) {
  return L.T == 512 ? launch_prog_t<R, 512>(L) : launch_prog_t<R, 256>(L);
}

template <typename R>
cudaError_t launch_stage(const EI* eis, const uint32_t* prefix, const Stage& s,
                         void* A, void* B, size_t arena, size_t rows,
                         const TrigRef& trig, unsigned grid, cudaStream_t st) {
  k_stage<R><<<grid, 256, 0, st>>>(eis, prefix, s.ei_begin, s.ei_end, s.items,
                                   static_cast<R*>(A), static_cast<R*>(B), arena, rows, trig);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_copy(const void* in, void* out, size_t total, int swap,
                        double scale, unsigned grid, cudaStream_t st) {
  k_copy_rows<R><<<grid, 256, 0, st>>>(static_cast<const R*>(in), static_cast<R*>(out),
                                       total, swap, static_cast<R>(scale));
  return cudaGetLastError();
}

#define AMQFT_INSTANTIATE_GENERIC(R)                                                   \
  template cudaError_t launch_prog<R>(const ProgLaunch&);                              \
  template cudaError_t launch_stage<R>(const EI*, const uint32_t*, const Stage&, void*, \
                                       void*, size_t, size_t, const TrigRef&, unsigned, \
                                       cudaStream_t);                                   \
  template cudaError_t launch_copy<R>(const void*, void*, size_t, int, double, unsigned, \
                                      cudaStream_t);

}  // namespace amqft_b200
