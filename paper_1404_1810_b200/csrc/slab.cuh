// slab.cuh -- interface of the column-slab passes (slab_kernel.cuh) for the
// code that schedules them (fourstep.cu) without the generated kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

#include "fast.cuh"

namespace amqft_b200 {
namespace slabk {

// Addressing of one pass (element units).  Column c of batch row g:
//   in  g in_row  + (c / qin)  qi + c % qin  + j  sj_in
//   out g out_row + ((c / qout) qo + c % qout) sw_out + jo sj_out
// (qin = qout = cols, qi = qo = 0: the identity; W divides qin and qout).
struct SlabPass {
  size_t in_row = 0, out_row = 0;
  unsigned cols = 0;
  unsigned qin = 0, qout = 0;
  size_t qi = 0, qo = 0;
  size_t sj_in = 0, sj_out = 0, sw_out = 1;
  unsigned tdiv = 1;       // twiddle column index = c / tdiv
  int twiddle = 0;         // multiply output jo by w^(tw.mul (c / tdiv) jo)
  int transposing = 0;     // lanes on consecutive jo (sj_out = 1) instead of consecutive columns
  ColTwiddle tw;
};

// One pass: the kernel instance for a column length, its constants and launcher.
template <typename R>
class SlabPassExec {
 public:
  virtual ~SlabPassExec() = default;
  virtual void run(const void* in, void* out, size_t rows, const SlabPass& p, bool inv_in, bool inv_out, R scale,
                   cudaStream_t st) = 0;
  virtual int width() const = 0;
};

}  // namespace slabk

// The pass of column length `len` (128 / 256 / 512 / 1024) for a variant;
// nullptr when there is no instance (fast.cu).
template <typename R>
std::unique_ptr<slabk::SlabPassExec<R>> make_slab_pass_rt(int variant, size_t len, const void* d_trig, uint32_t nmax,
                                                          int dev);

}  // namespace amqft_b200
