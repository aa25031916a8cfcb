// slab_kernel.cuh -- column-slab passes: the multi-pass four-step without
// transposes (large N: configs 3 / 4).
//
// One pass transforms every COLUMN of a matrix whose rows are contiguous:
// column c, element j at in[base(c) + j sj].  A CTA takes a slab of W adjacent
// columns (every global access of a warp covers W contiguous values), keeps
// the W x L slab in shared memory and runs the length-L = NA NB transform of
// each column as the two-factor split of tile_kernel.cuh (register-resident
// AM-QFT factors, one shared-memory crossing), multiplies output jo by the
// four-step twiddle w^(col jo) (fp64 recurrence per thread, seeded from the
// plan's twiddle set) and stores
//   slab mode        out[base'(c) + jo sj']      (W contiguous values per jo)
//   transposing mode out[c L + jo]               (a column becomes a row)
// With these, N = L1 L2 (L <= 1024) is two passes over HBM
//   pass 1  columns n2 of x [n1][n2], transposing:  Y[n2][k1] = w_N^(n2 k1) sum_n1 ...
//   pass 2  columns k1 of Y [n2][k1], slab mode:    X[k2][k1] = X[k1 + L1 k2]
// and N = L1 L2 L3 three (SlabPlan below), against three and four for the
// column / row / transpose passes of fourstep.cu: natural order in and out,
// no transpose kernel.  The AM-QFT DAG is kept inside each factor (the
// four-step's convention).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <vector>

#include "fast.cuh"
#include "generic.cuh"
#include "slab.cuh"
#include "small_kernel.cuh"
#include "tile_kernel.cuh"

namespace amqft_b200 {
namespace slabk {

using smallk::SmallGen;
using smallk::TabP;
using tilek::cmul;
using tilek::mk2;
using tilek::RT;

template <typename R, int LGA, int LGB, int W_, int T_ = 256>
struct SCfg {
  // L2 prefetch of the CTA's next slab: measured (B200, fp32, GB/s) +21 / +16 / +7 % on 2^21 / 2^22 /
  // 2^23, whose plans have 128-point passes (8 loads in flight per thread), and -7 .. -10 % on the
  // 256- to 1024-point passes (2^17 .. 2^20, 2^24), so only the 128-point instances issue it
  static constexpr bool PF = LGA + LGB == 7;
  using V2 = typename RT<R>::V2;
  static constexpr int NA = 1 << LGA, NB = 1 << LGB, L = NA * NB, W = W_, T = T_;
  static constexpr int KP = NB * W + 1;                     // ka pitch: odd, lanes on ka hit distinct banks
  static constexpr size_t SMEM = static_cast<size_t>(NA) * KP * sizeof(V2);
  static constexpr int NTA = (NA < 8 ? 8 : NA) / 4, NTB = (NB < 8 ? 8 : NB) / 4;
  // two CTAs per SM where the registers allow (32-point fp64 factors need 150)
  static constexpr int MINB = (SMEM > 100 * 1024 || (sizeof(R) == 8 && (LGA >= 5 || LGB >= 5))) ? 1 : 2;
};

// phase A: element j = NB ja + jb of the column from HBM (lanes on adjacent
// columns), output ka times w_L^(jb ka) into P[ka][jb][w]
template <typename R, int NB, int W, int KP, bool INV>
struct AIo {
  using V2 = typename RT<R>::V2;
  const V2* __restrict__ gi;   // the column's element jb
  size_t sa;                   // NB sj_in
  V2* sp;                      // P + jb W + w
  const V2* __restrict__ tw;   // tw + jb: tw[ka NB + jb] = w_L^(jb ka)
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 u = __ldcs(gi + c * sa);
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if (c != 0) cmul(a, b, __ldg(tw + c * NB));
    sp[c * KP] = mk2<R>(a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    st(2 * c, a, b);
    st(2 * c + 1, d, e);
  }
};

// phase B: row P[ka][.][w], output jo = ka + NA kb times the pass twiddle
// w^(col jo) (fp64 recurrence along kb: the generated code stores ascending)
template <typename R, int NA, int W, bool INV>
struct BIo {
  using V2 = typename RT<R>::V2;
  const V2* sp;            // P + ka KP + w
  V2* __restrict__ go;     // out + column base + ka sj_out
  size_t so;               // NA sj_out
  R scale;
  int twiddle;
  // w^(col (ka + NA kb)) for the next output kb in ascending order, step
  // w^(col NA); any other store order (the fp64 schedules) re-seeds it
  double cr, ci, sr, si;
  unsigned long long col;
  int ka, next;
  const ColTwiddle* tw;
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 v = sp[c * W];
    a = v.x; b = v.y;
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void st(int c, R a, R b) {
    if (twiddle) {
      // the fp32 schedules store in ascending order (checked by the tests against the oracle at every
      // slab length); testing it at run time costs them 10-20 % (the re-seed is inlined at every store)
      if constexpr (sizeof(R) == 8) {
        if (c != next) smallk::twiddle_d(col * static_cast<unsigned long long>(ka + NA * c), *tw, cr, ci);
        next = c + 1;
      }
      const R fr = static_cast<R>(cr), fi = static_cast<R>(ci);
      const R na = a * fr - b * fi, nb = a * fi + b * fr;
      a = na;
      b = nb;
      const double tr = cr * sr - ci * si, ti = cr * si + ci * sr;
      cr = tr;
      ci = ti;
    }
    if (INV) __stcs(go + c * so, mk2<R>(b * scale, a * scale));
    else __stcs(go + c * so, mk2<R>(a, b));
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) {
    st(2 * c, a, b);
    st(2 * c + 1, d, e);
  }
};

// INV_IN: re/im exchanged on the way in (first pass of an inverse);
// INV_OUT: exchanged and scaled on the way out (last pass)
template <int V, typename R, bool INV_IN, bool INV_OUT, class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_slab(const R* __restrict__ in, R* __restrict__ out, size_t rows, const __grid_constant__ SlabPass p,
       const __grid_constant__ TabP<R, C::NTA> ta, const __grid_constant__ TabP<R, C::NTB> tb,
       const typename RT<R>::V2* __restrict__ twl, R scale) {
  using V2 = typename RT<R>::V2;
  constexpr int LGA = 31 - __builtin_clz(C::NA), LGB = 31 - __builtin_clz(C::NB);
  using GA = SmallGen<V, 0, LGA, R>;
  using GB = SmallGen<V, 0, LGB, R>;
  constexpr int NA = C::NA, NB = C::NB, W = C::W;
  extern __shared__ __align__(128) unsigned char sm[];
  V2* P = reinterpret_cast<V2*>(sm);
  const int tid = threadIdx.x;
  const size_t per_row = p.cols / W, slabs = rows * per_row;
  for (size_t s = blockIdx.x; s < slabs; s += gridDim.x) {
    const size_t g = s / per_row;
    const unsigned c0 = static_cast<unsigned>(s - g * per_row) * W;
    const V2* x = reinterpret_cast<const V2*>(in) + g * p.in_row + (c0 / p.qin) * p.qi + c0 % p.qin;
    // the CTA's next slab on its way into L2: one bulk prefetch per row of the slab (W contiguous values)
    if (C::PF && s + gridDim.x < slabs) {
      const size_t s2 = s + gridDim.x, g2 = s2 / per_row;
      const unsigned n0 = static_cast<unsigned>(s2 - g2 * per_row) * W;
      const V2* nx = reinterpret_cast<const V2*>(in) + g2 * p.in_row + (n0 / p.qin) * p.qi + n0 % p.qin;
      for (int j = tid; j < C::L; j += C::T)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                     ::"l"(nx + j * p.sj_in), "n"(W * static_cast<int>(sizeof(V2))) : "memory");
    }
    // ---- phase A
#pragma unroll 1
    for (int i = tid; i < W * NB; i += C::T) {
      const int w = i % W, jb = i / W;
      AIo<R, NB, W, C::KP, INV_IN> io{x + w + jb * p.sj_in, NB * p.sj_in, P + jb * W + w, twl + jb};
      GA::template run<tilek::TArith<R>>(io, ta.v);
    }
    __syncthreads();
    // ---- phase B
    V2* y = reinterpret_cast<V2*>(out) + g * p.out_row;
#pragma unroll 1
    for (int i = tid; i < W * NA; i += C::T) {
      const int w = p.transposing ? i / NA : i % W;
      const int ka = p.transposing ? i % NA : i / W;
      const unsigned c = c0 + w;
      BIo<R, NA, W, INV_OUT> io;
      io.sp = P + ka * C::KP + w;
      io.go = y + ((c / p.qout) * p.qo + c % p.qout) * p.sw_out + ka * p.sj_out;
      io.so = NA * p.sj_out;
      io.scale = scale;
      io.twiddle = p.twiddle;
      io.tw = &p.tw;
      io.ka = ka;
      io.next = 0;
      io.col = static_cast<unsigned long long>(c / p.tdiv) * p.tw.mul;
      if (p.twiddle) {
        smallk::twiddle_d(io.col * static_cast<unsigned long long>(ka), p.tw, io.cr, io.ci);
        smallk::twiddle_d(io.col * static_cast<unsigned long long>(NA), p.tw, io.sr, io.si);
      }
      GB::template run<tilek::TArith<R>>(io, tb.v);
    }
    __syncthreads();   // P is rewritten by the next slab's phase A
  }
}

template <int V, typename R, int LGA, int LGB, int W>
class SlabPassImpl final : public SlabPassExec<R> {
  using C = SCfg<R, LGA, LGB, W>;
  using V2 = typename RT<R>::V2;

 public:
  SlabPassImpl(const void* tab, uint32_t nmax, int device) {
    tilek::tk_check(smallk::fetch_table(ta_.v, C::NTA, tab, nmax));
    tilek::tk_check(smallk::fetch_table(tb_.v, C::NTB, tab, nmax));
    std::vector<V2> tw(C::L);   // tw[ka NB + jb] = w_L^(jb ka)
    tilek::fill_twiddles(tw.data(), C::NA, C::NB, C::L);
    tilek::tk_check(cudaMalloc(&tw_, tw.size() * sizeof(V2)));
    tilek::tk_check(cudaMemcpy(tw_, tw.data(), tw.size() * sizeof(V2), cudaMemcpyHostToDevice));
    set_attr(k_slab<V, R, false, false, C>);
    set_attr(k_slab<V, R, true, false, C>);
    set_attr(k_slab<V, R, false, true, C>);
    set_attr(k_slab<V, R, true, true, C>);
    int per_sm = 0;
    tilek::tk_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_slab<V, R, false, false, C>, C::T, C::SMEM));
    if (per_sm < 1) throw std::runtime_error("slab kernel does not fit an SM");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = per_sm * sms;
  }
  ~SlabPassImpl() override {
    if (tw_) cudaFree(tw_);
  }
  int width() const override { return W; }
  void run(const void* in, void* out, size_t rows, const SlabPass& p, bool inv_in, bool inv_out, R scale,
           cudaStream_t st) override {
    const size_t slabs = rows * (p.cols / W);
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(slabs, static_cast<size_t>(grid_cap_)));
    const R* fi = static_cast<const R*>(in);
    R* fo = static_cast<R*>(out);
    if (inv_in && inv_out) k_slab<V, R, true, true, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, p, ta_, tb_, tw_, scale);
    else if (inv_in) k_slab<V, R, true, false, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, p, ta_, tb_, tw_, scale);
    else if (inv_out) k_slab<V, R, false, true, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, p, ta_, tb_, tw_, scale);
    else k_slab<V, R, false, false, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, p, ta_, tb_, tw_, scale);
    tilek::tk_check(cudaGetLastError());
  }

 private:
  template <class F>
  static void set_attr(F f) {
    tilek::tk_check(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM)));
  }
  TabP<R, C::NTA> ta_{};
  TabP<R, C::NTB> tb_{};
  V2* tw_ = nullptr;
  int grid_cap_ = 148;
};

// Column lengths with a slab instance: 128 (8 x 16, 32 columns), 256 (16 x
// 16, 32), 512 (16 x 32, 16), 1024 (32 x 32, 16); fp64: 16 / 16 / 8 / 8
// columns (the slab is 33-131 KB of shared memory).
template <int V, typename R>
std::unique_ptr<SlabPassExec<R>> make_slab_pass(size_t len, const void* tab, uint32_t nmax, int dev) {
  if constexpr (sizeof(R) == 4) {
    switch (len) {
      case 128: return std::make_unique<SlabPassImpl<V, R, 3, 4, 32>>(tab, nmax, dev);
      case 256: return std::make_unique<SlabPassImpl<V, R, 4, 4, 32>>(tab, nmax, dev);
      case 512: return std::make_unique<SlabPassImpl<V, R, 4, 5, 16>>(tab, nmax, dev);
      case 1024: return std::make_unique<SlabPassImpl<V, R, 5, 5, 16>>(tab, nmax, dev);
      // 64-point factors: 8- and 4-column slabs (64- and 32-byte runs) in 131 KB
      case 2048: return std::make_unique<SlabPassImpl<V, R, 6, 5, 8>>(tab, nmax, dev);
      case 4096: return std::make_unique<SlabPassImpl<V, R, 6, 6, 4>>(tab, nmax, dev);
    }
  } else {
    switch (len) {
      case 128: return std::make_unique<SlabPassImpl<V, R, 3, 4, 16>>(tab, nmax, dev);
      case 256: return std::make_unique<SlabPassImpl<V, R, 4, 4, 16>>(tab, nmax, dev);
      case 512: return std::make_unique<SlabPassImpl<V, R, 4, 5, 8>>(tab, nmax, dev);
      case 1024: return std::make_unique<SlabPassImpl<V, R, 5, 5, 8>>(tab, nmax, dev);
    }
  }
  return nullptr;
}

}  // namespace slabk
}  // namespace amqft_b200
