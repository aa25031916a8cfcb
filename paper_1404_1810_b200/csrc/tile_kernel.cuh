// tile_kernel.cuh -- four-step inside one CTA's shared memory (path 6).
//
// CDFT N = N1 N2 (fp32: N = 16 .. 4096, N1, N2 <= 64; N = 8192 .. 65536 as
// three factors, k_tile3 below, from 2^15 on a thread-block cluster; fp64:
// factors <= 32, N = 16 .. 1024 / 2048 .. 32768) in ONE pass over HBM:
// both factors are one-thread-per-transform AM-QFTs kept in registers -- the
// straight-line code codegen/gen_small.py traces from the plan compiler
// (SmallGen<V, 0, LOGN, R>, every line one reference add/sub/mul,
// variants.cpp:186-231 / elaborations.cpp), the same code k_small runs from
// HBM rows.  Decimation in frequency, n = N2 n1 + n2, k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_n2 w_N2^(n2 k2) [ w_N^(n2 k1) sum_n1 x[N2 n1 + n2] w_N1^(n1 k1) ]
// phase A  thread = (row, n2): the N1 inputs x[N2 n1 + n2] straight from HBM
//          (a warp's lanes take consecutive n2: every load instruction
//          covers 256 contiguous bytes), AM-QFT of length N1 in registers,
//          output k1 times w_N^(n2 k1) (host long double table, rounded once)
//          into the padded tile P[k1][n2] in shared memory;
// phase B  thread = (row, k1): row k1 of P (128-bit loads; the pitch of
//          N2 + 2 complex values makes a quarter-warp hit 8 distinct bank
//          groups), AM-QFT of length N2 in registers, output k2 straight to
//          HBM at X[k1 + N1 k2] (lanes on consecutive k1: 256 contiguous
//          bytes per store instruction).
// Shared-memory traffic is one write and one read of the row (the fused
// kernel of fast_kernel.cuh, which keeps the whole length-N DAG, makes six
// such round trips and is bound by them); the arithmetic is the same within
// 1 % (N2 ops(N1) + N1 ops(N2) + N twiddle multiplies vs ops(N)).  The AM-QFT
// DAG is kept inside each factor, not across the split (the four-step's
// convention, fourstep.cu), so the result is checked against the fp64 oracle
// of the same variant within 1e-5 log2 N; sub-transforms of length <= 64 are
// stable in fp32 for the sine-family variants 5-8 too (fast.cuh), so all 8
// variants run in fp32.  fp64 plans take this path where the result stays
// within 1e-12 of the CPU reference of the same variant (fast.cu
// tile_covers: variants 1-4 at every size, 5-8 up to N = 256; elsewhere the
// fused kernel's fp64 instance, bitwise the reference, keeps the plan).
// The inverse is the swap trick, fused into phase A's loads and phase B's
// stores.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <vector>

#include "fast.cuh"
#include "generic.cuh"
#include "small_kernel.cuh"

namespace amqft_b200 {
namespace tilek {

using smallk::SmallGen;
using smallk::TabP;

// Complex element and the tile pad (in complex values) that spreads the
// 128-bit row loads of a quarter-warp over 8 distinct bank groups: fp32 rows
// are read two values at a time (pitch / 2 odd), fp64 one (pitch odd).
template <typename R> struct RT;
template <> struct RT<float> {
  using V2 = float2;
  static constexpr int PAD = 2;
  static constexpr bool spread(int pitch) { return (pitch / 2) % 2 == 1; }
};
template <> struct RT<double> {
  using V2 = double2;
  static constexpr int PAD = 1;
  static constexpr bool spread(int pitch) { return pitch % 2 == 1; }
};
template <typename R> __device__ __forceinline__ typename RT<R>::V2 mk2(R a, R b);
template <> __device__ __forceinline__ float2 mk2<float>(float a, float b) { return make_float2(a, b); }
template <> __device__ __forceinline__ double2 mk2<double>(double a, double b) { return make_double2(a, b); }
// Arithmetic of the factors.  The split paths are held to the tolerance, not
// to bitwise equality with the reference, so the operators are plain ones
// that nvcc may contract into FMAs where a constant multiply feeds an add /
// subtract (one rounding less, one instruction less; config 2: 0.765 ->
// 0.744 ms).
template <typename R> struct TArith {
  static __device__ __forceinline__ R add(R a, R b) { return a + b; }
  static __device__ __forceinline__ R sub(R a, R b) { return a - b; }
  static __device__ __forceinline__ R mul(R a, R b) { return a * b; }
};

// a * w (complex)
template <typename R, typename V2>
__device__ __forceinline__ void cmul(R& a, R& b, const V2 w) {
  const R na = a * w.x - b * w.y, nb = a * w.y + b * w.x;
  a = na;
  b = nb;
}

// T: threads per CTA; MB: CTAs per SM the registers are budgeted for (0:
// by factor size); PF: bulk L2 prefetch of the CTA's next tile (-1: where a
// factor needs the 4-CTA register budget).
template <typename R, int LG1, int LG2, int T_ = 64, int MB_ = 0, int PF_ = -1>
struct TCfg {
  using V2 = typename RT<R>::V2;
  static constexpr int N1 = 1 << LG1, N2 = 1 << LG2, N = N1 * N2;
  static constexpr int LGM = LG1 > LG2 ? LG1 : LG2;
  static constexpr int T = T_;                                   // threads per CTA
  static constexpr int NMIN = N1 < N2 ? N1 : N2;
  static constexpr int R_ = T / NMIN > 0 ? T / NMIN : 1;        // rows per tile
  static constexpr int PITCH = N2 + RT<R>::PAD;                  // complex values per P row
  static constexpr int ROWP = N1 * PITCH;                        // complex values per tile row
  // Registers decide the CTAs per SM (64 threads each).  fp32: 64-point
  // factors 4 (246 registers: measured 0.906 ms against 1.07 ms at 6 CTAs /
  // 168 registers, config 2), 32-point 10, 16-point 16; fp64: 32-point 6
  // (150 registers), 16-point 12.
  static constexpr int LGR = LGM + (sizeof(R) == 8 ? 1 : 0);
  static constexpr int MINB = MB_ > 0 ? MB_ : (LGR >= 6 ? (sizeof(R) == 8 ? 6 : 4) : (LGR == 5 ? 10 : 16)) * 64 / T;
  // Measured (B200, 2^28 reals per launch): the 64 x 64 kernel is bound by
  // the latency of phase A's loads (4 CTAs of 2 warps per SM; long
  // scoreboard is the top stall); with the next tile on its way into L2
  // 0.912 -> 0.769 ms.  The small factors run 10-16 CTAs per SM and lose
  // 2-6 % with it.
  static constexpr bool PF = PF_ < 0 ? LGR >= 6 : PF_ != 0;
  static constexpr size_t SMEM = static_cast<size_t>(R_) * ROWP * sizeof(V2);
  static constexpr size_t SMEMX = SMEM + 2 * R_ * sizeof(R);   // + x[0], x[N/2] per row (DCT-0 rows)
  static constexpr int NT1 = (N1 < 8 ? 8 : N1) / 4, NT2 = (N2 < 8 ? 8 : N2) / 4;
  static_assert(RT<R>::spread(PITCH), "bank-group spread of the 128-bit row loads");
};

// The generated code moves a row in chunks: fp32 chunk c = complex values
// 2c, 2c+1 (four reals), fp64 chunk c = complex value c (two reals); every
// I/O object below serves both through the two overloads of ld / st.

// phase A: input n1 of column n2 from HBM (stride N2), output k1 times the
// twiddle into P[k1][n2]
// FN = 1 (RDFT rows, signal.hpp:122-124): the row is N reals, read as x + 0 i;
// the CDFT of a real row is C - i S, and the packed spectrum P[k] = C[k] (k <=
// N/2), P[N - k] = S[k] is Re X[k] for k <= N/2 and Im X[k] above (conjugate
// symmetry), so the last phase stores one real per output index.
// FN = 2 (A/B instance only, AMQFT_AB_TILE_TW=fly): CDFT rows with the twiddle
// w_N^(n2 k1) computed on the fly (sincospif of the exact integer phase)
// instead of read from the table -- the north-star's "computed on the fly or
// held in a table, chosen by measured GB/s": config 2 runs 0.738 ms (5822
// GB/s) with the table and 0.763 ms (5631 GB/s) on the fly, both 1.9e-7 from
// the CPU reference (profiles/r02_tile_twiddle_ab.log), so the table it is.
template <typename R, int N2, int PITCH, bool INV, int FN = 0>
struct AIo {
  using V2 = typename RT<R>::V2;
  const V2* __restrict__ gi;   // x + n2 (FN = 1: a pointer to reals)
  V2* sp;                      // P + n2
  const V2* __restrict__ tw;   // tw + n2: tw[k1 N2 + n2] = w_N^(n2 k1)
  int n2 = 0, lgn = 0;         // FN = 2: the thread's column and log2 N
  __device__ __forceinline__ V2 twiddle(int k1) const {
    if constexpr (FN == 2) {
      const unsigned e = (static_cast<unsigned>(n2) * static_cast<unsigned>(k1)) & ((1u << lgn) - 1u);
      float sn, cs;
      sincospif(static_cast<float>(e) * (2.0f / static_cast<float>(1u << lgn)), &sn, &cs);
      return mk2<R>(static_cast<R>(cs), static_cast<R>(-sn));
    } else {
      return __ldg(tw + k1 * N2);
    }
  }
  R* sx = nullptr;             // FN = 3: shared-memory copy of the row's x[0], x[N/2] for the last phase
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    if constexpr (FN == 1) {
      a = __ldcs(reinterpret_cast<const R*>(gi) + c * N2);
      b = R(0);
      return;
    }
    if constexpr (FN == 3 || FN == 4) {
      // DCT-0 / DST-0 rows (N/2 + 1 / N/2 - 1 cells, oracle.hpp:38-41) as the CDFT of the even /
      // odd extension y of length N: y[j] = x[j], y[N - j] = +-x[j] (DST-0: y[0] = y[N/2] = 0).
      // gi points at the row's first cell; element j = c N2 + n2.
      const R* xr = reinterpret_cast<const R*>(gi);
      const int nn = 1 << lgn, j = c * N2 + n2, m = 2 * j <= nn ? j : nn - j;
      b = R(0);
      if constexpr (FN == 3) {
        a = __ldcs(xr + m);
        if (j == 0) sx[0] = a;
        if (2 * j == nn) sx[1] = a;
      } else {
        a = (m == 0 || 2 * m == nn) ? R(0) : __ldcs(xr + m - 1);
        if (2 * j > nn) a = -a;
      }
      return;
    }
    const V2 u = __ldcs(gi + c * N2);
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if (c != 0) cmul(a, b, twiddle(c));   // k1 = 0: w = 1
    sp[c * PITCH] = mk2<R>(a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    const V2 w1 = twiddle(2 * c + 1);
    if (c != 0) cmul(a, b, twiddle(2 * c));
    cmul(d, e, w1);
    sp[(2 * c) * PITCH] = mk2<R>(a, b);
    sp[(2 * c + 1) * PITCH] = mk2<R>(d, e);
  }
};

// last phase: a contiguous row of the tile (128-bit loads), output k at
// X[base + STRIDE k]
template <typename R, int STRIDE, bool INV, int FN = 0>
struct BIo {
  using V2 = typename RT<R>::V2;
  const V2* sp;              // the row (16-byte aligned: even pitches in fp32)
  V2* __restrict__ go;       // X + base (FN = 1: a pointer to reals, P + base)
  R scale;
  int base = 0, half = 0;    // FN = 1, 3, 4: output index base + STRIDE c against N / 2
  R x0 = R(0), xh = R(0);    // FN = 3: the row's x[0] and x[N/2]
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 v = sp[c];
    a = v.x; b = v.y;
  }
  __device__ __forceinline__ void ld(int c, float& a, float& b, float& d, float& e) const {
    const float4 v = reinterpret_cast<const float4*>(sp)[c];
    a = v.x; b = v.y; d = v.z; e = v.w;
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if constexpr (FN == 1) {
      __stcs(reinterpret_cast<R*>(go) + c * STRIDE, base + c * STRIDE <= half ? a : b);
      return;
    }
    if constexpr (FN == 3) {   // DCT-0[k] = (Re X[k] + x[0] + (-1)^k x[N/2]) / 2, k <= N/2
      const int k = base + c * STRIDE;
      if (k <= half) __stcs(reinterpret_cast<R*>(go) + c * STRIDE, R(0.5) * (a + x0 + ((k & 1) ? -xh : xh)));
      return;
    }
    if constexpr (FN == 4) {   // DST-0[k] = -Im X[k] / 2, 0 < k < N/2 (cell k - 1)
      const int k = base + c * STRIDE;
      if (k > 0 && k < half) __stcs(reinterpret_cast<R*>(go) + c * STRIDE - 1, R(-0.5) * b);
      return;
    }
    if (INV) __stcs(go + c * STRIDE, mk2<R>(b * scale, a * scale));
    else __stcs(go + c * STRIDE, mk2<R>(a, b));
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    st(2 * c, a, b);
    st(2 * c + 1, d, e);
  }
};

template <int V, typename R, bool INV, class C, int FN = 0>
__global__ void __launch_bounds__(C::T, C::MINB)
k_tile(const R* __restrict__ in, R* __restrict__ out, size_t rows,
       const __grid_constant__ TabP<R, C::NT1> t1, const __grid_constant__ TabP<R, C::NT2> t2,
       const typename RT<R>::V2* __restrict__ tw, R scale) {
  using V2 = typename RT<R>::V2;
  constexpr int LG1 = 31 - __builtin_clz(C::N1), LG2 = 31 - __builtin_clz(C::N2);
  using G1 = SmallGen<V, 0, LG1, R>;
  using G2 = SmallGen<V, 0, LG2, R>;
  constexpr int N1 = C::N1, N2 = C::N2, N = C::N;
  extern __shared__ __align__(128) unsigned char sm[];
  V2* P = reinterpret_cast<V2*>(sm);
  R* SX = reinterpret_cast<R*>(sm + C::SMEM);   // FN = 3: x[0], x[N/2] of the tile's rows (2 R_ values)
  const int tid = threadIdx.x;
  const size_t tiles = (rows + C::R_ - 1) / C::R_;
  for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const size_t row0 = tile * C::R_;
    if constexpr (C::PF && FN < 3) {   // the CTA's next tile: one bulk prefetch into L2
      const size_t nrow = (tile + gridDim.x) * C::R_;
      if (tid == 0 && nrow + C::R_ <= rows)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                     ::"l"(in + nrow * (FN == 1 ? 1 : 2) * N),
                       "n"(C::R_ * N * static_cast<int>(FN == 1 ? sizeof(R) : sizeof(V2))) : "memory");
    }
    // ---- phase A: columns of x -> P (twiddled)
#pragma unroll 1
    for (int i = tid; i < C::R_ * N2; i += C::T) {
      const int r = i / N2, n2 = i % N2;
      if (row0 + r < rows) {
        // FN = 1: rows of N reals; FN = 3 / 4: rows of N/2 + 1 / N/2 - 1 reals, addressed from
        // their first cell (the pointers are reinterpreted in the loads)
        constexpr size_t CELLS = FN == 3 ? N / 2 + 1 : (FN == 4 ? N / 2 - 1 : N);
        const V2* src = FN == 1 ? reinterpret_cast<const V2*>(in + (row0 + r) * N + n2)
                        : (FN == 3 || FN == 4) ? reinterpret_cast<const V2*>(in + (row0 + r) * CELLS)
                                               : reinterpret_cast<const V2*>(in) + (row0 + r) * N + n2;
        AIo<R, N2, C::PITCH, INV, FN> io{src, P + r * C::ROWP + n2, tw + n2, n2, LG1 + LG2, SX + 2 * r};
        G1::template run<TArith<R>>(io, t1.v);
      }
    }
    __syncthreads();
    // ---- phase B: rows of P -> X
#pragma unroll 1
    for (int j = tid; j < C::R_ * N1; j += C::T) {
      const int r = j / N1, k1 = j % N1;
      if (row0 + r < rows) {
        constexpr size_t CELLS = FN == 3 ? N / 2 + 1 : (FN == 4 ? N / 2 - 1 : N);
        V2* dst = FN == 1 ? reinterpret_cast<V2*>(out + (row0 + r) * N + k1)
                  : (FN == 3 || FN == 4) ? reinterpret_cast<V2*>(out + (row0 + r) * CELLS + k1)
                                         : reinterpret_cast<V2*>(out) + (row0 + r) * N + k1;
        BIo<R, N1, INV, FN> io{P + r * C::ROWP + k1 * C::PITCH, dst, scale, k1, N / 2, FN == 3 ? SX[2 * r] : R(0),
                               FN == 3 ? SX[2 * r + 1] : R(0)};
        G2::template run<TArith<R>>(io, t2.v);
      }
    }
    __syncthreads();   // P is rewritten by the next tile's phase A
  }
}

// w_n^j for j < n as rows [k][m] = w_n^(k m), k < K, m < Mm: long double, rounded once
template <typename V2>
void fill_twiddles(V2* dst, int K, int Mm, long n) {
  using E = decltype(V2{}.x);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < Mm; ++m) {
      const long double a = two_pi * static_cast<long double>((static_cast<long>(k) * m) % n) / static_cast<long double>(n);
      dst[static_cast<size_t>(k) * Mm + m] = V2{static_cast<E>(cosl(a)), static_cast<E>(-sinl(a))};
    }
}

inline void tk_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

template <int V, typename R, int LG1, int LG2, int T = 64, int MB = 0, int PF = -1, int FN = 0>
class TilePlanImpl final : public FastPlan {
  using C = TCfg<R, LG1, LG2, T, MB, PF>;
  using V2 = typename RT<R>::V2;

 public:
  TilePlanImpl(const void* tab, uint32_t nmax, int device) {
    tk_check(smallk::fetch_table(t1_.v, C::NT1, tab, nmax));
    tk_check(smallk::fetch_table(t2_.v, C::NT2, tab, nmax));
    std::vector<V2> tw(C::N);   // tw[k1 N2 + n2] = w_N^(n2 k1)
    fill_twiddles(tw.data(), C::N1, C::N2, C::N);
    tk_check(cudaMalloc(&tw_, tw.size() * sizeof(V2)));
    tk_check(cudaMemcpy(tw_, tw.data(), tw.size() * sizeof(V2), cudaMemcpyHostToDevice));
    auto f0 = k_tile<V, R, false, C, FN>;
    tk_check(cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEMX)));
    if constexpr (FN == 0 || FN == 2) {
      auto f1 = k_tile<V, R, true, C, FN>;
      tk_check(cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEMX)));
    }
    int per_sm = 0;
    tk_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, C::T, C::SMEMX));
    if (per_sm < 1) throw std::runtime_error("tile four-step kernel does not fit an SM");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = per_sm * sms;
    launches = 1;
  }
  ~TilePlanImpl() override {
    if (tw_) cudaFree(tw_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    const size_t tiles = (rows + C::R_ - 1) / C::R_;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(tiles, static_cast<size_t>(grid_cap_)));
    const R scale = R(1) / static_cast<R>(C::N);
    if constexpr (FN == 1 || FN >= 3) {   // real rows: forward only (the engine composes their inverses)
      if (inverse) throw std::invalid_argument("the tile kernel's real rows have no inverse");
      k_tile<V, R, false, C, FN><<<grid, C::T, C::SMEMX, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                             t1_, t2_, tw_, scale);
    } else if (inverse) {
      k_tile<V, R, true, C, FN><<<grid, C::T, C::SMEMX, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                             t1_, t2_, tw_, scale);
    } else {
      k_tile<V, R, false, C, FN><<<grid, C::T, C::SMEMX, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                              t1_, t2_, tw_, scale);
    }
    tk_check(cudaGetLastError());
  }

 private:
  TabP<R, C::NT1> t1_{};
  TabP<R, C::NT2> t2_{};
  V2* tw_ = nullptr;
  int grid_cap_ = 148;
};

// ---- Three factors, N = N1 N2 N3 (the row no longer fits two register-
// resident factors).  n = N2 N3 n1 + N3 n2 + n3, k = k1 + N1 k2 + N1 N2 k3,
// M = N2 N3:
// phase A  thread = m = N3 n2 + n3: x[M n1 + m] from HBM (coalesced over m),
//          AM-QFT of length N1, times w_N^(m k1), into Y[k1][n2][n3];
// phase B  thread = (k1, n3): column n2 of Y[k1] in place (a thread reads
//          and rewrites its own cells), AM-QFT of length N2, times
//          w_M^(n3 k2);
// phase C  thread = (k2, k1), k1 fastest: row Y[k1][k2][.] with 128-bit
//          loads (pitches N3 + pad per k2 and N2 (N3 + pad) + pad per k1: a
//          quarter-warp hits 8 distinct bank groups), AM-QFT of length N3,
//          output k3 to X[k1 + N1 (k2 + N2 k3)] (lanes on consecutive k1).
// P > 1 (the row exceeds one SM's shared memory): one row per thread-block
// cluster of P CTAs.  CTA q owns the planes k1 in [q N1/P, (q+1) N1/P) of Y;
// in phase A it transforms the columns m in [q M/P, (q+1) M/P) and stores
// output k1 straight into the owner's shared memory over DSMEM
// (st.shared::cluster), the only exchange: (P-1)/P of the row.  Phases B and
// C run on the CTA's own planes.  Two cluster barriers per row: a full one
// after phase A (all planes complete), and a split one around the rest --
// a relaxed arrive after the CTA's phase C, the wait just before its first
// remote store of the next row -- so the next row's loads and arithmetic
// overlap the peers' phase C.
template <typename R, int LG1, int LG2, int LG3, int T_, int MB_, int P_ = 1>
struct T3Cfg {
  using V2 = typename RT<R>::V2;
  static constexpr int N1 = 1 << LG1, N2 = 1 << LG2, N3 = 1 << LG3, M = N2 * N3, N = N1 * M;
  static constexpr int T = T_, MINB = MB_, P = P_;
  static constexpr int K1 = N1 / P;                     // planes per CTA
  static constexpr int P3 = N3 + RT<R>::PAD;            // complex values per (k1, k2) row
  static constexpr int PM = N2 * P3 + RT<R>::PAD;       // complex values per k1 plane
  static constexpr int ROWP = K1 * PM;
  static constexpr size_t SMEM = static_cast<size_t>(ROWP) * sizeof(V2);
  static constexpr int NT1 = (N1 < 8 ? 8 : N1) / 4, NT2 = (N2 < 8 ? 8 : N2) / 4, NT3 = (N3 < 8 ? 8 : N3) / 4;
  static_assert(RT<R>::spread(P3) && RT<R>::spread(PM), "bank-group spread of the 128-bit row loads");
  static_assert(P == 1 || ((M / P) % T == 0 && K1 % 2 == 0), "whole warps in phase A; an output chunk has one owner");
};

__device__ __forceinline__ uint32_t tk_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tk_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// no fence: orders execution only ("this CTA has finished READING its planes"; the loads' values
// have been consumed).  The releasing form also waits for the thread's outstanding global stores
// of phase C -- ncu showed membar as the second stall of the 2^15 kernel (2.0 per issue): 3712 ->
// 3843 GB/s.  (Asynchronous DSMEM stores completing on the owner's mbarrier instead of the full
// barrier after phase A: correct, but slower -- 3384 GB/s at 2^15, fp64 2^14 3467 against 4112.)
__device__ __forceinline__ void tk_cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void tk_cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double a, double b) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}

// phase A, P = 1: output k1 into the CTA's own Y
template <typename R, int M, int PM, bool INV>
struct A3Io {
  using V2 = typename RT<R>::V2;
  const V2* __restrict__ gi;   // x + m
  V2* sp;                      // Y + n2 P3 + n3
  const V2* __restrict__ tw;   // tw1 + m: tw1[k1 M + m] = w_N^(m k1)
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 u = __ldcs(gi + c * M);
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if (c != 0) cmul(a, b, __ldg(tw + c * M));
    sp[c * PM] = mk2<R>(a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    const V2 w1 = __ldg(tw + (2 * c + 1) * M);
    if (c != 0) cmul(a, b, __ldg(tw + (2 * c) * M));
    cmul(d, e, w1);
    sp[(2 * c) * PM] = mk2<R>(a, b);
    sp[(2 * c + 1) * PM] = mk2<R>(d, e);
  }
};

// phase A of the cluster kernel: output k1 goes to plane k1 % K1 of CTA
// k1 / K1 (both compile-time per store); the first store of a row waits for
// the peers' phase C of the previous row (the split barrier)
template <typename R, int M, int PM, int K1, int P, bool INV>
struct A3IoC {
  using V2 = typename RT<R>::V2;
  const V2* __restrict__ gi;
  const V2* __restrict__ tw;
  uint32_t yb[P];    // the P CTAs' Y + n2 P3 + n3 in the cluster window
  bool wait;
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 u = __ldcs(gi + c * M);
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void put(int k1, R a, R b) const {
    st_cluster(yb[k1 / K1] + static_cast<uint32_t>((k1 % K1) * PM * sizeof(V2)), a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if (c != 0) cmul(a, b, __ldg(tw + c * M));
    else if (wait) tk_cluster_wait();   // warp-uniform: every lane of the warp is in this item
    put(c, a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    const V2 w1 = __ldg(tw + (2 * c + 1) * M);
    if (c != 0) cmul(a, b, __ldg(tw + (2 * c) * M));
    else if (wait) tk_cluster_wait();
    cmul(d, e, w1);
    put(2 * c, a, b);
    put(2 * c + 1, d, e);
  }
};

template <typename R, int N3, int P3>
struct B3Io {
  using V2 = typename RT<R>::V2;
  V2* sp;                      // Y + k1 PM + n3
  const V2* __restrict__ tw;   // tw2 + n3: tw2[k2 N3 + n3] = w_M^(n3 k2)
  __device__ __forceinline__ void ld(int c, R& a, R& b) const {
    const V2 u = sp[c * P3];
    a = u.x; b = u.y;
  }
  __device__ __forceinline__ void ld(int c, R& a, R& b, R& d, R& e) const {
    ld(2 * c, a, b);
    ld(2 * c + 1, d, e);
  }
  __device__ __forceinline__ void st(int c, R a, R b) const {
    if (c != 0) cmul(a, b, __ldg(tw + c * N3));
    sp[c * P3] = mk2<R>(a, b);
  }
  __device__ __forceinline__ void st(int c, R a, R b, R d, R e) const {
    const V2 w1 = __ldg(tw + (2 * c + 1) * N3);
    if (c != 0) cmul(a, b, __ldg(tw + (2 * c) * N3));
    cmul(d, e, w1);
    sp[(2 * c) * P3] = mk2<R>(a, b);
    sp[(2 * c + 1) * P3] = mk2<R>(d, e);
  }
};

template <int V, typename R, bool INV, class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_tile3(const R* __restrict__ in, R* __restrict__ out, size_t rows,
        const __grid_constant__ TabP<R, C::NT1> t1, const __grid_constant__ TabP<R, C::NT2> t2,
        const __grid_constant__ TabP<R, C::NT3> t3, const typename RT<R>::V2* __restrict__ tw1,
        const typename RT<R>::V2* __restrict__ tw2, R scale) {
  using V2 = typename RT<R>::V2;
  constexpr int LG1 = 31 - __builtin_clz(C::N1), LG2 = 31 - __builtin_clz(C::N2), LG3 = 31 - __builtin_clz(C::N3);
  using G1 = SmallGen<V, 0, LG1, R>;
  using G2 = SmallGen<V, 0, LG2, R>;
  using G3 = SmallGen<V, 0, LG3, R>;
  constexpr int N1 = C::N1, N2 = C::N2, N3 = C::N3, M = C::M, N = C::N, P = C::P, K1 = C::K1;
  extern __shared__ __align__(128) unsigned char sm[];
  V2* Y = reinterpret_cast<V2*>(sm);
  const int tid = threadIdx.x;
  // P > 1: one row per cluster; q = this CTA's rank (its planes and columns)
  uint32_t q = 0;
  uint32_t ywin[P];
  if constexpr (P > 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
#pragma unroll
    for (int k = 0; k < P; ++k)
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ywin[k]) : "r"(tk_u32(Y)), "r"(k));
  }
  (void)ywin;
  const size_t r_first = blockIdx.x / P, r_step = gridDim.x / P;
  for (size_t row = r_first; row < rows; row += r_step) {
    // the next row's inputs of this CTA: bulk prefetches into L2
    if (row + r_step < rows) {
      const R* nx = in + (row + r_step) * 2 * N;
      if constexpr (P == 1) {
        if (tid == 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                       ::"l"(nx), "n"(N * static_cast<int>(sizeof(V2))) : "memory");
      } else if (tid < N1) {   // N1 pieces of M/P columns
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                     ::"l"(nx + (static_cast<size_t>(tid) * M + q * (M / P)) * 2),
                       "n"(M / P * static_cast<int>(sizeof(V2))) : "memory");
      }
    }
    const V2* x = reinterpret_cast<const V2*>(in) + row * N;
    if constexpr (P == 1) {
#pragma unroll 1
      for (int m = tid; m < M; m += C::T) {
        A3Io<R, M, C::PM, INV> io{x + m, Y + (m / N3) * C::P3 + m % N3, tw1 + m};
        G1::template run<TArith<R>>(io, t1.v);
      }
      __syncthreads();
    } else {
#pragma unroll 1
      for (int mm = tid; mm < M / P; mm += C::T) {
        const int m = static_cast<int>(q) * (M / P) + mm;
        A3IoC<R, M, C::PM, K1, P, INV> io;
        io.gi = x + m;
        io.tw = tw1 + m;
        const uint32_t off = static_cast<uint32_t>(((m / N3) * C::P3 + m % N3) * sizeof(V2));
#pragma unroll
        for (int k = 0; k < P; ++k) io.yb[k] = ywin[k] + off;
        io.wait = mm == tid && row != r_first;   // first item of a row after the first
        G1::template run<TArith<R>>(io, t1.v);
      }
      tk_cluster_arrive();   // all planes complete and visible
      tk_cluster_wait();
    }
#pragma unroll 1
    for (int j = tid; j < K1 * N3; j += C::T) {
      const int n3 = j % N3, k1 = j / N3;
      B3Io<R, N3, C::P3> io{Y + k1 * C::PM + n3, tw2 + n3};
      G2::template run<TArith<R>>(io, t2.v);
    }
    __syncthreads();
#pragma unroll 1
    for (int j = tid; j < K1 * N2; j += C::T) {
      const int k1 = j % K1, k2 = j / K1;
      BIo<R, N1 * N2, INV> io{Y + k1 * C::PM + k2 * C::P3,
                              reinterpret_cast<V2*>(out) + row * N + (q * K1 + k1) + N1 * k2, scale};
      G3::template run<TArith<R>>(io, t3.v);
    }
    if constexpr (P == 1) __syncthreads();   // Y is rewritten by the next row's phase A
    else tk_cluster_arrive_relaxed();         // ... by the peers': the wait is in their first store
  }
  if constexpr (P > 1) {
    // balance the last arrive; no CTA exits while a peer may still store into it
    if (r_first < rows) tk_cluster_wait();
  }
}

template <int V, typename R, int LG1, int LG2, int LG3, int T, int MB, int P = 1>
class Tile3PlanImpl final : public FastPlan {
  using C = T3Cfg<R, LG1, LG2, LG3, T, MB, P>;
  using V2 = typename RT<R>::V2;

 public:
  Tile3PlanImpl(const void* tab, uint32_t nmax, int device) {
    tk_check(smallk::fetch_table(t1_.v, C::NT1, tab, nmax));
    tk_check(smallk::fetch_table(t2_.v, C::NT2, tab, nmax));
    tk_check(smallk::fetch_table(t3_.v, C::NT3, tab, nmax));
    // tw1[k1 M + m] = w_N^(m k1), tw2[k2 N3 + n3] = w_M^(n3 k2)
    std::vector<V2> tw(static_cast<size_t>(C::N) + C::M);
    fill_twiddles(tw.data(), C::N1, C::M, C::N);
    fill_twiddles(tw.data() + C::N, C::N2, C::N3, C::M);
    tk_check(cudaMalloc(&tw_, tw.size() * sizeof(V2)));
    tk_check(cudaMemcpy(tw_, tw.data(), tw.size() * sizeof(V2), cudaMemcpyHostToDevice));
    auto f0 = k_tile3<V, R, false, C>;
    auto f1 = k_tile3<V, R, true, C>;
    tk_check(cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM)));
    tk_check(cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (P == 1) {
      int per_sm = 0;
      tk_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, C::T, C::SMEM));
      if (per_sm < 1) throw std::runtime_error("three-factor tile kernel does not fit an SM");
      grid_cap_ = per_sm * sms;
    } else {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      fill_(&cfg, attr, P * sms, nullptr);
      int nc = 0;
      tk_check(cudaOccupancyMaxActiveClusters(&nc, f0, &cfg));
      if (nc < 1) throw std::runtime_error("three-factor tile kernel: no cluster of this size fits");
      grid_cap_ = nc * P;
    }
    launches = 1;
  }
  ~Tile3PlanImpl() override {
    if (tw_) cudaFree(tw_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    const R scale = R(1) / static_cast<R>(C::N);
    const R* fi = static_cast<const R*>(in);
    R* fo = static_cast<R*>(out);
    const V2* tw1 = tw_;
    const V2* tw2 = tw_ + C::N;
    cudaError_t e;
    if (P == 1) {
      const unsigned grid = static_cast<unsigned>(std::min<size_t>(rows, static_cast<size_t>(grid_cap_)));
      if (inverse) k_tile3<V, R, true, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, t1_, t2_, t3_, tw1, tw2, scale);
      else k_tile3<V, R, false, C><<<grid, C::T, C::SMEM, st>>>(fi, fo, rows, t1_, t2_, t3_, tw1, tw2, scale);
      e = cudaGetLastError();
    } else {
      const unsigned grid = static_cast<unsigned>(std::min<size_t>(rows * P, static_cast<size_t>(grid_cap_)));
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      fill_(&cfg, attr, static_cast<int>(grid), st);
      if (inverse) e = cudaLaunchKernelEx(&cfg, k_tile3<V, R, true, C>, fi, fo, rows, t1_, t2_, t3_, tw1, tw2, scale);
      else e = cudaLaunchKernelEx(&cfg, k_tile3<V, R, false, C>, fi, fo, rows, t1_, t2_, t3_, tw1, tw2, scale);
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    tk_check(e);
  }

 private:
  static void fill_(cudaLaunchConfig_t* cfg, cudaLaunchAttribute* attr, int grid, cudaStream_t st) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg->gridDim = dim3(static_cast<unsigned>(grid));
    cfg->blockDim = dim3(C::T);
    cfg->dynamicSmemBytes = C::SMEM;
    cfg->stream = st;
    cfg->attrs = attr;
    cfg->numAttrs = 1;
  }
  TabP<R, C::NT1> t1_{};
  TabP<R, C::NT2> t2_{};
  TabP<R, C::NT3> t3_{};
  V2* tw_ = nullptr;
  int grid_cap_ = 148;
};

// The split per size (fast.cu tile_split mirrors it for the op counts).
// Measured on the B200, ms per 2^28 reals (A/B instances built during
// development, tools/prof_fast.py): fp32 2048 as 64 x 32 0.780 (32 x 64: 0.803); 512 as 16 x 32 0.679
// (32 x 16: 0.717); 8192 as 32 x 16 x 16 at 256 threads x 2 CTAs 0.747 (16 x
// 16 x 32: 0.802; 128 threads x 3: 0.93); 16384 as 32 x 16 x 32 at 512
// threads 0.843 (16 x 32 x 32: 0.959, 32 x 32 x 16: 0.928); 2^15 on a cluster
// of 2 CTAs 1.14 (4 CTAs x 256 threads: 1.23); 2^16 on 4 CTAs as 32 x 32 x 64
// 1.42 (64 x 32 x 32: 1.52; 8 CTAs: 1.46 / 1.56) -- the multi-pass four-step
// ran both at 2.13.  Dead ends: twiddles in tensor memory (tcgen05.ld per
// chunk: 2.5 ms at N = 4096 against 0.91), 128-thread CTAs (0.953 against
// 0.912), N = 8 as 2 x 4 (no gain over the direct kernel).
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile(size_t n, const void* tab, uint32_t nmax, int dev) {
  if constexpr (sizeof(R) == 4 && V == 4) {   // A/B: config 2's twiddles on the fly (variant 4 only)
    const char* e = std::getenv("AMQFT_AB_TILE_TW");
    if (n == 4096 && e && e[0] == 'f') return std::make_unique<TilePlanImpl<V, R, 6, 6, 64, 0, -1, 2>>(tab, nmax, dev);
  }
  if constexpr (sizeof(R) == 4) {
    switch (n) {
      case 16: return std::make_unique<TilePlanImpl<V, R, 2, 2>>(tab, nmax, dev);
      case 32: return std::make_unique<TilePlanImpl<V, R, 2, 3>>(tab, nmax, dev);
      case 64: return std::make_unique<TilePlanImpl<V, R, 3, 3>>(tab, nmax, dev);
      case 128: return std::make_unique<TilePlanImpl<V, R, 3, 4>>(tab, nmax, dev);
      case 256: return std::make_unique<TilePlanImpl<V, R, 4, 4>>(tab, nmax, dev);
      case 512: return std::make_unique<TilePlanImpl<V, R, 4, 5>>(tab, nmax, dev);
      case 1024: return std::make_unique<TilePlanImpl<V, R, 5, 5>>(tab, nmax, dev);
      case 2048: return std::make_unique<TilePlanImpl<V, R, 6, 5>>(tab, nmax, dev);
      case 4096: return std::make_unique<TilePlanImpl<V, R, 6, 6>>(tab, nmax, dev);
      case 8192: return std::make_unique<Tile3PlanImpl<V, R, 5, 4, 4, 256, 2>>(tab, nmax, dev);
      case 16384: return std::make_unique<Tile3PlanImpl<V, R, 5, 4, 5, 512, 1>>(tab, nmax, dev);
      case 32768: return std::make_unique<Tile3PlanImpl<V, R, 5, 5, 5, 512, 1, 2>>(tab, nmax, dev);
      case 65536: return std::make_unique<Tile3PlanImpl<V, R, 5, 5, 6, 256, 1, 4>>(tab, nmax, dev);
    }
  } else {   // fp64: factors <= 32 points
    switch (n) {
      case 16: return std::make_unique<TilePlanImpl<V, R, 2, 2>>(tab, nmax, dev);
      case 32: return std::make_unique<TilePlanImpl<V, R, 2, 3>>(tab, nmax, dev);
      case 64: return std::make_unique<TilePlanImpl<V, R, 3, 3>>(tab, nmax, dev);
      case 128: return std::make_unique<TilePlanImpl<V, R, 3, 4>>(tab, nmax, dev);
      case 256: return std::make_unique<TilePlanImpl<V, R, 4, 4>>(tab, nmax, dev);
      case 512: return std::make_unique<TilePlanImpl<V, R, 4, 5>>(tab, nmax, dev);
      case 1024: return std::make_unique<TilePlanImpl<V, R, 5, 5>>(tab, nmax, dev);
      case 2048: return std::make_unique<Tile3PlanImpl<V, R, 3, 4, 4, 128, 4>>(tab, nmax, dev);
      case 4096: return std::make_unique<Tile3PlanImpl<V, R, 4, 4, 4, 256, 2>>(tab, nmax, dev);
      case 8192: return std::make_unique<Tile3PlanImpl<V, R, 5, 4, 4, 256, 1>>(tab, nmax, dev);
      case 16384: return std::make_unique<Tile3PlanImpl<V, R, 5, 4, 5, 256, 1, 2>>(tab, nmax, dev);
      case 32768: return std::make_unique<Tile3PlanImpl<V, R, 5, 5, 5, 256, 1, 4>>(tab, nmax, dev);
    }
  }
  return nullptr;
}

// RDFT rows (FunctionId::Rdft) as the CDFT of x + 0 i on the two-factor
// kernel: twice the arithmetic of the reference's RDFT (half a CDFT), but one
// pass over HBM at sizes whose only other path is the generic interpreter.
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile_rdft(size_t n, const void* tab, uint32_t nmax, int dev) {
  switch (n) {
    case 128: return std::make_unique<TilePlanImpl<V, R, 3, 4, 64, 0, -1, 1>>(tab, nmax, dev);
    case 256: return std::make_unique<TilePlanImpl<V, R, 4, 4, 64, 0, -1, 1>>(tab, nmax, dev);
    case 512: return std::make_unique<TilePlanImpl<V, R, 4, 5, 64, 0, -1, 1>>(tab, nmax, dev);
    case 1024: return std::make_unique<TilePlanImpl<V, R, 5, 5, 64, 0, -1, 1>>(tab, nmax, dev);
    case 2048:
      if constexpr (sizeof(R) == 4) return std::make_unique<TilePlanImpl<V, R, 6, 5, 64, 0, -1, 1>>(tab, nmax, dev);
      break;
    case 4096:
      if constexpr (sizeof(R) == 4) return std::make_unique<TilePlanImpl<V, R, 6, 6, 64, 0, -1, 1>>(tab, nmax, dev);
      break;
  }
  return nullptr;
}

// DCT-0 / DST-0 rows (FunctionId::Dct / Dst) as the CDFT of the even / odd extension: four times the
// reference's arithmetic, one pass, at sizes the small scalar kernels do not reach.  fn: 2 DCT-0, 3 DST-0.
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile_dctdst(int fn, size_t n, const void* tab, uint32_t nmax, int dev) {
#define AMQFT_TILE_REAL(LGA, LGB)                                                                          \
  return fn == AMQFT_FN_DCT ? std::unique_ptr<FastPlan>(new TilePlanImpl<V, R, LGA, LGB, 64, 0, -1, 3>(tab, nmax, dev)) \
                            : std::unique_ptr<FastPlan>(new TilePlanImpl<V, R, LGA, LGB, 64, 0, -1, 4>(tab, nmax, dev));
  switch (n) {
    case 256: AMQFT_TILE_REAL(4, 4)
    case 512: AMQFT_TILE_REAL(4, 5)
    case 1024: AMQFT_TILE_REAL(5, 5)
    case 2048:
      if constexpr (sizeof(R) == 4) { AMQFT_TILE_REAL(6, 5) }
      break;
    case 4096:
      if constexpr (sizeof(R) == 4) { AMQFT_TILE_REAL(6, 6) }
      break;
  }
#undef AMQFT_TILE_REAL
  return nullptr;
}

}  // namespace tilek
}  // namespace amqft_b200
