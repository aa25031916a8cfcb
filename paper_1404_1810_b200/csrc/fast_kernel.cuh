// fast_kernel.cuh -- fused AM-QFT CDFT kernel for sm_100a (path 2).
//
// One CTA runs a whole complex transform (N <= 8192 fp32, <= 4096 fp64) out
// of shared memory, persistent over the batch.  The formulation
// (tests/fast_model.py, proven bitwise against the oracle for all 8
// variants) keeps the four real chains of SplitComplex + SplitReal
// (Re/Im x Dct/Dst, src/elaborations.cpp:147-208) in natural index order,
// where every odd-function split of the recursion (variants.cpp:200-231)
// becomes an in-place mirror butterfly over nested segments and every AM
// conversion (elaborations.cpp:350-527) a pointwise multiply or a
// neighbour/serial operation on a strided residue class.
//
// Time-major variants 1,4,5,8 (forward = mirror network in time):
//   load      SplitComplex + SplitReal -> T (4 chains)
//   T-levels  mirror levels L = H .. 2LB, cooperative, in place on T
//   bottom    one thread per LB-segment: the remaining folds + spectra of
//             all blocks inside (generated straight-line code), T -> F;
//             one thread per chain for the cells at multiples of LB
//   U-levels  AM_B of the larger blocks, depth D-1 .. 0, on F
//   F-levels  SplitTimeParity recombination Dct/Dst(n), n = 2N/LB .. N
//   store     SplitReal + SplitComplex backward -> out
// Harmonic-major variants 2,3,6,7 run the transpose (chain folds, AM_F
// levels, bottom, mirror levels in frequency, store).
//
// Arithmetic goes through Arith<R> (__fadd_rn / __dadd_rn ...): no FMA
// contraction, so the fp64 instantiation reproduces the reference bitwise
// (serial recurrences included); the fp32 instantiation is the fast path.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>

#include "fast.cuh"
#include "fast_gen.cuh"
#include "generic.cuh"

namespace amqft_b200 {
namespace fastk {

template <int LOGLB>
__device__ __forceinline__ int ph(int i) { return i + (i >> LOGLB); }

__device__ __forceinline__ int parity(unsigned x) { return __popc(x) & 1; }

template <int V, typename R, int LOGN, int LOGLB>
struct FastCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int H = N / 2;
  static constexpr int LOGH = LOGN - 1;
  static constexpr int LB = 1 << LOGLB;
  static constexpr int LT = LOGH - LOGLB;        // depth of the bottom segments
  static constexpr int HP = H / LB;               // cells at multiples of LB
  static constexpr int NSEG = 4 * HP;             // bottom segments (4 chains)
  static constexpr int NT = NSEG + 32;            // + one warp for small chains
  static constexpr int CS = ((H + HP + 1) + 3) / 4 * 4;  // chain stride (skewed)
  static constexpr bool TM = (V == 1 || V == 4 || V == 5 || V == 8);
  static constexpr int SINE = V >= 5 ? 1 : 0;
  static constexpr bool CHAIN = (V == 1 || V == 5 || V == 3 || V == 7);
  static constexpr int UPC = N / 4 - N / (4 * LB);  // U items per chain
  static constexpr int UK = (4 * UPC + NT - 1) / NT;
  static constexpr size_t SMEM = 8 * CS * sizeof(R);
};

// Segment parameters at depth d: orientation, lens, residue (fast_model.segment_params).
template <int SINE>
__device__ __forceinline__ void seg_params(int lam_c, int s, int d, int* rho, int* lens, int* r) {
  *rho = d == 0 ? 0 : (s & 1);
  *lens = lam_c ^ (SINE & parity(static_cast<unsigned>(s ^ (s >> 1))));
  int res = 0, ln = lam_c, prev = 0;
  for (int i = 1; i <= d; ++i) {
    const int b = (s >> (d - i)) & 1;
    const int is_o = b != prev;
    res |= (is_o ^ ln) << (i - 1);
    ln ^= SINE & is_o;
    prev = b;
  }
  *r = res;
}

// Mirror level L over the four chains of buffer B (time-major forward when
// FWD, harmonic-major backward otherwise).  Items: N per level.
template <class C, typename R, bool FWD>
__device__ __forceinline__ void mirror_level(R* B, int lvl, int L, const R* tab, int nmax, R base) {
  using A = Arith<R>;
  const int half = L >> 1;
  const int lgh = 31 - __clz(half);
  const int lgL2 = lgh + 2;  // log2(2L)
  const int nseg_mask = (1 << (lvl - 1)) - 1;
  for (int g = threadIdx.x; g < C::N; g += C::NT) {
    const int v = g & (half - 1);
    if (v == 0) continue;
    const int s = (g >> lgh) & nseg_mask;
    const int c = g >> (C::LOGH - 1);
    const int lam_c = c & 1;
    const int rho = lvl == 1 ? 0 : (s & 1);
    const int lens = lam_c ^ (C::SINE & parity(static_cast<unsigned>(s ^ (s >> 1))));
    const int a = s * L;
    const int lo = a + v, hi = a + L - v;
    const int jc = rho ? hi : lo, mc = rho ? lo : hi;
    R* ch = B + c * C::CS;
    const R k = (v == (L >> 2)) ? base : __ldg(tab + (v * (nmax >> lgL2) - 1));
    const R p = ch[ph<C::LOGLB_>(jc)];
    const R q = ch[ph<C::LOGLB_>(mc)];
    if (FWD) {
      const R sm = A::add(p, q), df = A::sub(p, q);
      ch[ph<C::LOGLB_>(jc)] = lens ? df : sm;
      ch[ph<C::LOGLB_>(mc)] = A::mul(lens ? sm : df, k);
    } else {
      const R o = A::mul(q, k);
      ch[ph<C::LOGLB_>(jc)] = lens ? A::add(o, p) : A::add(p, o);
      ch[ph<C::LOGLB_>(mc)] = lens ? A::sub(o, p) : A::sub(p, o);
    }
  }
}

// Dct/Dst chain recombination (time-major backward, FWD=false) or fold
// (harmonic-major forward, FWD=true) at size n on buffer B.
template <class C, typename R, bool FWD>
__device__ __forceinline__ void chain_level(R* B, int n) {
  using A = Arith<R>;
  const int q = n >> 2;
  const int lgq = 31 - __clz(q);
  for (int g = threadIdx.x; g < n; g += C::NT) {
    const int c = g >> lgq;
    const int k = g & (q - 1);
    const int lam = c & 1;
    if (lam && k == 0) continue;
    R* ch = B + c * C::CS;
    const int i0 = ph<C::LOGLB_>(k), i1 = ph<C::LOGLB_>((n >> 1) - k);
    const R e = ch[i0], o = ch[i1];
    if (!FWD) {  // elaborations.cpp:310-329
      ch[i0] = lam ? A::add(o, e) : A::add(e, o);
      ch[i1] = lam ? A::sub(o, e) : A::sub(e, o);
    } else {     // elaborations.cpp:238-255 (a = e at m, b = o at n/2-m)
      ch[i0] = lam ? A::sub(e, o) : A::add(e, o);
      ch[i1] = lam ? A::add(e, o) : A::sub(e, o);
    }
  }
}

// AM conversion of the odd residue classes at depth `depth` (U-levels):
// time-major: AM_B on F; harmonic-major: AM_F on T.  Neighbour ops are
// staged through registers (read all, barrier, write all); serial
// recurrences are run in place by the class's j == 0 item.
template <class C, typename R>
__device__ void am_level(R* B, int depth) {
  using A = Arith<R>;
  constexpr int V = C::V_;
  R val[C::UK];
  int pos[C::UK];
#pragma unroll
  for (int u = 0; u < C::UK; ++u) {
    pos[u] = -1;
    const int g = threadIdx.x + u * C::NT;
    if (g >= 4 * C::UPC) continue;
    const int c = g / C::UPC;
    const int gp = g - c * C::UPC;
    const int t = (C::LOGN_ - 3) - (31 - __clz(C::N / 4 - 1 - gp));
    const int St = C::N / 4 - (C::N >> (t + 2));
    const int w = gp - St;
    const int r = w & ((1 << depth) - 1);
    const int j = w >> depth;
    const int lam_c = c & 1;
    const int m = (C::N >> (t + 2)) >> depth;
    if (m <= 2) continue;  // OO(8) base: no AM conversion
    const int q = m >> 1;
    const int lens = (C::SINE && depth > 0) ? ((r >> (depth - 1)) & 1) : lam_c;
    const int rO = r + ((1 - lens) << depth);
    const int hi = (C::N >> (t + 1)) - lam_c;
    const int stride = 2 << depth;
    R* ch = B + c * C::CS;
    auto cell = [&](int jj) { return ph<C::LOGLB_>(hi - (jj * stride + rO)); };
    if (C::CHAIN) {
      if (j == 0) pos[u] = (c << 24) | (t << 16) | r;  // run the class serially
      continue;
    }
    R out;
    if (C::TM) {
      if (V == 4) {
        out = lens == 0 ? (j < q - 1 ? A::add(ch[cell(j)], ch[cell(j + 1)]) : ch[cell(j)])
                        : (j > 0 ? A::add(ch[cell(j - 1)], ch[cell(j)]) : ch[cell(j)]);
      } else {  // V == 8
        out = lens == 0 ? (j > 0 ? A::sub(ch[cell(j)], ch[cell(j - 1)]) : ch[cell(j)])
                        : (j < q - 1 ? A::sub(ch[cell(j)], ch[cell(j + 1)]) : ch[cell(j)]);
      }
    } else {
      if (V == 2) {
        out = lens == 0 ? (j > 0 ? A::add(ch[cell(j)], ch[cell(j - 1)]) : ch[cell(j)])
                        : (j < q - 1 ? A::add(ch[cell(j + 1)], ch[cell(j)]) : ch[cell(j)]);
      } else {  // V == 6
        out = lens == 0 ? (j < q - 1 ? A::sub(ch[cell(j)], ch[cell(j + 1)]) : ch[cell(j)])
                        : (j > 0 ? A::sub(ch[cell(j)], ch[cell(j - 1)]) : ch[cell(j)]);
      }
    }
    val[u] = out;
    pos[u] = c * C::CS + cell(j);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < C::UK; ++u) {
    if (pos[u] < 0) continue;
    if (!C::CHAIN) {
      B[pos[u]] = val[u];
      continue;
    }
    // Serial recurrence over the class (elaborations.cpp:402-448, 472-513).
    const int c = pos[u] >> 24, t = (pos[u] >> 16) & 0xff, r = pos[u] & 0xffff;
    const int lam_c = c & 1;
    const int m = (C::N >> (t + 2)) >> depth;
    const int q = m >> 1;
    const int lens = (C::SINE && depth > 0) ? ((r >> (depth - 1)) & 1) : lam_c;
    const int rO = r + ((1 - lens) << depth);
    const int hi = (C::N >> (t + 1)) - lam_c;
    const int stride = 2 << depth;
    R* ch = B + c * C::CS;
    auto at = [&](int jj) -> R& { return ch[ph<C::LOGLB_>(hi - (jj * stride + rO))]; };
    if (C::TM) {
      // M1: cos asc/sub, sin desc/sub; M5: cos desc/add, sin asc/add
      const bool addop = V == 5;
      const bool desc = (V == 1) ? (lens == 1) : (lens == 0);
      const int s0 = desc ? q - 1 : 0, d = desc ? -1 : 1;
      R prev = A::mul(R(0.5), at(s0));
      at(s0) = prev;
      int p = s0;
      for (int k = 1; k < q; ++k) {
        p += d;
        prev = addop ? A::add(at(p), prev) : A::sub(at(p), prev);
        at(p) = prev;
      }
    } else {
      // M3: cos desc/sub, sin asc/sub; M7: cos asc/add, sin desc/add
      const bool addop = V == 7;
      const bool desc = (V == 3) ? (lens == 0) : (lens == 1);
      const int s0 = desc ? q - 1 : 0, d = desc ? -1 : 1;
      R prev = at(s0);
      int p = s0;
      for (int k = 1; k < q - 1; ++k) {
        p += d;
        prev = addop ? A::add(at(p), prev) : A::sub(at(p), prev);
        at(p) = prev;
      }
      p += d;
      const R tt = addop ? A::add(at(p), prev) : A::sub(at(p), prev);
      at(p) = A::mul(R(0.5), tt);
    }
  }
  __syncthreads();
}

template <int V, typename R, int LOGN, int LOGLB>
struct Cfg : FastCfg<V, R, LOGN, LOGLB> {
  static constexpr int V_ = V;
  static constexpr int LOGLB_ = LOGLB;
  static constexpr int LOGN_ = LOGN;
};

template <int V, typename R, int LOGN, int LOGLB>
__global__ void __launch_bounds__(Cfg<V, R, LOGN, LOGLB>::NT)
k_fast(const R* __restrict__ in, R* __restrict__ out, size_t rows,
       const R* __restrict__ tab, int nmax, int inverse, R scale) {
  using C = Cfg<V, R, LOGN, LOGLB>;
  using A = Arith<R>;
  using V2 = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  R* Tb = reinterpret_cast<R*>(smraw);
  R* Fb = Tb + 4 * C::CS;
  const int tid = threadIdx.x;
  const R base = __ldg(tab + (nmax / 4 - 1));
  constexpr int N = C::N, H = C::H;

  for (size_t row = blockIdx.x; row < rows; row += gridDim.x) {
    // ---- load: SplitComplex (elab.cpp:152-155) + SplitReal (185-197)
    const V2* x = reinterpret_cast<const V2*>(in + row * 2 * N);
    for (int m = tid; m <= H; m += C::NT) {
      V2 a = x[m];
      if (inverse) { const R tmp = a.x; a.x = a.y; a.y = tmp; }
      if (m == 0 || m == H) {
        Tb[0 * C::CS + ph<LOGLB>(m)] = a.x;
        Tb[2 * C::CS + ph<LOGLB>(m)] = a.y;
      } else {
        V2 b = x[N - m];
        if (inverse) { const R tmp = b.x; b.x = b.y; b.y = tmp; }
        Tb[0 * C::CS + ph<LOGLB>(m)] = A::add(a.x, b.x);
        Tb[1 * C::CS + ph<LOGLB>(m)] = A::sub(a.x, b.x);
        Tb[2 * C::CS + ph<LOGLB>(m)] = A::add(a.y, b.y);
        Tb[3 * C::CS + ph<LOGLB>(m)] = A::sub(a.y, b.y);
      }
    }
    __syncthreads();

    if (C::TM) {
#pragma unroll 1
      for (int lvl = 1; lvl <= C::LT; ++lvl) {
        mirror_level<C, R, true>(Tb, lvl, H >> (lvl - 1), tab, nmax, base);
        __syncthreads();
      }
    } else {
#pragma unroll 1
      for (int n = N; n >= 2 * (N / C::LB); n >>= 1) {
        chain_level<C, R, true>(Tb, n);
        __syncthreads();
      }
#pragma unroll 1
      for (int depth = 0; depth < C::LT; ++depth) am_level<C, R>(Tb, depth);
    }

    // ---- bottom: T -> F
    if (tid < C::NSEG) {
      const int half = C::HP / 2;
      const int h = tid % half;
      const int rest = tid / half;
      const int part = rest & 1, rho_bit = (rest >> 1) & 1, lam_bit = (rest >> 2) & 1;
      const int c = part * 2 + lam_bit;
      const int s = 2 * h + rho_bit;
      int rho, lens, r;
      seg_params<C::SINE>(lam_bit, s, C::LT, &rho, &lens, &r);
      Bottom<V, C::LB>::template run<R, A, LOGLB>(rho, lens, Tb + c * C::CS, Fb + c * C::CS,
                                                  s * C::LB, tab, nmax, base, N, C::LT, r,
                                                  lam_bit);
    } else if (tid < C::NSEG + 4) {
      const int c = tid - C::NSEG;
      Small<V, C::HP>::template run<R, A, LOGLB, C::LB>(c & 1, Tb + c * C::CS, Fb + c * C::CS,
                                                        base);
    }
    __syncthreads();

    if (C::TM) {
#pragma unroll 1
      for (int depth = C::LT - 1; depth >= 0; --depth) am_level<C, R>(Fb, depth);
#pragma unroll 1
      for (int n = 2 * (N / C::LB); n <= N; n <<= 1) {
        chain_level<C, R, false>(Fb, n);
        __syncthreads();
      }
    } else {
#pragma unroll 1
      for (int lvl = C::LT; lvl >= 1; --lvl) {
        mirror_level<C, R, false>(Fb, lvl, H >> (lvl - 1), tab, nmax, base);
        __syncthreads();
      }
    }

    // ---- store: SplitReal bwd (elab.cpp:199-208) + SplitComplex bwd (162-183)
    V2* y = reinterpret_cast<V2*>(out + row * 2 * N);
    for (int k = tid; k <= H; k += C::NT) {
      const R rd = Fb[0 * C::CS + ph<LOGLB>(k)];
      const R id = Fb[2 * C::CS + ph<LOGLB>(k)];
      V2 lo, hi;
      if (k == 0 || k == H) {
        lo.x = rd;
        lo.y = id;
      } else {
        const R rs = Fb[1 * C::CS + ph<LOGLB>(k)];
        const R is = Fb[3 * C::CS + ph<LOGLB>(k)];
        lo.x = A::add(rd, is);
        lo.y = A::sub(id, rs);
        hi.x = A::sub(rd, is);
        hi.y = A::add(id, rs);
      }
      if (inverse) {
        lo = V2{A::mul(lo.y, scale), A::mul(lo.x, scale)};
        hi = V2{A::mul(hi.y, scale), A::mul(hi.x, scale)};
      }
      y[k] = lo;
      if (k != 0 && k != H) y[N - k] = hi;
    }
    __syncthreads();
  }
}

template <int V, typename R, int LOGN, int LOGLB>
class FastPlanImpl final : public FastPlan {
 public:
  FastPlanImpl(const void* tab, uint32_t nmax, int device) : tab_(static_cast<const R*>(tab)),
                                                              nmax_(nmax) {
    using C = Cfg<V, R, LOGN, LOGLB>;
    auto fn = k_fast<V, R, LOGN, LOGLB>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM));
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::NT, C::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = std::max(1, per_sm) * sms;
    launches = 1;
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    using C = Cfg<V, R, LOGN, LOGLB>;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(rows, static_cast<size_t>(grid_cap_)));
    k_fast<V, R, LOGN, LOGLB><<<grid, C::NT, C::SMEM, st>>>(
        static_cast<const R*>(in), static_cast<R*>(out), rows, tab_, static_cast<int>(nmax_),
        inverse, R(1) / R(C::N));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }

 private:
  const R* tab_;
  uint32_t nmax_;
  int grid_cap_ = 148;
};

template <int V, typename R>
std::unique_ptr<FastPlan> make_for_variant(size_t n, const void* tab, uint32_t nmax, int dev) {
  if constexpr (sizeof(R) == 4) {
    switch (n) {
      case 1024: return std::make_unique<FastPlanImpl<V, R, 10, 5>>(tab, nmax, dev);
      case 2048: return std::make_unique<FastPlanImpl<V, R, 11, 6>>(tab, nmax, dev);
      case 4096: return std::make_unique<FastPlanImpl<V, R, 12, 6>>(tab, nmax, dev);
      case 8192: return std::make_unique<FastPlanImpl<V, R, 13, 6>>(tab, nmax, dev);
    }
  } else {
    switch (n) {
      case 1024: return std::make_unique<FastPlanImpl<V, R, 10, 5>>(tab, nmax, dev);
      case 2048: return std::make_unique<FastPlanImpl<V, R, 11, 5>>(tab, nmax, dev);
      case 4096: return std::make_unique<FastPlanImpl<V, R, 12, 5>>(tab, nmax, dev);
    }
  }
  return nullptr;
}

}  // namespace fastk
}  // namespace amqft_b200
