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
// Arithmetic goes through KArith<R>: fp64 = Arith<double> (__dadd_rn ...,
// no FMA contraction), so the fp64 instantiation reproduces the reference
// bitwise (serial recurrences included); the fp32 instantiation is the fast
// path (contractable operators).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "fast.cuh"
// The fused kernel reads the AM constant table from its parameter space:
// the generated code's compile-time slots become constant-bank operands.
#define AMQFT_TABLD(t, i) ((t)[i])
#include "gen/fast_gen.cuh"   // generated at build time by codegen/gen_fast.py
#include "generic.cuh"
#include "trig.hpp"

#ifndef AMQFT_RPC
#define AMQFT_RPC 2   // rows per CTA (fp32, N <= 4096): both rows' warps run each phase in lockstep
#endif
#ifndef AMQFT_TMA_STAGE
#define AMQFT_TMA_STAGE 1   // stage the next row with cp.async.bulk (else direct loads)
#endif
#ifndef AMQFT_SLOT_BARRIER
#define AMQFT_SLOT_BARRIER 1
#endif
#ifndef AMQFT_TMA_STORE
#define AMQFT_TMA_STORE 1   // fp32 N <= 4096: assemble the output row in smem, one bulk store
#endif

namespace amqft_b200 {
namespace fastk {

// Kernel arithmetic.  fp64: Arith<double> (__dadd_rn..., never contracted),
// so the fp64 instance stays bitwise the reference.  fp32 (the fast path,
// checked against the fp64 oracle within 1e-5 log2 N): plain operators,
// which nvcc may contract into FFMA where a constant multiply feeds an add
// (one instruction instead of two; FFMA rounds once, so it is never less
// accurate than FMUL + FADD).
#ifndef AMQFT_FP32_CONTRACT
#define AMQFT_FP32_CONTRACT 1
#endif
// Measured (B200, config-2 shapes): contraction speeds up N = 4096 by 3-4 %
// (all variants) but slows N = 1024 / 2048 / 8192 by 2-10 %, so it is used
// at N = 4096 only.
template <typename R, int LOGN> struct KArith : Arith<R> {};
struct ContractF {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
};
#if AMQFT_FP32_CONTRACT
template <> struct KArith<float, 12> : ContractF {};
#endif

__device__ __forceinline__ int parity(unsigned x) { return __popc(x) & 1; }

// Kernel-parameter copy of the constant table (N/4 values: 4-8 KB).
template <typename R, int K>
struct TabParam {
  R v[K];
};

// IO: the element type of the rows in HBM (and of the TMA staging buffer);
// R: the arithmetic type.  IO = float with R = double is the fp32-I/O,
// fp64-compute instance for the sine-family variants 5-8, whose recurrences
// amplify rounding beyond the fp32 tolerance from N = 512 on (SURVEY §8(c)
// item 2): the DAG and its fp64 rounding are the reference's, only the
// final result is rounded to fp32.
// P > 1: the cluster four-step (k_fast with P CTAs per transform of length
// P N, one length-N row per CTA; see cluster_exchange below).
template <int V, typename R, int LOGN, int LOGLB, typename IO = R, int P = 1>
struct Cfg {
  static constexpr int V_ = V;
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGN_ = LOGN;
  static constexpr int H = N / 2;
  static constexpr int LOGH = LOGN - 1;
  static constexpr int LB = 1 << LOGLB;
  static constexpr int LOGLB_ = LOGLB;
  static constexpr int LT = LOGH - LOGLB;        // depth of the bottom segments
  static constexpr int HP = H / LB;               // cells at multiples of LB
  static constexpr int NSEG = 4 * HP;             // bottom segments (4 chains)
  // threads: top levels use 4*LB, the AM phase 8 warps, the bottom 4 warps
  // (N <= 4096: + 4 small-chain lanes on the others) or NSEG = 256 threads
  // (N = 8192: + two warps for the small chains, one per lam)
  static constexpr int NT0 = (4 * LB > NSEG + 64 ? 4 * LB : NSEG + 64);
  static constexpr int NT = NSEG >= 256 ? NT0 : 256;
  // chain stride: holds the skewed (H + H/LB + 1) and the swizzled
  // (32-aligned blocks up to H) layouts; +16 staggers the chains' banks.
  static constexpr int CS = ((H + HP + 1 > H + H / 32 + 1 ? H + HP + 1 : H + H / 32 + 1) + 31) / 32 * 32 + 16;
  static constexpr bool TM = (V == 1 || V == 4 || V == 5 || V == 8);
  static constexpr int SINE = V >= 5 ? 1 : 0;
  static constexpr bool CHAIN = (V == 1 || V == 5 || V == 3 || V == 7);
  // Serial recurrences in the reference's order (one thread per class):
  // only the fp64 instance that must stay bitwise the reference.  fp32 and
  // the fp32-I/O fp64 instance evaluate them as segmented warp scans
  // (re-associated; for the fp64-compute instance the difference to the
  // serial order is fp64 rounding, far below the fp32 output rounding).
  static constexpr bool SERIAL = CHAIN && sizeof(R) == 8 && std::is_same<IO, R>::value;
  // top-level constants in tensor memory (fp32 instances, see tmem_ld)
#ifndef AMQFT_TOP_TMEM
#define AMQFT_TOP_TMEM 1
#endif
  static constexpr bool TOP_TMEM = AMQFT_TOP_TMEM && sizeof(R) == 4;
  // T, F (4 chains each) + the TMA staging buffer for the next row + mbarrier
  static constexpr size_t STAGE_OFF = 8 * CS * sizeof(R);
  // + mbarriers: the TMA stage (P == 1) / prefetch, staging-full, staging-free (P > 1)
  static constexpr size_t SMEM = AMQFT_TMA_STAGE ? STAGE_OFF + 2 * N * sizeof(IO) + (P > 1 ? 32 : 16) : STAGE_OFF;
  // Rows per CTA: two fp32 rows (N <= 4096) share one 512-thread CTA, each
  // with its own T/F/staging slot; every phase runs on both rows' warps at
  // once, so the phase's straight-line code is fetched once per SM for two
  // rows (instruction fetch was the top stall with one row per CTA).
  // Measured (B200, config 2, tools/ab_kernel.py, with the bulk store):
  // v4 1.646 -> 1.600 ms, v2 1.741 -> 1.568, v3 2.327 -> 1.936 against one
  // row per CTA (two CTAs per SM).
#ifdef AMQFT_RPC_FORCE   // A/B builds (tools/ab_kernel.cu)
  static constexpr int RPC = (P == 1 && sizeof(R) == 4 && LOGN <= 12) ? AMQFT_RPC_FORCE : 1;
#else
  static constexpr int RPC = (P == 1 && sizeof(R) == 4 && LOGN <= 12) ? AMQFT_RPC : 1;
#endif
  static constexpr int NTB = NT * RPC;
  static constexpr size_t SLOT = (SMEM + 127) / 128 * 128;
  static constexpr size_t SMEM_BLOCK = SLOT * RPC;
  // Bank-conflict layouts: skew (i + i/LB) on the buffer holding the
  // index-space mirror network (T for time-major, F for harmonic-major);
  // one pad word per 32 (i + i/32) on the other one (per-lane class runs,
  // recombination sets j*64 +- k at immediate offsets).
  // The pad is shifted per chain (31 for Dct chains, 0 for Dst chains) so
  // every lane's 32-cell class run lies inside one padded block.
  // Chain bases.  The bottom's warps pair chain c with chain c+2 (same
  // orientation and lens, so no divergence); the Im chains are shifted so
  // the two halves of the warp hit disjoint banks: by 1 word on the skewed
  // buffer (lanes cover even banks) and by 16 on the padded one (lanes
  // cover a 16-bank half).  Modelled in tools/bank_model.cpp.
  static constexpr int SH_SKEW = 1, SH_SWZ = 16;
  static __host__ __device__ __forceinline__ constexpr int co_sk(int c) { return c * CS + (c >> 1) * SH_SKEW; }
  static __host__ __device__ __forceinline__ constexpr int co_sw(int c) { return c * CS + (c >> 1) * SH_SWZ; }
  static __host__ __device__ __forceinline__ constexpr int coT(int c) { return TM ? co_sk(c) : co_sw(c); }
  static __host__ __device__ __forceinline__ constexpr int coF(int c) { return TM ? co_sw(c) : co_sk(c); }
  static __device__ __forceinline__ int skew(int i) { return i + (i >> LOGLB); }
  static __device__ __forceinline__ int swz(int i, int lam) { return i + ((i + (lam ? 0 : 31)) >> 5); }
  // The index-space buffer (T time-major, F harmonic-major) stores odd
  // LB-segments reversed (cell a + u at a + LB - u, 0 < u < LB), skewed.
  // A reversed segment is exactly the orientation-1 segment of the mirror
  // network (fast_model: rho = 1 swaps the roles of a + v and a + L - v at
  // every level), so the bottom runs one code path (rho = 0) for every
  // segment and the top's cells are all B + v + s (LB + 1).
  static __device__ __forceinline__ int ipos(int i) {
    const int s = i >> LOGLB, u = i & (LB - 1);
    const int j = ((s & 1) && u) ? i + LB - 2 * u : i;
    return j + s;
  }
  static __device__ __forceinline__ int pt(int i, int lam) { return TM ? ipos(i) : swz(i, lam); }
  static __device__ __forceinline__ int pf(int i, int lam) { return TM ? swz(i, lam) : ipos(i); }
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

// Dct/Dst chain recombination (time-major backward, FWD=false) or fold
// (harmonic-major forward, FWD=true) at size n on an unskewed buffer.
template <class C, typename R, bool FWD>
__device__ __forceinline__ void chain_level(R* B, int n, int tid) {
  using A = KArith<R, C::LOGN_>;
  const int q = n >> 2;
  const int lgq = 31 - __clz(q);
  for (int g = tid; g < n; g += C::NT) {
    const int c = g >> lgq;
    const int k = g & (q - 1);
    const int lam = c & 1;
    if (lam && k == 0) continue;
    R* ch = B + C::co_sw(c);
    const int i0 = C::swz(k, lam), i1 = C::swz((n >> 1) - k, lam);
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

// ---- Serial AM recurrences (variants 1,3,5,7): AM_B M1/M5
// (elaborations.cpp:472-513) or AM_F M3/M7 (402-448) along each odd class
// of the big top blocks, one thread per class, in place (swizzled buffer).
template <class C, int DEPTH, typename R>
__device__ __forceinline__ void chain_class(R* ch, int lam_c, int t, int r) {
  using A = KArith<R, C::LOGN_>;
  constexpr int V = C::V_;
  constexpr int stride = 2 << DEPTH;
  const int q = C::N >> (t + DEPTH + 3);
  const int lens = (C::SINE && DEPTH > 0) ? ((r >> (DEPTH - 1)) & 1) : lam_c;
  const int rO = r + ((1 - lens) << DEPTH);
  const int hi = (C::N >> (t + 1)) - lam_c;
  const int c0 = hi - rO;
  auto at = [&](int jj) -> R& { return ch[C::swz(c0 - jj * stride, lam_c)]; };
  // M1: cos asc/sub, sin desc/sub; M5: cos desc/add, sin asc/add (AM_B);
  // M3: cos desc/sub, sin asc/sub; M7: cos asc/add, sin desc/add (AM_F)
  const bool addop = C::TM ? (V == 5) : (V == 7);
  const bool desc = C::TM ? ((V == 1) ? (lens == 1) : (lens == 0)) : ((V == 3) ? (lens == 0) : (lens == 1));
  const int s0 = desc ? q - 1 : 0, d = desc ? -1 : 1;
  // The recurrence runs in the reference's serial order (bitwise); the
  // operands stream through registers a run of KC at a time (independent
  // loads issued together), so each step costs one dependent add instead of
  // a shared-memory round trip.
  constexpr int KC = 8;
  R prev = R(0);
  auto step = [&](R& v, int k) {
    if (C::TM) {            // y_0 = C_0 / 2, y_k = C_k -/+ y_(k-1)
      prev = k == 0 ? A::mul(R(0.5), v) : (addop ? A::add(v, prev) : A::sub(v, prev));
      v = prev;
    } else if (k == 0) {    // y_0 = C_0, y_k = C_k -/+ y_(k-1), the last one halved
      prev = v;
    } else {
      const R y = addop ? A::add(v, prev) : A::sub(v, prev);
      v = k == q - 1 ? A::mul(R(0.5), y) : y;
      prev = y;
    }
  };
  if (q >= KC) {            // q is a power of two: whole runs, no predicates
#pragma unroll 1
    for (int k0 = 0; k0 < q; k0 += KC) {
      R v[KC];
#pragma unroll
      for (int i = 0; i < KC; ++i) v[i] = at(s0 + (k0 + i) * d);
#pragma unroll
      for (int i = 0; i < KC; ++i) step(v[i], k0 + i);
#pragma unroll
      for (int i = 0; i < KC; ++i) at(s0 + (k0 + i) * d) = v[i];
    }
  } else {
#pragma unroll 1
    for (int k = 0; k < q; ++k) {
      R v = at(s0 + k * d);
      step(v, k);
      at(s0 + k * d) = v;
    }
  }
}

template <class C, int DEPTH, typename R>
__device__ __forceinline__ void am_chains(R* B, int tid) {
  // one thread per odd class (serial recurrence); classes with m <= 2 skip
  int idx = tid;
  constexpr int classes = 1 << DEPTH;
  for (int g = idx; g < 4 * C::LOGLB_ * classes; g += C::NT) {
    const int c = g / (C::LOGLB_ * classes);
    const int rem = g - c * (C::LOGLB_ * classes);
    const int t = rem / classes;
    const int r = rem - t * classes;
    const int q = C::N >> (t + DEPTH + 3);
    if (q < 2) continue;
    chain_class<C, DEPTH, R>(B + C::co_sw(c), c & 1, t, r);
  }
  __syncthreads();
}

template <class C, int DEPTH, typename R>
__device__ __forceinline__ void am_level(R* B, int tid) {
  am_chains<C, DEPTH, R>(B, tid);
}

// Depth loops unrolled at compile time.
template <class C, typename R, int D>
__device__ __forceinline__ void am_levels_desc(R* B, int tid) {  // D-1 .. 0
  if constexpr (D > 0) {
    am_level<C, D - 1, R>(B, tid);
    am_levels_desc<C, R, D - 1>(B, tid);
  }
}
template <class C, typename R, int D, int I = 0>
__device__ __forceinline__ void am_levels_asc(R* B, int tid) {  // 0 .. D-1
  if constexpr (I < D) {
    am_level<C, I, R>(B, tid);
    am_levels_asc<C, R, D, I + 1>(B, tid);
  }
}

// ---- Register-resident AM phase (non-recurrent variants 2,4,6,8).
// Every odd-class neighbour operation of every depth for the big top
// blocks (t < log2 LB) runs out of registers: warp pair (2c, 2c+1) owns
// chain c; top block 0 is one warp, blocks 1.. share the second warp; each
// lane owns RR = N/128 consecutive positions of its block (natural order,
// cell(p) = hi - p).  Halo values cross lanes with warp shuffles; the last
// lane of a block takes the class-end copy, so segment boundaries inside a
// warp never consume foreign data.
template <class C, bool BWD, int LAM, int D>
struct AmPos {
  static constexpr int V = C::V_;
  static constexpr int RR = C::N / 128;
  static constexpr int S = 2 << D;
  // low bits of the block position p = i*RR + l are those of l (S <= RR)
  static constexpr int lens(int l) { return (C::SINE && D > 0) ? ((l >> (D - 1)) & 1) : LAM; }
  static constexpr bool is_o(int l) { return ((l >> D) & 1) == 1 - lens(l); }
  static constexpr bool right(int l) {
    return BWD ? ((V == 4) ? (lens(l) == 0) : (lens(l) == 1))    // AM_B M4 / M8
               : ((V == 2) ? (lens(l) == 1) : (lens(l) == 0));   // AM_F M2 / M6
  }
};

template <class C, typename R, bool BWD, int LAM, int D>
__device__ __forceinline__ void am_depth(R (&x)[C::N / 128], bool last_lane, bool first_lane,
                                         bool blk_ok) {
  using A = KArith<R, C::LOGN_>;
  using P = AmPos<C, BWD, LAM, D>;
  constexpr int RR = P::RR, S = P::S;
  constexpr bool ADD = BWD ? (C::V_ == 4) : (C::V_ == 2);
  static_assert(S <= RR, "class stride must fit a lane's run");
  // 1) halos (pre-update values of the neighbour lane), only the ones used
  R hr[S], hl[S];
#pragma unroll
  for (int l = RR - S; l < RR; ++l)
    if (P::is_o(l) && P::right(l)) hr[l + S - RR] = __shfl_down_sync(0xffffffffu, x[l + S - RR], 1);
#pragma unroll
  for (int l = 0; l < S; ++l)
    if (P::is_o(l) && !P::right(l)) hl[l] = __shfl_up_sync(0xffffffffu, x[l - S + RR], 1);
  if (!blk_ok) return;
  // 2) right-halo ops ascending, left-halo ops descending: in place, every
  //    neighbour read happens before that neighbour is updated.
#pragma unroll
  for (int l = 0; l < RR; ++l) {
    if (!(P::is_o(l) && P::right(l))) continue;
    const R cj = x[l];
    const R cn = (l + S < RR) ? x[(l + S) % RR] : hr[(l + S) % RR];
    const R o = ADD ? A::add(cj, cn) : A::sub(cj, cn);
    x[l] = (l + S >= RR && last_lane) ? cj : o;     // class end: copy
  }
#pragma unroll
  for (int l = RR - 1; l >= 0; --l) {
    if (!(P::is_o(l) && !P::right(l))) continue;
    const R cj = x[l];
    const R cn = (l - S >= 0) ? x[(l - S + RR) % RR] : hl[l % S];
    const R o = ADD ? A::add(cj, cn) : A::sub(cj, cn);
    x[l] = (l - S < 0 && first_lane) ? cj : o;      // class start: copy
  }
}

// ---- Serial recurrences (variants 1,3,5,7) as warp scans, fp32 only.
// AM_B M1/M5 (elaborations.cpp:472-513): y_0 = C_0/2, y_k = C_k -/+ y_(k-1);
// AM_F M3/M7 (elaborations.cpp:402-448): y_0 = C_0, y_k = C_k -/+ y_(k-1),
// last y halved.  Along one odd class in its direction, y is a chain of
// affine maps y -> C + s y (s = -1 sub, +1 add): each lane scans its own
// RR/S elements, the lanes of a block combine their (A, s^m) aggregates
// with a segmented shuffle scan, and every element is fixed up with the
// prefix from the lanes before it.  Re-associated, so only the fp32 fast
// path uses it; fp64 keeps the reference's serial order (bitwise).
template <class C, typename R, bool BWD, int LAM, int D>
__device__ __forceinline__ void am_scan_depth(R (&x)[C::N / 128], int i, int nl, bool blk_ok) {
  using A = KArith<R, C::LOGN_>;
  using P = AmPos<C, BWD, LAM, D>;
  constexpr int V = C::V_;
  constexpr int RR = P::RR, S = P::S, M = RR / S;
  constexpr bool ADD = BWD ? (V == 5) : (V == 7);
  static_assert(S <= RR, "class stride must fit a lane's run");
#pragma unroll
  for (int rho = 0; rho < S; ++rho) {
    if (!P::is_o(rho)) continue;
    const int lens = P::lens(rho);
    const bool desc = BWD ? ((V == 1) ? (lens == 1) : (lens == 0))    // M1 / M5
                          : ((V == 3) ? (lens == 0) : (lens == 1));   // M3 / M7
    const int pos = desc ? (nl - 1 - i) : i;       // lane rank in the class direction
    // local inclusive scan of this lane's elements (in direction), y_in = 0
    R loc[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int l = rho + (desc ? (M - 1 - j) : j) * S;
      R e = x[l];
      if (BWD && j == 0 && pos == 0) e = A::mul(R(0.5), e);   // AM_B seed C_0 / 2
      loc[j] = j == 0 ? e : (ADD ? A::add(e, loc[j - 1]) : A::sub(e, loc[j - 1]));
    }
    // segmented inclusive scan of the lane aggregates (A, s^M) over the block
    R acc = loc[M - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const R o = desc ? __shfl_down_sync(0xffffffffu, acc, d) : __shfl_up_sync(0xffffffffu, acc, d);
      const bool neg = !ADD && (M & 1) && (d & 1);            // factor s^(M d)
      if (pos >= d) acc = neg ? A::sub(acc, o) : A::add(acc, o);
    }
    // exclusive prefix without another shuffle: acc = A_own + s^M y_in
    constexpr bool SIGN_NEG = !ADD && (M & 1);
    R yin = SIGN_NEG ? A::sub(loc[M - 1], acc) : A::sub(acc, loc[M - 1]);
    if (pos == 0) yin = R(0);
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int l = rho + (desc ? (M - 1 - j) : j) * S;
      const bool negj = !ADD && ((j & 1) == 0);               // s^(j+1)
      R y = negj ? A::sub(loc[j], yin) : A::add(loc[j], yin);
      if (!BWD && j == M - 1 && pos == nl - 1) y = A::mul(R(0.5), y);   // AM_F final halving
      if (blk_ok) x[l] = y;
    }
  }
}

template <class C, typename R, bool BWD, int LAM>
__device__ __forceinline__ void am_depths(R (&x)[C::N / 128], bool last_lane, bool first_lane,
                                          int Mt, int i, int nl) {
  auto step = [&](auto dtag) {
    constexpr int D = decltype(dtag)::value;
    if constexpr (C::CHAIN)
      am_scan_depth<C, R, BWD, LAM, D>(x, i, nl, (Mt >> (D + 1)) >= 2);
    else
      am_depth<C, R, BWD, LAM, D>(x, last_lane, first_lane, (Mt >> (D + 1)) >= 2);
  };
  static_assert(C::LT <= 6, "depth range");
  if constexpr (BWD) {
    if constexpr (C::LT > 5) step(std::integral_constant<int, 5>());
    if constexpr (C::LT > 4) step(std::integral_constant<int, 4>());
    if constexpr (C::LT > 3) step(std::integral_constant<int, 3>());
    if constexpr (C::LT > 2) step(std::integral_constant<int, 2>());
    if constexpr (C::LT > 1) step(std::integral_constant<int, 1>());
    step(std::integral_constant<int, 0>());
  } else {
    step(std::integral_constant<int, 0>());
    if constexpr (C::LT > 1) step(std::integral_constant<int, 1>());
    if constexpr (C::LT > 2) step(std::integral_constant<int, 2>());
    if constexpr (C::LT > 3) step(std::integral_constant<int, 3>());
    if constexpr (C::LT > 4) step(std::integral_constant<int, 4>());
    if constexpr (C::LT > 5) step(std::integral_constant<int, 5>());
  }
}

template <class C, typename R, bool BWD>
__device__ __forceinline__ void am_phase_regs(R* B, int tid) {
  constexpr int RR = C::N / 128;
  constexpr int LOGR = C::LOGN_ - 7;
  const int warp = tid >> 5, lane = tid & 31;
  const int c = warp >> 1;
  int t, i;
  if ((warp & 1) == 0) {
    t = 0;
    i = lane;
  } else {
    t = 1 + (lane >= 16) + (lane >= 24) + (lane >= 28) + (lane >= 30) + (lane >= 31);
    i = lane - (32 - (64 >> t));
  }
  const bool active = warp < 8 && t < C::LOGLB_;
  const int tt = active ? t : 0;
  const int lam_c = c & 1;
  const int Mt = C::N >> (tt + 2);
  const int nl = 32 >> tt;                       // lanes of this block
  const int cell0 = (C::N >> (tt + 1)) - lam_c - (i << LOGR);
  // runs end on a padded-block boundary: phys(cell0 - l) = phys(cell0) - l - l/32
  R* chb = B + C::co_sw(c & 3) + C::swz(cell0, lam_c);
  R x[RR];
#pragma unroll
  for (int l = 0; l < RR; ++l) x[l] = active ? chb[-(l + (l >> 5))] : R(0);
  const bool last_lane = i == nl - 1, first_lane = i == 0;
  if (lam_c) am_depths<C, R, BWD, 1>(x, last_lane, first_lane, Mt, i, nl);
  else am_depths<C, R, BWD, 0>(x, last_lane, first_lane, Mt, i, nl);
  if (active) {
#pragma unroll
    for (int l = 0; l < RR; ++l) chb[-(l + (l >> 5))] = x[l];
  }
}

// ---- Multiples of 32 (the k = 0 class of the generated recombination,
// N = 4096: cells y = 32 i, i in [0, 64], physical 33 i in both pads), one
// warp per chain instead of one serial lane: lane l holds i = l and
// i = 64 - l, lane 0 also i = 32.  Level t (n = 128 << t) pairs
// (i, 2^(t+1) - i), i < 2^t: in-lane at t = 5 and for lane 0 at t = 4,
// one shuffle otherwise.  Same operations and operand order as
// codegen/gen_fast.py emit_pair (Dct chains use every cell; Dst chains skip
// i = 0 and i = 64), so the fp64 instance stays bitwise.
template <typename R, bool FOLD, int LAM, int LG>
__device__ __forceinline__ void pair_op(R e, R o, R& e2, R& o2) {
  using A = KArith<R, LG>;
  if (!FOLD) {  // SplitTimeParity bwd (elaborations.cpp:310-329)
    e2 = LAM ? A::add(o, e) : A::add(e, o);
    o2 = LAM ? A::sub(o, e) : A::sub(e, o);
  } else {      // SplitHarmonicParity fwd (elaborations.cpp:238-255)
    e2 = LAM ? A::sub(e, o) : A::add(e, o);
    o2 = LAM ? A::add(e, o) : A::sub(e, o);
  }
}

// Predicated (no lane-dependent branches): every lane evaluates the pair
// op and keeps its result only where it owns a cell of the pair.
// General form for HW in {8, 16, 32}: cells i in [0, 2 HW] (y = i W/2,
// physical ST i), lane l holds i = l (l <= 2 HW), for HW = 32 also
// i = 64 - l, for HW >= 16 lane 0 also i = 32; levels t = 0 .. log2 HW.
template <typename R, bool FOLD, int LAM, int HW, int ST, int LG>
__device__ __forceinline__ void special_class_l(R* ch, int lane) {
  static_assert(HW == 8 || HW == 16 || HW == 32, "special class size");
  constexpr int NC = 2 * HW;
  constexpr int TMAX = HW == 32 ? 5 : (HW == 16 ? 4 : 3);
  const bool has = lane <= NC;
  R a = has ? ch[ST * lane] : R(0);
  R b = HW == 32 ? ch[ST * (64 - lane)] : R(0);
  R m = HW >= 16 ? ch[ST * 32] : R(0);             // used by lane 0 only
  const bool own0 = !(LAM && lane == 0);           // Dst chains: no cell 0 / 2 HW
  auto level = [&](int t) {
    R e2, o2;
    if (t == 5) {                                  // in-lane pairs (i, 64 - i)
      pair_op<R, FOLD, LAM, LG>(a, b, e2, o2);
      a = own0 ? e2 : a;
      b = own0 ? o2 : b;
      return;
    }
    const int P = 2 << t, Hh = 1 << t;
    const int src = lane <= P ? (P - lane) & 31 : lane;
    const R pv = __shfl_sync(0xffffffffu, a, src);
    const R other = (t == 4 && lane == 0) ? m : pv;
    const bool lower = lane < Hh && own0;
    const bool upper = lane > Hh && lane <= P && !(LAM && lane == P);
    pair_op<R, FOLD, LAM, LG>(lower ? a : other, lower ? other : a, e2, o2);
    if (t == 4 && lane == 0 && !LAM) m = o2;
    a = lower ? e2 : (upper ? o2 : a);
  };
  if (FOLD) {
#pragma unroll
    for (int t = TMAX; t >= 0; --t) level(t);
  } else {
#pragma unroll
    for (int t = 0; t <= TMAX; ++t) level(t);
  }
  if (own0 && has) ch[ST * lane] = a;
  if (HW == 32 && own0) ch[ST * (64 - lane)] = b;
  if (HW >= 16 && lane == 0 && !LAM) ch[ST * 32] = m;
}

template <typename R, bool FOLD, int HW, int ST, int LG>
__device__ __forceinline__ void special_class(R* ch, int lam, int lane) {
  if (lam) special_class_l<R, FOLD, 1, HW, ST, LG>(ch, lane);   // warp-uniform
  else special_class_l<R, FOLD, 0, HW, ST, LG>(ch, lane);
}

// Recombination (TM, FOLD = false) / fold (HM, FOLD = true) of all four
// chains on buffer B for n = 2N/LB .. N: generated thread sets {j WR +- k}
// (WR = max(64, N/LB)) for n >= 2 WR, the levels below 2 WR level by level;
// the k = 0 class (multiples of WR/2) cooperatively, one warp per chain.
// Every thread of the row calls it (it contains the row barriers).
template <class C, typename R, bool FOLD, class Sync>
__device__ __forceinline__ void recombine(R* B, int tid, bool act, Sync row_sync) {
  using A = KArith<R, C::LOGN_>;
  constexpr int N = C::N, H = C::H;
  constexpr int WR = (N / C::LB > 64) ? N / C::LB : 64;
  constexpr int HWR = H / WR;
  constexpr int ST = WR / 2 + WR / 64;
  constexpr int n0 = 2 * (N / C::LB);
  constexpr int GT = 2 * WR;                       // generated-set threads (4 chains x WR/2)
  auto pre = [&]() {
    if constexpr (!FOLD) {
#pragma unroll 1
      for (int n = n0; n < 2 * WR; n <<= 1) {
        if (act) chain_level<C, R, false>(B, n, tid);
        row_sync();
      }
    }
  };
  auto post = [&]() {
    if constexpr (FOLD) {
#pragma unroll 1
      for (int n = WR; n >= n0; n >>= 1) {
        row_sync();
        if (act) chain_level<C, R, true>(B, n, tid);
      }
    }
  };
  pre();
  if (act) {
    if (tid < GT) {
      const int c = tid / (WR / 2), k = tid % (WR / 2);
      if (k) {
        if constexpr (FOLD) Recomb<WR, HWR>::template fold<R, A>(c & 1, B + C::co_sw(c), k);
        else Recomb<WR, HWR>::template run<R, A>(c & 1, B + C::co_sw(c), k);
      }
    } else if (GT == 128 && tid < 256) {
      const int c = (tid >> 5) - 4;
      special_class<R, FOLD, HWR, ST, C::LOGN_>(B + C::co_sw(c), c & 1, tid & 31);
    } else if (GT == 256 && tid >= 256 && tid < C::NT) {
      // spare warps 8.. take the four chains' k = 0 classes in turn
      constexpr int NW = (C::NT - 256) / 32;
#pragma unroll 1
      for (int c = (tid - 256) >> 5; c < 4; c += NW)
        special_class<R, FOLD, HWR, ST, C::LOGN_>(B + C::co_sw(c), c & 1, tid & 31);
    }
  }
  post();
}

// ---- TMA bulk staging of the next row (cp.async.bulk + mbarrier).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Bulk store smem -> global (cp.async.bulk, bulk-group completion).
__device__ __forceinline__ void bulk_store(void* gdst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_u32(src)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {   // smem source reusable
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {        // global writes complete
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- Tensor memory holds the top levels' constants (fp32 instances).
// Each top thread needs Top::NK distinct constants f(pi (u0 +- v) / L) that
// depend on its offset v only, the same for every row it processes; a
// warp's tcgen05.ld reads its TMEM lane quadrant (warp % 4), and every warp
// of a quadrant has the same v range (v = 32 (warp & 1) + lane), so one copy
// per quadrant, written once per kernel, serves every row.  The per-row
// constant loads leave the L1 / shared-memory data path (on which the
// kernel is bound) for tensor memory's own.
constexpr uint32_t kTmemCols = 64;
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// one warp: allocate kTmemCols columns, address to *dst (shared memory)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(dst)), "n"(kTmemCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kTmemCols) : "memory");
}
#define AMQFT_R8(a, o) "=r"(a[o]), "=r"(a[o + 1]), "=r"(a[o + 2]), "=r"(a[o + 3]), "=r"(a[o + 4]), "=r"(a[o + 5]), \
                       "=r"(a[o + 6]), "=r"(a[o + 7])
#define AMQFT_W8(a, o) "r"(a[o]), "r"(a[o + 1]), "r"(a[o + 2]), "r"(a[o + 3]), "r"(a[o + 4]), "r"(a[o + 5]), \
                       "r"(a[o + 6]), "r"(a[o + 7])
// 32x32b shape: lane l of the warp reads / writes columns [col, col + K) of
// TMEM lane 32 (warp % 4) + l (taddr carries lane << 16 | column)
template <int K>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[K]) {
  static_assert(K == 8 || K == 16 || K == 32 || K == 64, "TMEM load width");
  if constexpr (K == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : AMQFT_R8(r, 0) : "r"(taddr));
  } else {
#pragma unroll
    for (int c = 0; c < K; c += 8)   // x8 pieces: 8 registers per instruction
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : AMQFT_R8(r, c) : "r"(taddr + static_cast<uint32_t>(c)));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <int K>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[K]) {
#pragma unroll
  for (int c = 0; c < K; c += 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr + static_cast<uint32_t>(c)), AMQFT_W8(r, c) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
#undef AMQFT_R8
#undef AMQFT_W8
constexpr int pow2_at_least_8(int k) { return k <= 8 ? 8 : k <= 16 ? 16 : k <= 32 ? 32 : 64; }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// ---- Cluster four-step (P > 1): one transform of length P N per cluster of
// P CTAs, N = the fused kernel's row length.  Decimation in frequency,
// n = N n1 + n2, k = k1 + P k2:
//   X[k1 + P k2] = sum_n2 w_N^(n2 k2) [ w_(PN)^(n2 k1) sum_n1 x[N n1 + n2] w_P^(n1 k1) ]
// CTA q owns the chunk n2 in [q N/P, (q+1) N/P): its P input pieces (one
// per quarter n1, contiguous, every input byte read once chip-wide) are
// TMA-prefetched into the dead T buffer one row ahead; the P-point DFTs and
// the twiddle run in registers, and y_k1[n2] goes straight into CTA k1's
// staging row with st.async over DSMEM, completing bytes on CTA k1's
// "full" mbarrier (the only exchange: (P-1)/P of a row per CTA).  A CTA
// that has read its staging row arrives on every CTA's "free" mbarrier.
// Then every CTA runs the ordinary fused phases on its staged row and
// writes X[k1 + P k2] (stride P) to HBM.  The AM-QFT DAG runs inside each
// length-N row; fp32 error: the fused kernel's plus one P-point DFT and one
// twiddle rounding.
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// asynchronous remote store, completing its bytes on the remote mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, float2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               ::"r"(addr), "f"(v.x), "f"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, double2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(addr), "d"(v.x), "d"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t mbar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mbar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// In-register radix-2 DFT of P points (forward sign), w[k] = w_P^k.
template <int P, typename V2>
__device__ __forceinline__ void small_dft(V2 (&a)[P], const V2 (&w)[P]) {
  // bit-reversed order
#pragma unroll
  for (int i = 0; i < P; ++i) {
    int j = 0;
#pragma unroll
    for (int b = 1, t = i; b < P; b <<= 1, t >>= 1) j = (j << 1) | (t & 1);
    if (j > i) {
      const V2 t2 = a[i];
      a[i] = a[j];
      a[j] = t2;
    }
  }
#pragma unroll
  for (int len = 2; len <= P; len <<= 1) {
#pragma unroll
    for (int i = 0; i < P; i += len) {
#pragma unroll
      for (int j = 0; j < len / 2; ++j) {
        const V2 tw = w[j * (P / len)];
        const V2 u = a[i + j], b = a[i + j + len / 2];
        const V2 v{b.x * tw.x - b.y * tw.y, b.x * tw.y + b.y * tw.x};
        a[i + j] = V2{u.x + v.x, u.y + v.y};
        a[i + j + len / 2] = V2{u.x - v.x, u.y - v.y};
      }
    }
  }
}

// Prefetch of CTA q's P input pieces of big transform `row` into `dst`
// (piece n1 at dst + n1 N/P complex values), one TMA bulk copy each.
template <typename IO, int P, int N>
__device__ __forceinline__ void cluster_prefetch(const IO* __restrict__ xrow, void* dst, int q, uint64_t* bar) {
  constexpr uint32_t CHB = N / P * 2 * sizeof(IO);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(CHB * P) : "memory");
#pragma unroll 1
  for (int n1 = 0; n1 < P; ++n1)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(static_cast<unsigned char*>(dst) + n1 * CHB)),
                 "l"(xrow + (static_cast<size_t>(n1) * N + static_cast<size_t>(q) * (N / P)) * 2), "r"(CHB),
                 "r"(smem_u32(bar))
                 : "memory");
}

// The exchange: CTA q fills the staging rows of all P CTAs of its cluster
// from its prefetched pieces `src`.  ctw[j] = w_(PN)^j, j < P N (host long
// double, rounded to R).
template <typename R, typename IO, int P, int N, int NT, bool INV>
__device__ __forceinline__ void cluster_exchange(const IO* src, IO* Sb, uint64_t* full, int q, int tid,
                                                 const void* __restrict__ ctw_) {
  using V2 = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  using IO2 = typename std::conditional<sizeof(IO) == 4, float2, double2>::type;
  using E = decltype(IO2{}.x);
  const V2* ctw = static_cast<const V2*>(ctw_);
  constexpr int CH = N / P;   // n2 per CTA
  static_assert(CH % NT == 0, "exchange tiling");
  constexpr int IT = CH / NT;
  V2 w[P];
#pragma unroll
  for (int k = 0; k < P; ++k) w[k] = ctw[k * N];   // w_P^k = w_(PN)^(kN)
  const IO2* x2 = reinterpret_cast<const IO2*>(src);
  // peer windows: mapa once per peer (a CTA's window is linear)
  uint32_t rsb[P], rfb[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    rsb[k] = mapa(smem_u32(Sb), static_cast<uint32_t>(k));
    rfb[k] = mapa(smem_u32(full), static_cast<uint32_t>(k));
  }
  // w_(PN)^n2 for every n2 of the thread (coalesced, issued up front); the
  // powers w^(n2 k1) by repeated multiplication (P - 2 roundings at most)
  V2 w1[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) w1[it] = ctw[q * CH + it * NT + tid];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int j = it * NT + tid, n2 = q * CH + j;
    V2 a[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) {
      const IO2 v = x2[n1 * CH + j];
      a[n1] = INV ? V2{static_cast<R>(v.y), static_cast<R>(v.x)} : V2{static_cast<R>(v.x), static_cast<R>(v.y)};
    }
    small_dft<P>(a, w);
    V2 t = w1[it];
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      V2 y = a[k1];
      if (k1) {
        y = V2{y.x * t.x - y.y * t.y, y.x * t.y + y.y * t.x};
        if (k1 + 1 < P) t = V2{t.x * w1[it].x - t.y * w1[it].y, t.x * w1[it].y + t.y * w1[it].x};
      }
      st_async(rsb[k1] + static_cast<uint32_t>(n2) * sizeof(IO2), IO2{static_cast<E>(y.x), static_cast<E>(y.y)},
               rfb[k1]);
    }
  }
}

#ifdef AMQFT_PHASE_TIMING
// Instrumented build only (tools/phase_timing): CTA 0 accumulates, per
// phase, the cycles thread 0 spends between phase boundaries
// (g_phase_cycles) and, per warp, the cycles until the warp reaches the
// phase's barrier (g_warp_work[phase][warp]).
__device__ unsigned long long g_phase_cycles[16];
__device__ unsigned long long g_warp_work[16][16];
#define PHASE_MARK(k)                                                          \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                 \
      const long long now = clock64();                                         \
      if ((k) > 0) atomicAdd(&g_phase_cycles[(k) - 1], (unsigned long long)(now - t_prev)); \
      t_prev = now;                                                            \
    }                                                                          \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) w_start = clock64();       \
  } while (0)
#define WORK_MARK(k)                                                           \
  do {                                                                         \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                            \
      atomicAdd(&g_warp_work[k][threadIdx.x >> 5], (unsigned long long)(clock64() - w_start)); \
  } while (0)
#else
#define PHASE_MARK(k) do {} while (0)
#define WORK_MARK(k) do {} while (0)
#endif

// MODE 0: CDFT forward; 1: CDFT inverse (swap trick); 2: RDFT forward, two
// real rows per kernel row (row A -> chains 0/1, row B -> chains 2/3: the
// same Dct/Dst chains as the Re/Im halves of a CDFT, variants.cpp:190-209).
template <int V, typename R, int LOGN, int LOGLB, int MODE, typename IO = R, int P = 1>
#ifndef AMQFT_FAST_MINB
#define AMQFT_FAST_MINB 2
#endif
// min blocks per SM: 2 only where two CTAs fit in shared memory (one-row
// fp32 CTAs up to N = 4096); otherwise let ptxas use up to 255 registers
__global__ void __launch_bounds__(
#ifdef AMQFT_LB_THREADS   // register-budget experiments (tools/ab_kernel.cu)
                                  AMQFT_LB_THREADS,
#else
                                  Cfg<V, R, LOGN, LOGLB, IO, P>::NTB,
#endif
                                  ((Cfg<V, R, LOGN, LOGLB, IO, P>::RPC == 1 && sizeof(R) == 4 &&
                                    2 * Cfg<V, R, LOGN, LOGLB, IO, P>::SMEM_BLOCK <= 227 * 1024)
                                       ? AMQFT_FAST_MINB : 1))
k_fast(const IO* __restrict__ in, IO* __restrict__ out, size_t rows_in,
       const __grid_constant__ TabParam<R, (1 << LOGN) / 4> tparam, const R* __restrict__ ltab, int nmax_unused,
       R scale, const void* __restrict__ ctw) {
  (void)nmax_unused;
  // the plan compacts its table to Nmax = N (k_compact_table), so every
  // generated slot index is a compile-time constant into the parameter space
  const R* tab = tparam.v;
  constexpr int nmax = 1 << LOGN;
  constexpr bool INV = MODE == 1;
  constexpr bool RDFT = MODE == 2;
  // kernel rows: CDFT rows, or pairs of RDFT rows (the last one maybe single)
  const size_t rows = RDFT ? (rows_in + 1) / 2 : rows_in;
#ifdef AMQFT_PHASE_TIMING
  long long t_prev = 0, w_start = 0;
#endif
  using C = Cfg<V, R, LOGN, LOGLB, IO, P>;
  using A = KArith<R, C::LOGN_>;
  using V2 = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  static_assert(P == 1 || MODE != 2, "the cluster four-step runs CDFT rows");
  // P > 1: the swap-trick inverse swaps in the exchange (input of the whole
  // P N transform) and swaps + scales in the store
  constexpr bool INV_IN = MODE == 1 && P == 1;
  using IO2 = typename std::conditional<sizeof(IO) == 4, float2, double2>::type;
  // rows in HBM / staging (IO) <-> arithmetic (R)
  auto cvt_in = [](IO2 v) -> V2 { return V2{static_cast<R>(v.x), static_cast<R>(v.y)}; };
  auto cvt_out = [](V2 v) -> IO2 {
    using E = decltype(IO2{}.x);
    return IO2{static_cast<E>(v.x), static_cast<E>(v.y)};
  };
  extern __shared__ __align__(128) unsigned char smraw[];
  // row slot: threads [slot*NT, (slot+1)*NT) own row slot of each pair
  const int tid = threadIdx.x % C::NT;
  const int slot = threadIdx.x / C::NT;
  unsigned char* sm = smraw + slot * C::SLOT;
  R* Tb = reinterpret_cast<R*>(sm);
  R* Fb = Tb + 4 * C::CS;
  IO* Sb = reinterpret_cast<IO*>(sm + C::STAGE_OFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::STAGE_OFF + 2 * C::N * sizeof(IO));
  constexpr size_t RSTEP = C::RPC;   // rows per CTA iteration
  // Barrier of one row slot.  AMQFT_SLOT_BARRIER=1 (default): a named
  // barrier per slot, the two rows drift apart (measured 1.58 -> 1.54 ms,
  // v4); 0: the CTA barrier, both rows in lockstep.
  auto row_sync = [&]() {
    if constexpr (AMQFT_SLOT_BARRIER && C::RPC > 1)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(C::NT) : "memory");
    else
      __syncthreads();
  };
  const R base = tab[nmax / 4 - 1];
  // TMEM: the slot-0 barrier block's spare word holds the allocation address
  using TopT = Top<C::LB, C::LT, LOGN, C::SINE>;
  constexpr int NKP = pow2_at_least_8(TopT::NK);
  uint32_t tbase = 0;
  if constexpr (C::TOP_TMEM) {
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smraw + C::STAGE_OFF + 2 * C::N * sizeof(IO) + 8);
    if (threadIdx.x < 32) tmem_alloc(tslot);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tbase = *tslot;
    if (threadIdx.x < 128) {   // warp q fills quadrant q: v = 32 (q & 1) + lane
      const int v = 32 * ((threadIdx.x >> 5) & 1) + (threadIdx.x & 31);
      float kf[NKP];
#pragma unroll
      for (int j = 0; j < NKP; ++j) kf[j] = 0.0f;
      TopT::template fill<float>(kf, v, reinterpret_cast<const float*>(ltab), static_cast<float>(base));
      uint32_t kw[NKP];
#pragma unroll
      for (int j = 0; j < NKP; ++j) kw[j] = __float_as_uint(kf[j]);
      tmem_st<NKP>(tbase + ((threadIdx.x & 96u) << 16), kw);
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  // this warp's view of its quadrant's constants
  auto top_consts = [&](float (&kk)[NKP]) {
    uint32_t kw[NKP];
    tmem_ld<NKP>(tbase + ((threadIdx.x & 96u) << 16), kw);
#pragma unroll
    for (int j = 0; j < NKP; ++j) kk[j] = __uint_as_float(kw[j]);
  };
  (void)top_consts;
  constexpr int N = C::N, H = C::H;
  constexpr uint32_t ROW_BYTES = 2 * N * sizeof(IO);
  // load/store: 256 threads, cells tid + 256 it; address steps per it
  constexpr int IO_T = 256, IO_IT = H / IO_T;
  static_assert(H % IO_T == 0 && C::NT >= IO_T, "IO tiling");
  constexpr int IDX_STEP = IO_T + IO_T / C::LB;          // ipos: skew by segment
  constexpr int SWZ_STEP = IO_T + IO_T / 32;             // swz: one pad per 32
  constexpr int PT_STEP = C::TM ? IDX_STEP : SWZ_STEP;
  constexpr int PF_STEP = C::TM ? SWZ_STEP : IDX_STEP;
  // Output through a bulk store: the row is assembled in the F buffer (free
  // once read; next written by the following row's bottom phase, after
  // thread 0 has waited for the bulk read) and leaves with one cp.async.bulk.
  constexpr bool BULK_ST = P == 1 && AMQFT_TMA_STORE && sizeof(IO) == 4 && IO_IT <= 8 &&
                           4 * C::CS * sizeof(R) >= 2 * N * sizeof(IO);
  // cluster four-step: cluster id / count, this CTA's k1
  const size_t cl_id = P > 1 ? blockIdx.x / P : 0, cl_n = P > 1 ? gridDim.x / P : 1;
  const int q = P > 1 ? static_cast<int>(cluster_rank()) : 0;
  (void)q;
  // P > 1: bar = the prefetch of this CTA's input pieces (into T), full =
  // the staging row's bytes from the P exchangers, freeb = all P CTAs have
  // read their staging rows (one remote arrive each)
  uint64_t* full = bar + 1;
  uint64_t* freeb = bar + 2;
  (void)full;
  (void)freeb;
#if AMQFT_TMA_STAGE
  if (tid == 0) {
    mbar_init(bar, 1);
    if constexpr (P > 1) {
      mbar_init(full, 1);
      mbar_init(freeb, P);
    }
    fence_mbar_init();
  }
  row_sync();
  uint32_t xpar = 0;   // P > 1: phase of full / freeb
  if constexpr (P > 1) {
    // every CTA's barriers are initialised before any remote arrive; the
    // staging rows start free (one arrive per CTA on every freeb)
    cluster_arrive();
    cluster_wait();
    if (tid == 0) {
      for (int k = 0; k < P; ++k) mbar_arrive_remote(mapa(smem_u32(freeb), static_cast<uint32_t>(k)));
      if (cl_id < rows) cluster_prefetch<IO, P, N>(in + cl_id * 2 * N * P, Tb, q, bar);
    }
  }
  // bytes of kernel row kr (an odd RDFT batch ends with a single real row)
  auto row_bytes = [&](size_t kr) -> uint32_t {
    return (RDFT && 2 * kr + 1 >= rows_in) ? ROW_BYTES / 2 : ROW_BYTES;
  };
  if (P == 1 && tid == 0 && blockIdx.x * RSTEP + slot < rows)
    tma_load_1d(Sb, in + (blockIdx.x * RSTEP + slot) * 2 * N, row_bytes(blockIdx.x * RSTEP + slot), bar);
  uint32_t parity = 0;
#else
  (void)Sb;
  (void)bar;
  (void)ROW_BYTES;
#endif

  const size_t r_first = P > 1 ? cl_id : blockIdx.x * RSTEP;
  const size_t r_step = P > 1 ? cl_n : gridDim.x * RSTEP;
  for (size_t r0 = r_first; r0 < rows; r0 += r_step) {
    // every thread reaches every barrier; a slot past the last row idles
    const size_t row = r0 + slot;
    const bool act = row < rows;
    PHASE_MARK(0);
    if constexpr (P > 1) {
      // this CTA's input pieces are in T; every CTA has read its staging row
      mbar_wait(bar, parity);
      parity ^= 1;
      mbar_wait(freeb, xpar);
      if (tid == 0) mbar_expect_tx(full, static_cast<uint32_t>(2 * N * sizeof(IO)));
      cluster_exchange<R, IO, P, C::N, C::NT, MODE == 1>(reinterpret_cast<const IO*>(Tb), Sb, full, q, tid, ctw);
      mbar_wait(full, xpar);   // my staging row is complete
      xpar ^= 1;
    }
    // ---- load: SplitComplex (elab.cpp:152-155) + SplitReal (185-197)
    // from the TMA-staged row; then prefetch the CTA's next row.
#if AMQFT_TMA_STAGE
    if (P == 1 && act) {
      mbar_wait(bar, parity);
      parity ^= 1;
    }
    const IO2* x = reinterpret_cast<const IO2*>(Sb);
#else
    const IO2* x = reinterpret_cast<const IO2*>(in + row * 2 * N);
#endif
    // Cells m = tid + 256 it (it < H/256) and m = H (thread 0): the
    // physical offsets are linear in it (256 is a multiple of both layout
    // periods), so every store is an immediate offset from a per-thread
    // base.  INV (swap-trick inverse): re/im exchanged on the way in.
    if (act && tid < IO_T) {
      const int q0 = C::pt(tid, 0), q1 = C::pt(tid, 1);
      R* t0 = Tb + C::coT(0) + q0;
      R* t1 = Tb + C::coT(1) + q1;
      R* t2 = Tb + C::coT(2) + q0;
      R* t3 = Tb + C::coT(3) + q1;
      // all staged reads first (the compiler cannot hoist them over the
      // T stores itself: both are shared memory), then the stores
      // RDFT: rows A and B (N reals each) take the places of re and im
      const IO* xa = reinterpret_cast<const IO*>(x);
      const IO* xb = xa + N;
      V2 av[IO_IT], bv[IO_IT];
#pragma unroll
      for (int it = 0; it < IO_IT; ++it) {
        const int m = tid + it * IO_T;
        const int mm = (N - m) & (N - 1);   // m = 0: in range, unused
        if constexpr (RDFT) {
          av[it] = cvt_in(IO2{xa[m], xb[m]});
          bv[it] = cvt_in(IO2{xa[mm], xb[mm]});
        } else {
          av[it] = cvt_in(x[m]);
          bv[it] = cvt_in(x[mm]);
        }
      }
#pragma unroll
      for (int it = 0; it < IO_IT; ++it) {
        V2 a = av[it], b = bv[it];
        if (INV_IN) {
          a = V2{a.y, a.x};
          b = V2{b.y, b.x};
        }
        if (it == 0 && tid == 0) {   // m = 0: Dct chains only
          t0[0] = a.x;
          t2[0] = a.y;
          continue;
        }
        t0[it * PT_STEP] = A::add(a.x, b.x);
        t1[it * PT_STEP] = A::sub(a.x, b.x);
        t2[it * PT_STEP] = A::add(a.y, b.y);
        t3[it * PT_STEP] = A::sub(a.y, b.y);
      }
      if (tid == 0) {                // m = H
        V2 a = cvt_in(RDFT ? IO2{xa[H], xb[H]} : x[H]);
        if (INV_IN) a = V2{a.y, a.x};
        Tb[C::coT(0) + C::pt(H, 0)] = a.x;
        Tb[C::coT(2) + C::pt(H, 0)] = a.y;
      }
    }
    WORK_MARK(0);
    row_sync();
    if constexpr (P > 1) {   // staging row consumed: tell every CTA of the cluster
      if (tid == 0)
        for (int k = 0; k < P; ++k) mbar_arrive_remote(mapa(smem_u32(freeb), static_cast<uint32_t>(k)));
    }
#if AMQFT_TMA_STAGE
    if (P == 1 && tid == 0 && row + gridDim.x * RSTEP < rows) {
      fence_proxy_async();
      tma_load_1d(Sb, in + (row + gridDim.x * RSTEP) * 2 * N, row_bytes(row + gridDim.x * RSTEP), bar);
    }
#endif
    PHASE_MARK(1);

    if constexpr (C::TM) {
      // top mirror levels (generated, 2^LT cells per thread) || small chains
      if (act && tid < 4 * C::LB) {
        const int c = tid >> LOGLB, v = tid & (C::LB - 1);
        if constexpr (C::TOP_TMEM) {
          float kk[NKP];
          top_consts(kk);   // the whole warp (tcgen05.ld is warp-collective)
          if (v > 0) TopT::template fwd_k<R, A>(c & 1, Tb + C::coT(c), v, reinterpret_cast<const R*>(kk));
        } else if (v > 0) {
          TopT::template fwd<R, A>(c & 1, Tb + C::coT(c), v, ltab, base);
        }
      }
    } else {
      // chain folds n = N .. 2N/LB (generated sets, cooperative k = 0 class)
      recombine<C, R, true>(Tb, tid, act, row_sync);
      row_sync();
      // serial recurrences: fp64 in the reference order (bitwise), fp32 as warp scans
      if constexpr (C::SERIAL) am_levels_asc<C, R, C::LT>(Tb, tid);   // RPC = 1
      else if (act) am_phase_regs<C, R, false>(Tb, tid);
      // small-chain folds (cells [0, N/LB] of T, untouched by the AM
      // levels): lane 31 of chain c's second warp is idle in the AM phase
    }
    // the previous row's bulk store has long finished reading F (a load and
    // a top phase ago); make it formal before the bottom writes F
    if (BULK_ST && tid == 0) bulk_wait_read_all();
    WORK_MARK(1);
    row_sync();
    PHASE_MARK(2);

    // ---- bottom: T -> F (generated).  Segment code depends only on lam
    // (odd segments stored reversed, Cfg::ipos).  N >= 4096: one thread per
    // LB-segment runs all classes (loads hoisted).  N <= 2048 (few
    // segments): warp w of warps 0-3 runs class group (w/2: class 0 |
    // classes 1..) of the lam = w%2 segments, one per lane.
    constexpr bool SPLIT = C::NSEG <= 64;
    constexpr int BT = SPLIT ? 128 : C::NSEG;        // bottom threads
    if (!act) {
    } else if (tid < BT) {
      if constexpr (SPLIT) {
        const int w = tid >> 5, g = tid & 31;
        const int lam_bit = w & 1;
        if (g < 2 * C::HP) {
          const int c = lam_bit + 2 * (g / C::HP), sg = g % C::HP;
          int rho, lens, r;
          seg_params<C::SINE>(lam_bit, sg, C::LT, &rho, &lens, &r);
          if (w >> 1)
            Bottom<V, C::LB>::template run<R, A, LOGLB, C::LT, 1>(0, lens, Tb + C::coT(c), Fb + C::coF(c),
                                                                  sg * C::LB, tab, nmax, base, N, r, lam_bit);
          else
            Bottom<V, C::LB>::template run<R, A, LOGLB, C::LT, 0>(0, lens, Tb + C::coT(c), Fb + C::coF(c),
                                                                  sg * C::LB, tab, nmax, base, N, r, lam_bit);
        }
      } else {
        const int half = C::HP / 2;
        const int h = tid % half;
        const int rest = tid / half;
        const int part = rest & 1, rho_bit = (rest >> 1) & 1, lam_bit = (rest >> 2) & 1;
        const int c = part * 2 + lam_bit;
        const int sg = 2 * h + rho_bit;
        int rho, lens, r;
        seg_params<C::SINE>(lam_bit, sg, C::LT, &rho, &lens, &r);
        // all classes in one function, every T load hoisted above the F stores
        Bottom<V, C::LB>::template run<R, A, LOGLB, C::LT, 2>(0, lens, Tb + C::coT(c), Fb + C::coF(c),
                                                              sg * C::LB, tab, nmax, base, N, r, lam_bit);
      }
    } else {
      // the small chains (cells at multiples of LB; disjoint from the
      // segments' cells in T and F), one lane per chain, on the first lane
      // of four warps past the bottom threads where the block has them
      constexpr int SPARE = C::NT - BT;
      constexpr int STR = SPARE / 4 >= 32 ? 32 : SPARE / 4;
      const int l = tid - BT;
      // SPARE = 64: two warps, chains (0, 2) on the first and (1, 3) on the
      // second (one code path per warp); otherwise one lane per warp
      const int cc = SPARE == 64 ? ((l >> 5) | (((l & 31) >> 4) << 1)) : l / STR;
      if ((SPARE == 64 ? (l & 15) == 0 : l % STR == 0) && cc < 4) {
        SmallFull<V, C::HP, LOGN>::template run<R, A, LOGLB, C::LB>(cc & 1, Tb + C::coT(cc), Fb + C::coF(cc),
                                                                     tab, base);
      }
    }
    WORK_MARK(2);
    row_sync();
    PHASE_MARK(3);
    if constexpr (P > 1) {   // T is dead until the next load: prefetch the next row's pieces into it
      if (tid == 0 && row + r_step < rows) {
        fence_proxy_async();
        cluster_prefetch<IO, P, N>(in + (row + r_step) * 2 * N * P, Tb, q, bar);
      }
    }

    if constexpr (C::TM) {
      if constexpr (C::SERIAL) am_levels_desc<C, R, C::LT>(Fb, tid);  // RPC = 1
      else if (act) am_phase_regs<C, R, true>(Fb, tid);
      // small-chain recombination Dct/Dst(4..N/LB) on F cells [0, N/LB]
      // (disjoint from the AM levels): lane 31 of chain c's second warp
      WORK_MARK(3);
      row_sync();
      PHASE_MARK(4);
      // chain recombination n = 2N/LB .. N (generated sets, cooperative k = 0 class)
      recombine<C, R, false>(Fb, tid, act, row_sync);
      WORK_MARK(4);
      row_sync();
    } else {
      if (act && tid < 4 * C::LB) {
        const int c = tid >> LOGLB, v = tid & (C::LB - 1);
        if constexpr (C::TOP_TMEM) {
          float kk[NKP];
          top_consts(kk);
          if (v > 0) TopT::template bwd_k<R, A>(c & 1, Fb + C::coF(c), v, reinterpret_cast<const R*>(kk));
        } else if (v > 0) {
          TopT::template bwd<R, A>(c & 1, Fb + C::coF(c), v, ltab, base);
        }
      }
      WORK_MARK(4);
      row_sync();
    }
    PHASE_MARK(5);

    // ---- store: SplitReal bwd (elab.cpp:199-208) + SplitComplex bwd (162-183)
    // P > 1: X[k1 + P k2], k1 = q (stride P in the big row)
    IO2* y = reinterpret_cast<IO2*>(out + row * 2 * N * P) + q;
    constexpr int OS = P;
    if constexpr (BULK_ST) {
      // read all cells (registers), barrier, write the natural-order row
      // over F, barrier, one bulk store per row
      V2 lo[IO_IT], hi[IO_IT], yH;
      if (act && tid < IO_T) {
        const int q0 = C::pf(tid, 0), q1 = C::pf(tid, 1);
        const R* f0 = Fb + C::coF(0) + q0;
        const R* f1 = Fb + C::coF(1) + q1;
        const R* f2 = Fb + C::coF(2) + q0;
        const R* f3 = Fb + C::coF(3) + q1;
#pragma unroll
        for (int it = 0; it < IO_IT; ++it) {
          const R rd = f0[it * PF_STEP], id = f2[it * PF_STEP];
          const R rs = f1[it * PF_STEP], is = f3[it * PF_STEP];   // k = 0: unused
          if constexpr (RDFT) {      // SplitReal bwd: copies (Dct k, Dst N-k)
            lo[it] = V2{rd, id};
            hi[it] = V2{rs, is};
          } else {
            lo[it] = V2{A::add(rd, is), A::sub(id, rs)};
            hi[it] = V2{A::sub(rd, is), A::add(id, rs)};
          }
          if (it == 0 && tid == 0) lo[0] = V2{rd, id};            // k = 0: Dct chains only
          if (INV) {
            lo[it] = V2{A::mul(lo[it].y, scale), A::mul(lo[it].x, scale)};
            hi[it] = V2{A::mul(hi[it].y, scale), A::mul(hi[it].x, scale)};
          }
        }
        if (tid == 0) {              // k = H
          const R rd = Fb[C::coF(0) + C::pf(H, 0)], id = Fb[C::coF(2) + C::pf(H, 0)];
          yH = INV ? V2{A::mul(id, scale), A::mul(rd, scale)} : V2{rd, id};
        }
      }
      row_sync();
      if (act && tid < IO_T) {
        if constexpr (RDFT) {        // rows A | B, N reals each
          IO* oa = reinterpret_cast<IO*>(Fb);
          IO* ob = oa + N;
#pragma unroll
          for (int it = 0; it < IO_IT; ++it) {
            const int k = tid + it * IO_T;
            oa[k] = static_cast<IO>(lo[it].x);
            ob[k] = static_cast<IO>(lo[it].y);
            if (!(it == 0 && tid == 0)) {
              oa[N - k] = static_cast<IO>(hi[it].x);
              ob[N - k] = static_cast<IO>(hi[it].y);
            }
          }
          if (tid == 0) {
            oa[H] = static_cast<IO>(yH.x);
            ob[H] = static_cast<IO>(yH.y);
          }
        } else {
          IO2* ob = reinterpret_cast<IO2*>(Fb);
#pragma unroll
          for (int it = 0; it < IO_IT; ++it) {
            const int k = tid + it * IO_T;
            ob[k] = cvt_out(lo[it]);
            if (!(it == 0 && tid == 0)) ob[N - k] = cvt_out(hi[it]);
          }
          if (tid == 0) ob[H] = cvt_out(yH);
        }
        fence_proxy_async();         // generic-proxy writes -> async proxy
      }
      row_sync();
      if (act && tid == 0) bulk_store(y, Fb, row_bytes(row));
    } else {
      // Cells k = tid + 256 it and k = H (thread 0), immediate offsets as in
      // the load.  INV: re/im exchanged and scaled by 1/N on the way out.
      if constexpr (RDFT) {
        if (act && tid < IO_T) {
          const bool two = 2 * row + 1 < rows_in;
          IO* ya = out + row * 2 * N;
          IO* yb = ya + N;
          const int q0 = C::pf(tid, 0), q1 = C::pf(tid, 1);
          const R* f0 = Fb + C::coF(0) + q0;
          const R* f1 = Fb + C::coF(1) + q1;
          const R* f2 = Fb + C::coF(2) + q0;
          const R* f3 = Fb + C::coF(3) + q1;
#pragma unroll
          for (int it = 0; it < IO_IT; ++it) {
            const int k = tid + it * IO_T;
            ya[k] = static_cast<IO>(f0[it * PF_STEP]);
            if (two) yb[k] = static_cast<IO>(f2[it * PF_STEP]);
            if (it == 0 && tid == 0) continue;
            ya[N - k] = static_cast<IO>(f1[it * PF_STEP]);
            if (two) yb[N - k] = static_cast<IO>(f3[it * PF_STEP]);
          }
          if (tid == 0) {
            ya[H] = static_cast<IO>(Fb[C::coF(0) + C::pf(H, 0)]);
            if (two) yb[H] = static_cast<IO>(Fb[C::coF(2) + C::pf(H, 0)]);
          }
        }
      } else {
      if (act && tid < IO_T) {
          const int q0 = C::pf(tid, 0), q1 = C::pf(tid, 1);
          const R* f0 = Fb + C::coF(0) + q0;
          const R* f1 = Fb + C::coF(1) + q1;
          const R* f2 = Fb + C::coF(2) + q0;
          const R* f3 = Fb + C::coF(3) + q1;
  #pragma unroll
          for (int it = 0; it < IO_IT; ++it) {
            const int k = tid + it * IO_T;
            const R rd = f0[it * PF_STEP], id = f2[it * PF_STEP];
            if (it == 0 && tid == 0) {   // k = 0: Dct chains only
              y[0] = cvt_out(INV ? V2{A::mul(id, scale), A::mul(rd, scale)} : V2{rd, id});
              continue;
            }
            const R rs = f1[it * PF_STEP], is = f3[it * PF_STEP];
            V2 lo{A::add(rd, is), A::sub(id, rs)};
            V2 hi{A::sub(rd, is), A::add(id, rs)};
            if (INV) {
              lo = V2{A::mul(lo.y, scale), A::mul(lo.x, scale)};
              hi = V2{A::mul(hi.y, scale), A::mul(hi.x, scale)};
            }
            y[k * OS] = cvt_out(lo);
            y[(N - k) * OS] = cvt_out(hi);
          }
          if (tid == 0) {                // k = H
            const R rd = Fb[C::coF(0) + C::pf(H, 0)], id = Fb[C::coF(2) + C::pf(H, 0)];
            y[H * OS] = cvt_out(INV ? V2{A::mul(id, scale), A::mul(rd, scale)} : V2{rd, id});
          }
        }
      }
      }
    WORK_MARK(5);
    // No barrier here: the next row's load writes only T (and the staging
    // buffer through TMA), whose last readers are behind earlier barriers;
    // F is next written after two more barriers.
    PHASE_MARK(6);
  }
  if (BULK_ST && tid == 0) bulk_wait_all();   // smem must outlive the last bulk store
  if constexpr (C::TOP_TMEM) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (threadIdx.x < 32) tmem_dealloc(tbase);
  }
  if constexpr (P > 1) {   // no CTA leaves while a peer may still arrive on its barriers
    cluster_arrive();
    cluster_wait();
  }
}

// Per-level compacted constants for the top mirror levels:
// ltab[off_i + u] = tab[u * nmax / (2 L_i) - 1] (bitwise the TrigTable
// values), L_i = H >> (i-1), u in [1, L_i/2), so a warp's lanes (consecutive
// v) read consecutive words at every level.
template <typename R>
__global__ void k_level_table(const R* __restrict__ tab, R* __restrict__ ltab, int H, int LT,
                              int nmax) {
  int off = 0;
  for (int i = 1; i <= LT; ++i) {
    const int L = H >> (i - 1);
    for (int u = threadIdx.x + blockIdx.x * blockDim.x; u < L / 2; u += blockDim.x * gridDim.x)
      ltab[off + u] = u == 0 ? R(0) : tab[u * (nmax / (2 * L)) - 1];
    off += L / 2;
  }
}

// The generated small-chain code indexes the constant table with
// compile-time slots for Nmax = N.  A plan whose table was built for a
// larger Nmax (table_max_n, or a four-step sub-transform) uses this
// compacted copy: slot s of the Nmax = N table is slot (s+1) Nmax/N - 1 of
// the big one, bitwise the same value (TrigTable level sharing,
// variants.cpp:281).
template <typename R>
__global__ void k_compact_table(const R* __restrict__ tab, R* __restrict__ out, int n, int nmax) {
  const int ratio = nmax / n;
  for (int s = threadIdx.x + blockIdx.x * blockDim.x; s < n / 4; s += blockDim.x * gridDim.x)
    out[s] = tab[(s + 1) * ratio - 1];
}

template <int V, typename R, int LOGN, int LOGLB, bool RDFT_ROWS, typename IO = R>
class FastPlanImpl final : public FastPlan {
 public:
  FastPlanImpl(const void* tab, uint32_t nmax, int device) : tab_(static_cast<const R*>(tab)),
                                                              nmax_(nmax) {
    using C = Cfg<V, R, LOGN, LOGLB, IO>;
    // (fp32-I/O fp64-compute instances receive the plan's fp64 copy of the
    // table: tab is always of type R)
    if (nmax_ != static_cast<uint32_t>(C::N)) {
      cudaError_t e0 = cudaMalloc(&own_tab_, sizeof(R) * (C::N / 4));
      if (e0 != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e0));
      k_compact_table<R><<<8, 256>>>(tab_, own_tab_, C::N, static_cast<int>(nmax_));
      tab_ = own_tab_;
      nmax_ = C::N;
    }
    // CDFT plans: forward (MODE 0) and inverse (1); RDFT plans: MODE 2
    auto fn = k_fast<V, R, LOGN, LOGLB, RDFT_ROWS ? 2 : 0, IO>;
    auto fi = k_fast<V, R, LOGN, LOGLB, RDFT_ROWS ? 2 : 1, IO>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::SMEM_BLOCK));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fi, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM_BLOCK));
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::NTB, C::SMEM_BLOCK);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = std::max(1, per_sm) * sms;
    launches = 1;
    e = cudaMalloc(&ltab_, sizeof(R) * C::H);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    k_level_table<R><<<8, 256>>>(tab_, ltab_, C::H, C::LT, static_cast<int>(nmax_));
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    e = cudaMemcpy(tparam_.v, tab_, sizeof(tparam_.v), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }
  ~FastPlanImpl() override {
    if (ltab_) cudaFree(ltab_);
    if (own_tab_) cudaFree(own_tab_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    using C = Cfg<V, R, LOGN, LOGLB, IO>;
    const size_t krows = RDFT_ROWS ? (rows + 1) / 2 : rows;   // kernel rows
    const size_t units = (krows + C::RPC - 1) / C::RPC;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(units, static_cast<size_t>(grid_cap_)));
    if (RDFT_ROWS)
      k_fast<V, R, LOGN, LOGLB, 2, IO><<<grid, C::NTB, C::SMEM_BLOCK, st>>>(
          static_cast<const IO*>(in), static_cast<IO*>(out), rows, tparam_, ltab_, static_cast<int>(nmax_), R(1),
          nullptr);
    else if (inverse)
      k_fast<V, R, LOGN, LOGLB, 1, IO><<<grid, C::NTB, C::SMEM_BLOCK, st>>>(
          static_cast<const IO*>(in), static_cast<IO*>(out), rows, tparam_, ltab_, static_cast<int>(nmax_),
          R(1) / R(C::N), nullptr);
    else
      k_fast<V, R, LOGN, LOGLB, 0, IO><<<grid, C::NTB, C::SMEM_BLOCK, st>>>(
          static_cast<const IO*>(in), static_cast<IO*>(out), rows, tparam_, ltab_, static_cast<int>(nmax_),
          R(1) / R(C::N), nullptr);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }

 private:
  const R* tab_;
  TabParam<R, (1 << LOGN) / 4> tparam_{};
  R* own_tab_ = nullptr;
  R* ltab_ = nullptr;
  uint32_t nmax_;
  int grid_cap_ = 148;
};

// Cluster four-step plan: CDFT rows of length P * 4096 on clusters of P
// CTAs (k_fast<..., P>), one persistent cluster per group of SMs.
template <int V, typename R, typename IO, int P>
class ClusterPlanImpl final : public FastPlan {
  static constexpr int LOGN = 12, LOGLB = 6;
  using C = Cfg<V, R, LOGN, LOGLB, IO, P>;
  using V2 = typename std::conditional<sizeof(R) == 4, float2, double2>::type;

 public:
  ClusterPlanImpl(const void* tab, uint32_t nmax, int device) {
    const R* t = static_cast<const R*>(tab);
    if (nmax != static_cast<uint32_t>(C::N)) {
      check_(cudaMalloc(&own_tab_, sizeof(R) * (C::N / 4)));
      k_compact_table<R><<<8, 256>>>(t, own_tab_, C::N, static_cast<int>(nmax));
      t = own_tab_;
    }
    check_(cudaMalloc(&ltab_, sizeof(R) * C::H));
    k_level_table<R><<<8, 256>>>(t, ltab_, C::H, C::LT, C::N);
    check_(cudaDeviceSynchronize());
    check_(cudaMemcpy(tparam_.v, t, sizeof(tparam_.v), cudaMemcpyDeviceToHost));
    // w_(PN)^j, j < P N, long double rounded once to R
    const size_t NN = static_cast<size_t>(P) * C::N;
    std::vector<V2> tw(NN);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (size_t j = 0; j < NN; ++j) {
      const long double a = two_pi * static_cast<long double>(j) / static_cast<long double>(NN);
      tw[j] = V2{static_cast<R>(cosl(a)), static_cast<R>(-sinl(a))};
    }
    check_(cudaMalloc(&ctw_, NN * sizeof(V2)));
    check_(cudaMemcpy(ctw_, tw.data(), NN * sizeof(V2), cudaMemcpyHostToDevice));
    for (auto fn : {k_fast<V, R, LOGN, LOGLB, 0, IO, P>, k_fast<V, R, LOGN, LOGLB, 1, IO, P>}) {
      check_(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM_BLOCK)));
      if (P > 8) check_(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(P * 148);
    cfg.blockDim = dim3(C::NTB);
    cfg.dynamicSmemBytes = C::SMEM_BLOCK;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    check_(cudaOccupancyMaxActiveClusters(&nc, k_fast<V, R, LOGN, LOGLB, 0, IO, P>, &cfg));
    if (nc < 1) throw std::runtime_error("cluster four-step: no cluster of this size fits an SM group");
    max_clusters_ = nc;
    (void)device;
    launches = 1;
  }
  ~ClusterPlanImpl() override {
    if (ltab_) cudaFree(ltab_);
    if (own_tab_) cudaFree(own_tab_);
    if (ctw_) cudaFree(ctw_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    const unsigned nc = static_cast<unsigned>(std::min<size_t>(rows, static_cast<size_t>(max_clusters_)));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(P * nc);
    cfg.blockDim = dim3(C::NTB);
    cfg.dynamicSmemBytes = C::SMEM_BLOCK;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const R scale = R(1) / R(static_cast<double>(P) * C::N);
    cudaError_t e;
    if (inverse)
      e = cudaLaunchKernelEx(&cfg, k_fast<V, R, LOGN, LOGLB, 1, IO, P>, static_cast<const IO*>(in),
                             static_cast<IO*>(out), rows, tparam_, static_cast<const R*>(ltab_), C::N, scale,
                             static_cast<const void*>(ctw_));
    else
      e = cudaLaunchKernelEx(&cfg, k_fast<V, R, LOGN, LOGLB, 0, IO, P>, static_cast<const IO*>(in),
                             static_cast<IO*>(out), rows, tparam_, static_cast<const R*>(ltab_), C::N, scale,
                             static_cast<const void*>(ctw_));
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }

 private:
  static void check_(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }
  TabParam<R, (1 << LOGN) / 4> tparam_{};
  R* own_tab_ = nullptr;
  R* ltab_ = nullptr;
  V2* ctw_ = nullptr;
  int max_clusters_ = 1;
};

// Sizes run by the cluster four-step (fast.cu decides per size).
inline bool cluster_size_ok(size_t n) { return n >= 8192 && n <= 65536; }

template <int V, typename R, typename IO = R>
std::unique_ptr<FastPlan> make_cluster(size_t n, const void* tab, uint32_t nmax, int dev) {
  switch (n) {
    case 8192: return std::make_unique<ClusterPlanImpl<V, R, IO, 2>>(tab, nmax, dev);
    case 16384: return std::make_unique<ClusterPlanImpl<V, R, IO, 4>>(tab, nmax, dev);
    case 32768: return std::make_unique<ClusterPlanImpl<V, R, IO, 8>>(tab, nmax, dev);
    case 65536: return std::make_unique<ClusterPlanImpl<V, R, IO, 16>>(tab, nmax, dev);
  }
  return nullptr;
}

template <int V, typename R, bool RD, typename IO = R>
std::unique_ptr<FastPlan> make_sized(size_t n, const void* tab, uint32_t nmax, int dev) {
  switch (n) {
    case 1024: return std::make_unique<FastPlanImpl<V, R, 10, 6, RD, IO>>(tab, nmax, dev);
    case 2048: return std::make_unique<FastPlanImpl<V, R, 11, 6, RD, IO>>(tab, nmax, dev);
    case 4096: return std::make_unique<FastPlanImpl<V, R, 12, 6, RD, IO>>(tab, nmax, dev);
    case 8192:
      if constexpr (sizeof(R) == 4) return std::make_unique<FastPlanImpl<V, R, 13, 6, RD, IO>>(tab, nmax, dev);
      break;
  }
  return nullptr;
}

}  // namespace fastk
}  // namespace amqft_b200
