// generic.cuh -- sm_100a schedule-interpreter kernels (exact order).
//
// Device evaluation of the elaboration instances produced by plan.cpp.
// Every item computes ONE output cell with the reference's operation on the
// reference's operands in the reference's order (file:line per case below);
// arithmetic goes through __dadd_rn/__dsub_rn/__dmul_rn (or the fp32
// equivalents), which are never contracted into FMA, so fp64 results are
// bitwise those of amqft::execute.
#pragma once

#include <cstdint>

#include "generic_exec.hpp"
#include "plan.hpp"

namespace amqft_b200 {

template <typename R> struct Arith;
template <> struct Arith<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
};
template <> struct Arith<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
};

template <typename R>
__device__ __forceinline__ R trig_value(const TrigRef& t, uint32_t index, uint32_t n) {
  if (t.on_the_fly) {
    const double x = 2.0 * static_cast<double>(index) / static_cast<double>(n);
    double v;
    switch (t.kind) {
      case 0: v = 2.0 * cospi(x); break;
      case 1: v = 2.0 * sinpi(x); break;
      case 2: v = 1.0 / (2.0 * cospi(x)); break;
      default: v = 1.0 / (2.0 * sinpi(x)); break;
    }
    return static_cast<R>(v);
  }
  return static_cast<const R*>(t.table)[index * (t.nmax / n) - 1];
}

template <typename R>
__device__ __forceinline__ R trig_base(const TrigRef& t) {
  return static_cast<const R*>(t.table)[t.nmax / 4 - 1];
}

// One output cell of EI `e`: returns its value and position (relative to
// e.off) through *dst.  L(p) loads the source cell at relative position p.
// Chains (OP_CHAIN_*) are not items of this function.
template <typename R, typename Load>
__device__ __forceinline__ R eval_item(const EI& e, uint32_t i, uint32_t* dst,
                                       const TrigRef& trig, Load L) {
  using A = Arith<R>;
  const uint32_t n = e.n;
  *dst = i;
  switch (e.op) {
    case OP_SC_F:  // elaborations.cpp:152-155
      return i < n ? L(2 * i) : L(2 * (i - n) + 1);
    case OP_SC_B: {  // elaborations.cpp:166-181; A at [0,n), B at [n,2n)
      const uint32_t k = i >> 1, im = i & 1;
      if (k == 0 || k == n / 2) return im ? L(n + k) : L(k);
      if (k < n / 2) return im ? A::sub(L(n + k), L(n - k))      // im(k) = B[k] - A[n-k]
                               : A::add(L(k), L(2 * n - k));     // re(k) = A[k] + B[n-k]
      const uint32_t j = n - k;
      return im ? A::add(L(n + j), L(k))                         // im(n-j) = B[j] + A[n-j]
                : A::sub(L(j), L(n + k));                        // re(n-j) = A[j] - B[n-j]
    }
    case OP_SR_F: {  // elaborations.cpp:190-195
      if (i == 0 || i == n / 2) return L(i);
      if (i < n / 2) return A::add(L(i), L(n - i));
      const uint32_t m = i - n / 2;  // Dst cell m-1 holds s(m)
      return A::sub(L(m), L(n - m));
    }
    case OP_SR_B:  // elaborations.cpp:203-206
      return i <= n / 2 ? L(i) : L(3 * n / 2 - i);
    case OP_GATHER: {  // elaborations.cpp:288-295 (n = mother cells, aux = ce)
      const uint32_t ce = e.aux;
      return i < ce ? L(2 * i + e.lens) : L(2 * (i - ce) + 1 - e.lens);
    }
    case OP_SCATTER:  // elaborations.cpp:268-275
      return ((i & 1u) == e.lens) ? L(i >> 1) : L(e.aux + (i >> 1));
    case OP_SH_F_DCT: {  // elaborations.cpp:238-255, DctFull mother
      if (i <= n / 4) return i == n / 4 ? L(i) : A::add(L(i), L(n / 2 - i));
      const uint32_t j = i - (n / 4 + 1);
      return A::sub(L(j), L(n / 2 - j));
    }
    case OP_SH_F_DST: {  // DstFull mother: position = index - 1
      if (i < n / 4 - 1) return A::sub(L(i), L(n / 2 - i - 2));
      const uint32_t idx = i - (n / 4 - 1) + 1;
      return idx == n / 4 ? L(idx - 1) : A::add(L(idx - 1), L(n / 2 - idx - 1));
    }
    case OP_SH_F_ODD: {  // odd-time mother: pairs (p, mc-1-p)
      const uint32_t mc = n / 4;
      if (i < mc / 2) return e.lens ? A::sub(L(i), L(mc - 1 - i)) : A::add(L(i), L(mc - 1 - i));
      const uint32_t j = i - mc / 2;
      return e.lens ? A::add(L(j), L(mc - 1 - j)) : A::sub(L(j), L(mc - 1 - j));
    }
    case OP_ST_B_DCT: {  // elaborations.cpp:310-319; E at 0, O at n/4+1
      const uint32_t o = n / 4 + 1;
      if (i < n / 4) return A::add(L(i), L(o + i));
      if (i == n / 4) return L(i);
      const uint32_t j = n / 2 - i;
      return A::sub(L(j), L(o + j));
    }
    case OP_ST_B_DST: {  // elaborations.cpp:320-329; E at 0, O at n/4-1
      const uint32_t o = n / 4 - 1;
      const uint32_t k = i + 1;
      if (k < n / 4) return A::add(L(o + k - 1), L(k - 1));
      if (k == n / 4) return L(o + n / 4 - 1);
      const uint32_t j = n / 2 - k;
      return A::sub(L(o + j - 1), L(j - 1));
    }
    case OP_ST_B_ODD: {  // odd-harmonic mother; E at 0, O at mc/2
      const uint32_t mc = n / 4, o = mc / 2;
      if (i < o) return e.lens ? A::add(L(o + i), L(i)) : A::add(L(i), L(o + i));
      const uint32_t j = mc - 1 - i;
      return e.lens ? A::sub(L(o + j), L(j)) : A::sub(L(j), L(o + j));
    }
    case OP_AM_F: {  // elaborations.cpp:359-398
      const uint32_t q = e.aux;
      const uint32_t m = e.am;
      if (m == 1 || m == 4 || m == 5 || m == 8)
        return A::mul(L(i), trig_value<R>(trig, 2 * i + 1, n));
      if (m == 2) {
        if (e.lens == 0) return i == 0 ? L(0) : A::add(L(i), L(i - 1));
        return i == q - 1 ? L(q - 1) : A::add(L(i + 1), L(i));
      }
      /* m == 6 */
      if (e.lens == 0) return i == q - 1 ? L(q - 1) : A::sub(L(i), L(i + 1));
      return i == 0 ? L(0) : A::sub(L(i), L(i - 1));
    }
    case OP_AM_B: {  // elaborations.cpp:460-526
      const uint32_t q = e.aux;
      const uint32_t m = e.am;
      if (m == 2 || m == 3 || m == 6 || m == 7)
        return A::mul(L(i), trig_value<R>(trig, 2 * i + 1, n));
      if (m == 4) {
        if (e.lens == 0) return i < q - 1 ? A::add(L(i), L(i + 1)) : L(q - 1);
        return i == 0 ? L(0) : A::add(L(i - 1), L(i));
      }
      /* m == 8 */
      if (e.lens == 0) return i == 0 ? L(0) : A::sub(L(i), L(i - 1));
      return i < q - 1 ? A::sub(L(i), L(i + 1)) : L(q - 1);
    }
    case OP_BASE_CDFT2:  // variants.cpp:360-363; cells re0, im0, re1, im1
      return i < 2 ? A::add(L(i), L(i + 2)) : A::sub(L(i - 2), L(i));
    case OP_BASE_PAIR2:  // variants.cpp:366-371
      return i == 0 ? A::add(L(0), L(1)) : A::sub(L(0), L(1));
    case OP_BASE_OO8:  // variants.cpp:390
      return A::mul(L(0), trig_base<R>(trig));
  }
  return R(0);
}

// Serial recurrences (M3/M7 forward, elaborations.cpp:402-448; M1/M5
// backward, elaborations.cpp:472-513), run by one thread.  Reads source
// cells through L, writes outputs through S.
template <typename R, typename Load, typename Store>
__device__ void run_chain(const EI& e, Load L, Store S) {
  using A = Arith<R>;
  const int q = static_cast<int>(e.aux);
  const bool desc = e.flags & FL_DESC;
  const bool add = e.flags & FL_ADD;
  const int s = desc ? q - 1 : 0;
  const int d = desc ? -1 : 1;
  const R half = R(0.5);
  if (e.op == OP_CHAIN_F) {
    if (q == 1) {
      S(0, A::mul(half, L(0)));
      return;
    }
    R prev = L(s);
    S(s, prev);
    int p = s;
    for (int k = 1; k < q - 1; ++k) {
      p += d;
      prev = add ? A::add(L(p), prev) : A::sub(L(p), prev);
      S(p, prev);
    }
    p += d;
    const R t = add ? A::add(L(p), prev) : A::sub(L(p), prev);
    S(p, A::mul(half, t));
    return;
  }
  R prev = A::mul(half, L(s));
  S(s, prev);
  int p = s;
  for (int k = 1; k < q; ++k) {
    p += d;
    prev = add ? A::add(L(p), prev) : A::sub(L(p), prev);
    S(p, prev);
  }
}

// Locate the EI of item g inside stage [b, e) by its exclusive prefix.
__device__ __forceinline__ uint32_t find_ei(const uint32_t* __restrict__ prefix,
                                            uint32_t b, uint32_t e, uint32_t g) {
  uint32_t lo = b, hi = e - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(prefix + mid) <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace amqft_b200
