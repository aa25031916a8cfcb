// small_kernel.cuh -- small CDFTs, one row per thread (path 4).
//
// k_small: for N <= 64 (fp32) / N <= 32 (fp64) a thread owns one row: the traced
// stage program of the plan compiler, emitted as straight-line code by
// codegen/gen_small.py (small_gen.cuh), keeps the row in registers.  Every
// line is one reference add/sub/mul on the reference operands (no FMA
// contraction, Arith<R>), so the fp64 instance is bitwise amqft::execute for
// all 8 variants, in both execution orders.
//
// Data movement (HBM-bound; ~0.3-1.2 flop/B):
//  * rows of <= 64 B: straight from global memory, 16-byte vector loads and
//    stores per thread (a warp touches 32 consecutive rows, every fetched
//    sector is used);
//  * larger rows: a CTA tile of T rows is staged in shared memory by one
//    cp.async.bulk per row into slots padded by 16 bytes (so the 8 lanes of
//    a quarter-warp reading the same 16-byte chunk of 8 rows hit 8 distinct
//    bank groups), transformed in place, and written back by one bulk store
//    per row.
// k_coop (below): N = 128..512 (fp32) / 64..256 (fp64), a row per lane and
// one warp per subtree role.
// The inverse is the swap trick (x = swap(DFT(swap(X))) / N), fused into the
// chunk loads and stores.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "fast.cuh"
#include "generic.cuh"

#ifndef AMQFT_COL_STAGED
// TMA-staged column tiles (k_small_colt) where cols % 128 == 0.  Measured
// (B200, table twiddles): no better than the direct column kernel (fp32
// 2^15 / 2^16 / 2^17: 1.21 / 1.18 / 1.46 vs 1.10 / 1.35 / 1.54 TB/s), so off.
#define AMQFT_COL_STAGED 0
#endif

namespace amqft_b200 {
namespace smallk {

// generated per variant (codegen/gen_small.py -> gen/small_gen_v<V>.cuh,
// included by small_v<V>.cu before this header)
template <int V, int F, int LOGN, typename R> struct SmallGen;
template <int V, int LOGN, typename R> struct SmallRoles;

template <typename R, int K>
struct TabP {
  R v[K];
};

template <typename R> struct Vec;
template <> struct Vec<float> { using T = float4; static constexpr int W = 4; };
template <> struct Vec<double> { using T = double2; static constexpr int W = 2; };

// Chunk I/O of one row (p: the row in global or shared memory).
template <typename R, bool INV> struct RowIO;
template <bool INV> struct RowIO<float, INV> {
  float4* p;
  float scale;
  __device__ __forceinline__ void ld(int c, float& a, float& b, float& d, float& e) const {
    const float4 v = p[c];
    if (INV) { a = v.y; b = v.x; d = v.w; e = v.z; }
    else { a = v.x; b = v.y; d = v.z; e = v.w; }
  }
  __device__ __forceinline__ void st(int c, float a, float b, float d, float e) const {
    using A = Arith<float>;
    if (INV) p[c] = make_float4(A::mul(b, scale), A::mul(a, scale), A::mul(e, scale), A::mul(d, scale));
    else p[c] = make_float4(a, b, d, e);
  }
};
template <bool INV> struct RowIO<double, INV> {
  double2* p;
  double scale;
  __device__ __forceinline__ void ld(int c, double& a, double& b) const {
    const double2 v = p[c];
    if (INV) { a = v.y; b = v.x; }
    else { a = v.x; b = v.y; }
  }
  __device__ __forceinline__ void st(int c, double a, double b) const {
    using A = Arith<double>;
    if (INV) p[c] = make_double2(A::mul(b, scale), A::mul(a, scale));
    else p[c] = make_double2(a, b);
  }
};

// Global-memory variant: the input comes from `in`, the output goes to `out`.
template <typename R, bool INV> struct GRowIO;
template <bool INV> struct GRowIO<float, INV> {
  const float4* pi;   // may alias po (in-place rows): no __restrict__
  float4* po;
  float scale;
  __device__ __forceinline__ void ld(int c, float& a, float& b, float& d, float& e) const {
    const float4 v = pi[c];
    if (INV) { a = v.y; b = v.x; d = v.w; e = v.z; }
    else { a = v.x; b = v.y; d = v.z; e = v.w; }
  }
  __device__ __forceinline__ void st(int c, float a, float b, float d, float e) const {
    using A = Arith<float>;
    if (INV) __stcs(po + c, make_float4(A::mul(b, scale), A::mul(a, scale), A::mul(e, scale), A::mul(d, scale)));
    else __stcs(po + c, make_float4(a, b, d, e));
  }
};
template <bool INV> struct GRowIO<double, INV> {
  const double2* pi;
  double2* po;
  double scale;
  __device__ __forceinline__ void ld(int c, double& a, double& b) const {
    const double2 v = pi[c];
    if (INV) { a = v.y; b = v.x; }
    else { a = v.x; b = v.y; }
  }
  __device__ __forceinline__ void st(int c, double a, double b) const {
    using A = Arith<double>;
    if (INV) __stcs(po + c, make_double2(A::mul(b, scale), A::mul(a, scale)));
    else __stcs(po + c, make_double2(a, b));
  }
};

// Slots s < nt of the Nmax = 4 nt table are slots (s + 1) nmax / (4 nt) - 1
// of the plan's table (TrigTable level sharing, variants.cpp:281): one
// strided copy.
template <typename R>
cudaError_t fetch_table(R* dst, int nt, const void* tab, uint32_t nmax) {
  const size_t ratio = nmax / (4u * static_cast<uint32_t>(nt));
  return cudaMemcpy2D(dst, sizeof(R), static_cast<const R*>(tab) + (ratio - 1), ratio * sizeof(R), sizeof(R),
                      static_cast<size_t>(nt), cudaMemcpyDeviceToHost);
}

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// F: 0 CDFT rows (2N interleaved reals), 1 RDFT rows (N reals, packed
// spectrum, signal.hpp:122-124)
template <typename R, int LOGN, int F = 0>
struct SCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int CELLS = F == 0 ? 2 * N : N;
  static constexpr int NT = (N < 8 ? 8 : N) / 4;      // constant table (Nmax = max(N, 8))
  static constexpr int ROWB = CELLS * static_cast<int>(sizeof(R));
  static constexpr bool DIRECT = ROWB <= 64;   // measured: 128-B rows are faster staged
  static constexpr int STRIDE = ROWB + 16;             // padded slot (bytes)
  static constexpr int T = 128;                        // rows (threads) per CTA
  static constexpr size_t SMEM = DIRECT ? 0 : static_cast<size_t>(T) * STRIDE + 16;
};

template <int V, typename R, int LOGN, bool INV, int F = 0>
__global__ void __launch_bounds__(128)
k_small(const R* __restrict__ in, R* __restrict__ out, size_t rows,
        const __grid_constant__ TabP<R, SCfg<R, LOGN, F>::NT> tp, R scale) {
  using C = SCfg<R, LOGN, F>;
  using G = SmallGen<V, F, LOGN, R>;
  using VT = typename Vec<R>::T;
  constexpr int CELLS = C::CELLS;
  const int tid = threadIdx.x;
  if constexpr (C::DIRECT) {
    for (size_t row = blockIdx.x * size_t(C::T) + tid; row < rows; row += size_t(gridDim.x) * C::T) {
      GRowIO<R, INV> io{reinterpret_cast<const VT*>(in + row * CELLS), reinterpret_cast<VT*>(out + row * CELLS),
                        scale};
      G::template run<Arith<R>>(io, tp.v);
    }
  } else {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(C::T) * C::STRIDE);
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(1) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;
    const size_t tiles = (rows + C::T - 1) / C::T;
    for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const size_t row0 = tile * C::T;
      const int nr = static_cast<int>(rows - row0 < size_t(C::T) ? rows - row0 : size_t(C::T));
      if (warp == 0) {
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                       ::"r"(s_u32(bar)), "r"(static_cast<uint32_t>(nr * C::ROWB)) : "memory");
        __syncwarp();
        for (int r = lane; r < nr; r += 32)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(s_u32(sm + size_t(r) * C::STRIDE)), "l"(in + (row0 + r) * CELLS), "r"(C::ROWB),
                "r"(s_u32(bar)) : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n}" ::"r"(s_u32(bar)), "r"(parity) : "memory");
      parity ^= 1;
      if (tid < nr) {
        RowIO<R, INV> io{reinterpret_cast<VT*>(sm + size_t(tid) * C::STRIDE), scale};
        G::template run<Arith<R>>(io, tp.v);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (warp == 0) {
        for (int r = lane; r < nr; r += 32)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(out + (row0 + r) * CELLS), "r"(s_u32(sm + size_t(r) * C::STRIDE)), "r"(C::ROWB)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
    }
    if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// ---- Cooperative rows (fp32 N = 128..512, fp64 N = 64..256): a 32-row
// tile per CTA, lane = row, one warp per generated role
// (SmallRoles<V, LOGN, R>::run).  Band B: a role loads the input chunks of
// its subtrees, barrier, runs them, stores the values the tail reads at
// their arena positions; band C: loads those chunks, barrier, computes and
// stores whole output chunks.  The barriers are named (bar.sync 1) and
// reached from every role's own code path.
// Band-B roles come in Re/Im pairs (generated code shared, part = 0 / 1):
// ldp returns the chunk's Re cells (part 1: its Im cells; the swap-trick
// inverse exchanges them), str/st1 store at the cut position shifted by
// part * HALF cells (the Im half of the arena).
template <typename R, bool INV, int NTH, int HALF> struct CoopIO;
template <bool INV, int NTH, int HALF> struct CoopIO<float, INV, NTH, HALF> : RowIO<float, INV> {
  __device__ __forceinline__ void ldp(int c, int part, float& a, float& b) const {
    const float4 v = this->p[c];
    const bool im = (part != 0) != INV;
    a = im ? v.y : v.x;
    b = im ? v.w : v.z;
  }
  __device__ __forceinline__ void ldr(int c, float& a, float& b, float& d, float& e) const {
    const float4 v = this->p[c];
    a = v.x; b = v.y; d = v.z; e = v.w;
  }
  __device__ __forceinline__ void str(int c, int part, float a, float b, float d, float e) const {
    this->p[c + part * (HALF / 4)] = make_float4(a, b, d, e);
  }
  __device__ __forceinline__ void st1(int q, int part, float a) const {
    reinterpret_cast<float*>(this->p)[q + part * HALF] = a;
  }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync 1, %0;" ::"n"(NTH) : "memory"); }
};
template <bool INV, int NTH, int HALF> struct CoopIO<double, INV, NTH, HALF> : RowIO<double, INV> {
  __device__ __forceinline__ void ldp(int c, int part, double& a) const {
    const double2 v = this->p[c];
    a = ((part != 0) != INV) ? v.y : v.x;
  }
  __device__ __forceinline__ void ldr(int c, double& a, double& b) const {
    const double2 v = this->p[c];
    a = v.x; b = v.y;
  }
  __device__ __forceinline__ void str(int c, int part, double a, double b) const {
    this->p[c + part * (HALF / 2)] = make_double2(a, b);
  }
  __device__ __forceinline__ void st1(int q, int part, double a) const {
    reinterpret_cast<double*>(this->p)[q + part * HALF] = a;
  }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync 1, %0;" ::"n"(NTH) : "memory"); }
};

template <int V, typename R, int LOGN>
struct CCfg {
  using G = SmallRoles<V, LOGN, R>;
  static constexpr int N = 1 << LOGN;
  static constexpr int NT = N / 4;
  static constexpr int ROWS = G::ROWS;          // 32, or 16 (lanes 16-31 duplicate rows 0-15)
  static constexpr int NTH = 32 * G::R;
  static constexpr int ROWB = 2 * N * static_cast<int>(sizeof(R));
  static constexpr int STRIDE = ROWB + 16;
  static constexpr size_t SMEM = static_cast<size_t>(ROWS) * STRIDE + 16;
};

template <int V, typename R, int LOGN, bool INV>
__global__ void __launch_bounds__(CCfg<V, R, LOGN>::NTH)
k_coop(const R* __restrict__ in, R* __restrict__ out, size_t rows,
       const __grid_constant__ TabP<R, CCfg<V, R, LOGN>::NT> tp, R scale) {
  using C = CCfg<V, R, LOGN>;
  using VT = typename Vec<R>::T;
  constexpr int N = C::N;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(C::ROWS) * C::STRIDE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;
  const size_t tiles = (rows + C::ROWS - 1) / C::ROWS;
  for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const size_t row0 = tile * C::ROWS;
    const int nr = static_cast<int>(rows - row0 < size_t(C::ROWS) ? rows - row0 : size_t(C::ROWS));
    if (warp == 0) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(s_u32(bar)), "r"(static_cast<uint32_t>(nr * C::ROWB)) : "memory");
      __syncwarp();
      if (lane < nr)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(s_u32(sm + size_t(lane) * C::STRIDE)), "l"(in + (row0 + lane) * 2 * N), "r"(C::ROWB),
              "r"(s_u32(bar)) : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(s_u32(bar)), "r"(parity) : "memory");
    parity ^= 1;
    // every lane runs (lanes past the tile's rows on stale data, not
    // stored): the roles' named barriers count all NTH threads
    CoopIO<R, INV, C::NTH, C::G::HALF> io;
    io.p = reinterpret_cast<VT*>(sm + size_t(lane % C::ROWS) * C::STRIDE);
    io.scale = scale;
    C::G::template run<Arith<R>>(warp, io, tp.v);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      if (lane < nr)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(out + (row0 + lane) * 2 * N), "r"(s_u32(sm + size_t(lane) * C::STRIDE)), "r"(C::ROWB)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int V, typename R, int LOGN>
class CoopPlanImpl final : public FastPlan {
  using C = CCfg<V, R, LOGN>;

 public:
  CoopPlanImpl(const void* tab, uint32_t nmax, int device) {
    cudaError_t e = fetch_table(tp_.v, C::NT, tab, nmax);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    auto f0 = k_coop<V, R, LOGN, false>;
    auto f1 = k_coop<V, R, LOGN, true>;
    e = cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, C::NTH, C::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    if (per_sm < 1) throw std::runtime_error("cooperative small kernel does not fit an SM");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = per_sm * sms;
    launches = 1;
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    const size_t tiles = (rows + C::ROWS - 1) / C::ROWS;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(tiles, static_cast<size_t>(grid_cap_)));
    const R scale = R(1) / R(C::N);
    if (inverse)
      k_coop<V, R, LOGN, true><<<grid, C::NTH, C::SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out),
                                                              rows, tp_, scale);
    else
      k_coop<V, R, LOGN, false><<<grid, C::NTH, C::SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out),
                                                               rows, tp_, scale);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }

 private:
  TabP<R, C::NT> tp_{};
  int grid_cap_ = 148;
};

// ---- Column mode (four-step first pass): thread = (matrix, column n2);
// element n1 of the column at in[(n1 cols + n2)], consecutive threads on
// consecutive columns (every load and store instruction of a warp touches
// 256 contiguous bytes).  Output k1 goes to out[(k1 cols + n2)] times
// w_N^(n2 k1) (fp64 twiddle, as the four-step transposes).
template <typename R>
__device__ __forceinline__ void col_twiddle(R& x, R& y, unsigned long long j, const ColTwiddle& t) {
  j &= (1ull << t.logn) - 1ull;
  R fr, fi;
  if constexpr (sizeof(R) == 4) {
    if (t.onthefly) {   // fp32 plans: sincospif of the exact integer phase (no table reads)
      float sn, cs;
      sincospif(static_cast<float>(static_cast<double>(j) * (2.0 / static_cast<double>(1ull << t.logn))), &sn, &cs);
      fr = cs;
      fi = -sn;
    } else {
      const double2 a = t.hi[j >> t.logb], b = t.lo[j & ((1ull << t.logb) - 1ull)];
      fr = static_cast<R>(a.x * b.x - a.y * b.y);
      fi = static_cast<R>(a.x * b.y + a.y * b.x);
    }
  } else {
    double wr, wi;
    if (t.onthefly) {
      double sn, cs;
      sincospi(static_cast<double>(j) * 2.0 / static_cast<double>(1ull << t.logn), &sn, &cs);
      wr = cs;
      wi = -sn;
    } else {
      const double2 a = t.hi[j >> t.logb], b = t.lo[j & ((1ull << t.logb) - 1ull)];
      wr = a.x * b.x - a.y * b.y;
      wi = a.x * b.y + a.y * b.x;
    }
    fr = static_cast<R>(wr);
    fi = static_cast<R>(wi);
  }
  const R nx = x * fr - y * fi, ny = x * fi + y * fr;
  x = nx;
  y = ny;
}

// fp64 value of w_N^j from the plan's twiddle set (tables, or sincospi).
__device__ __forceinline__ void twiddle_d(unsigned long long j, const ColTwiddle& t, double& wr, double& wi) {
  j &= (1ull << t.logn) - 1ull;
  if (t.onthefly) {
    double sn, cs;
    sincospi(static_cast<double>(j) * 2.0 / static_cast<double>(1ull << t.logn), &sn, &cs);
    wr = cs;
    wi = -sn;
  } else {
    const double2 a = t.hi[j >> t.logb], b = t.lo[j & ((1ull << t.logb) - 1ull)];
    wr = a.x * b.x - a.y * b.y;
    wi = a.x * b.y + a.y * b.x;
  }
}

// Twiddles of one column, w^(col k) for the outputs k in store order: the
// generated code stores output chunks in ascending k (the last stage,
// SplitComplex bwd, produces them in order), so each is the previous one
// times w^col in fp64 (~1e-14 after 64 steps); any other order falls back
// to the direct value.  Replaces a table pair (or a sincospif) per element.
struct TwRec {
  double cr = 1.0, ci = 0.0, sr = 1.0, si = 0.0;
  unsigned long long base = 0;
  int next = 0;
  ColTwiddle tw;
  __device__ __forceinline__ void init(unsigned long long col_mul, const ColTwiddle& t) {
    tw = t;
    base = col_mul;
    twiddle_d(col_mul, t, sr, si);
  }
  template <typename R>
  __device__ __forceinline__ void apply(int k, R& x, R& y) {
    if (k != next) twiddle_d(base * static_cast<unsigned long long>(k), tw, cr, ci);
    const R fr = static_cast<R>(cr), fi = static_cast<R>(ci);
    const R nx = x * fr - y * fi, ny = x * fi + y * fr;
    x = nx;
    y = ny;
    const double tr = cr * sr - ci * si, ti = cr * si + ci * sr;
    cr = tr;
    ci = ti;
    next = k + 1;
  }
};

template <typename R, bool INV> struct ColIO;
template <bool INV> struct ColIO<float, INV> {   // chunk c = complex 2c, 2c+1
  const float2* __restrict__ pi;
  float2* __restrict__ po;
  size_t stride;
  TwRec tr;
  __device__ __forceinline__ void ld(int c, float& a, float& b, float& d, float& e) const {
    const float2 u = __ldg(pi + size_t(2 * c) * stride), v = __ldg(pi + size_t(2 * c + 1) * stride);
    if (INV) { a = u.y; b = u.x; d = v.y; e = v.x; }
    else { a = u.x; b = u.y; d = v.x; e = v.y; }
  }
  __device__ __forceinline__ void st(int c, float a, float b, float d, float e) {
    tr.apply(2 * c, a, b);
    tr.apply(2 * c + 1, d, e);
    po[size_t(2 * c) * stride] = make_float2(a, b);
    po[size_t(2 * c + 1) * stride] = make_float2(d, e);
  }
};
template <bool INV> struct ColIO<double, INV> {  // chunk c = complex c
  const double2* pi;
  double2* po;
  size_t stride;
  TwRec tr;
  __device__ __forceinline__ void ld(int c, double& a, double& b) const {
    const double2 u = __ldg(pi + size_t(c) * stride);
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void st(int c, double a, double b) {
    tr.apply(c, a, b);
    po[size_t(c) * stride] = make_double2(a, b);
  }
};

template <int V, typename R, int LOGN, bool INV>
__global__ void __launch_bounds__(128)
k_small_col(const R* __restrict__ in, R* __restrict__ out, size_t mats, size_t cols,
            const __grid_constant__ TabP<R, SCfg<R, LOGN, 0>::NT> tp, const ColTwiddle tw) {
  using C2T = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  using G = SmallGen<V, 0, LOGN, R>;
  constexpr size_t N = size_t(1) << LOGN;
  const size_t total = mats * cols;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total; t += size_t(gridDim.x) * blockDim.x) {
    const size_t mat = t / cols, col = t - mat * cols;
    const size_t base = mat * N * cols + col;
    ColIO<R, INV> io{reinterpret_cast<const C2T*>(in) + base, reinterpret_cast<C2T*>(out) + base, cols, TwRec{}};
    io.tr.init(static_cast<unsigned long long>(col) * tw.mul, tw);
    G::template run<Arith<R>>(io, tp.v);
  }
}

// Staged variant (cols a multiple of 128): a tile of 128 consecutive
// columns arrives by N bulk copies of one contiguous 128-element run each
// into smem [n1][128]; thread t transforms column t out of shared memory
// (lanes on consecutive 8/16-byte elements: conflict-free) and the tile
// leaves by N bulk stores.  The TMA keeps every row of the tile in flight
// at once, which the direct loads above do not.
template <typename R, bool INV> struct ColSIO;
template <bool INV> struct ColSIO<float, INV> {
  float2* s;
  int t;
  unsigned long long col;
  ColTwiddle tw;
  __device__ __forceinline__ void ld(int c, float& a, float& b, float& d, float& e) const {
    const float2 u = s[(2 * c) * 128 + t], v = s[(2 * c + 1) * 128 + t];
    if (INV) { a = u.y; b = u.x; d = v.y; e = v.x; }
    else { a = u.x; b = u.y; d = v.x; e = v.y; }
  }
  __device__ __forceinline__ void st(int c, float a, float b, float d, float e) const {
    col_twiddle(a, b, col * tw.mul * static_cast<unsigned long long>(2 * c), tw);
    col_twiddle(d, e, col * tw.mul * static_cast<unsigned long long>(2 * c + 1), tw);
    s[(2 * c) * 128 + t] = make_float2(a, b);
    s[(2 * c + 1) * 128 + t] = make_float2(d, e);
  }
};
template <bool INV> struct ColSIO<double, INV> {
  double2* s;
  int t;
  unsigned long long col;
  ColTwiddle tw;
  __device__ __forceinline__ void ld(int c, double& a, double& b) const {
    const double2 u = s[c * 128 + t];
    if (INV) { a = u.y; b = u.x; }
    else { a = u.x; b = u.y; }
  }
  __device__ __forceinline__ void st(int c, double a, double b) const {
    col_twiddle(a, b, col * tw.mul * static_cast<unsigned long long>(c), tw);
    s[c * 128 + t] = make_double2(a, b);
  }
};

template <int V, typename R, int LOGN, bool INV>
__global__ void __launch_bounds__(128)
k_small_colt(const R* __restrict__ in, R* __restrict__ out, size_t mats, size_t cols,
             const __grid_constant__ TabP<R, SCfg<R, LOGN, 0>::NT> tp, const ColTwiddle tw) {
  using C2T = typename std::conditional<sizeof(R) == 4, float2, double2>::type;
  using G = SmallGen<V, 0, LOGN, R>;
  constexpr int N = 1 << LOGN;
  constexpr uint32_t SEG = 128 * sizeof(C2T);
  extern __shared__ __align__(128) unsigned char sm[];
  C2T* tile_s = reinterpret_cast<C2T*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(N) * SEG);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;
  const size_t cb = cols / 128, tiles = mats * cb;
  for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const size_t mat = tile / cb, col0 = (tile - mat * cb) * 128;
    const C2T* src = reinterpret_cast<const C2T*>(in) + mat * size_t(N) * cols + col0;
    C2T* dst = reinterpret_cast<C2T*>(out) + mat * size_t(N) * cols + col0;
    if (warp == 0) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(s_u32(bar)), "r"(static_cast<uint32_t>(N) * SEG) : "memory");
      __syncwarp();
      for (int k = lane; k < N; k += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(s_u32(tile_s + size_t(k) * 128)), "l"(src + size_t(k) * cols), "r"(SEG), "r"(s_u32(bar))
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(s_u32(bar)), "r"(parity) : "memory");
    parity ^= 1;
    ColSIO<R, INV> io{tile_s, tid, static_cast<unsigned long long>(col0 + tid), tw};
    G::template run<Arith<R>>(io, tp.v);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      for (int k = lane; k < N; k += 32)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst + size_t(k) * cols), "r"(s_u32(tile_s + size_t(k) * 128)), "r"(SEG) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int V, typename R, int LOGN, int F = 0>
class SmallPlanImpl final : public FastPlan {
  using C = SCfg<R, LOGN, F>;

 public:
  SmallPlanImpl(const void* tab, uint32_t nmax, int device) {
    // the generated slots index the Nmax = max(N, 8) table; a larger table
    // holds the same values at slot (s + 1) nmax / Nsmall - 1 (TrigTable
    // level sharing, variants.cpp:281)
    cudaError_t e = fetch_table(tp_.v, C::NT, tab, nmax);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    auto f0 = k_small<V, R, LOGN, false, F>;
    auto f1 = k_small<V, R, LOGN, true, F>;
    if (C::SMEM > 48 * 1024) {
      e = cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
      if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, C::T, C::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = std::max(1, per_sm) * sms;
    launches = 1;
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    const size_t tiles = (rows + C::T - 1) / C::T;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(tiles, static_cast<size_t>(grid_cap_)));
    const R scale = R(1) / R(C::N);
    if (inverse)
      k_small<V, R, LOGN, true, F><<<grid, C::T, C::SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                             tp_, scale);
    else
      k_small<V, R, LOGN, false, F><<<grid, C::T, C::SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                              tp_, scale);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }
  bool exec_columns(const void* in, void* out, size_t mats, size_t cols, int inverse, const ColTwiddle& tw,
                    cudaStream_t st) override {
    if constexpr (F != 0) {   // CDFT rows only
      (void)in, (void)out, (void)mats, (void)cols, (void)inverse, (void)tw, (void)st;
      return false;
    } else {
#if AMQFT_COL_STAGED
    if (cols % 128 == 0 && C::N >= 4) {
      constexpr size_t SMEM = size_t(C::N) * 128 * 2 * sizeof(R) + 16;
      auto f0 = k_small_colt<V, R, LOGN, false>;
      auto f1 = k_small_colt<V, R, LOGN, true>;
      if (!colt_ready_) {
        cudaError_t e0 = cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM));
        if (e0 == cudaSuccess)
          e0 = cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM));
        int per_sm = 0;
        if (e0 == cudaSuccess) e0 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, 128, SMEM);
        if (e0 != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e0));
        colt_grid_ = std::max(1, per_sm) * 148;
        colt_ready_ = true;
      }
      const size_t tiles = mats * (cols / 128);
      const unsigned g = static_cast<unsigned>(std::min<size_t>(tiles, static_cast<size_t>(colt_grid_)));
      if (inverse)
        f1<<<g, 128, SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out), mats, cols, tp_, tw);
      else
        f0<<<g, 128, SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out), mats, cols, tp_, tw);
      const cudaError_t e1 = cudaGetLastError();
      if (e1 != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e1));
      return true;
    }
#endif
    const size_t total = mats * cols;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((total + 127) / 128, size_t(148) * 16));
    if (inverse)
      k_small_col<V, R, LOGN, true><<<grid, 128, 0, st>>>(static_cast<const R*>(in), static_cast<R*>(out), mats,
                                                           cols, tp_, tw);
    else
      k_small_col<V, R, LOGN, false><<<grid, 128, 0, st>>>(static_cast<const R*>(in), static_cast<R*>(out), mats,
                                                            cols, tp_, tw);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    return true;
    }
  }

 private:
  bool colt_ready_ = false;
  int colt_grid_ = 148;
  TabP<R, C::NT> tp_{};
  int grid_cap_ = 148;
};

template <int V, typename R>
std::unique_ptr<FastPlan> make_small_sized(size_t n, const void* tab, uint32_t nmax, int dev) {
  switch (n) {
    case 2: return std::make_unique<SmallPlanImpl<V, R, 1>>(tab, nmax, dev);
    case 4: return std::make_unique<SmallPlanImpl<V, R, 2>>(tab, nmax, dev);
    case 8: return std::make_unique<SmallPlanImpl<V, R, 3>>(tab, nmax, dev);
    case 16: return std::make_unique<SmallPlanImpl<V, R, 4>>(tab, nmax, dev);
    case 32: return std::make_unique<SmallPlanImpl<V, R, 5>>(tab, nmax, dev);
    case 64:
      if constexpr (sizeof(R) == 4) return std::make_unique<SmallPlanImpl<V, R, 6>>(tab, nmax, dev);
      else return std::make_unique<CoopPlanImpl<V, R, 6>>(tab, nmax, dev);
    case 128: return std::make_unique<CoopPlanImpl<V, R, 7>>(tab, nmax, dev);
    case 256: return std::make_unique<CoopPlanImpl<V, R, 8>>(tab, nmax, dev);
    case 512:
      if constexpr (sizeof(R) == 4) return std::make_unique<CoopPlanImpl<V, R, 9>>(tab, nmax, dev);
      break;
  }
  return nullptr;
}

template <int V, typename R>
std::unique_ptr<FastPlan> make_small_rdft(size_t n, const void* tab, uint32_t nmax, int dev) {
  switch (n) {
    case 2:
      if constexpr (sizeof(R) == 8) return std::make_unique<SmallPlanImpl<V, R, 1, 1>>(tab, nmax, dev);
      break;
    case 4: return std::make_unique<SmallPlanImpl<V, R, 2, 1>>(tab, nmax, dev);
    case 8: return std::make_unique<SmallPlanImpl<V, R, 3, 1>>(tab, nmax, dev);
    case 16: return std::make_unique<SmallPlanImpl<V, R, 4, 1>>(tab, nmax, dev);
    case 32: return std::make_unique<SmallPlanImpl<V, R, 5, 1>>(tab, nmax, dev);
    case 64: return std::make_unique<SmallPlanImpl<V, R, 6, 1>>(tab, nmax, dev);
    case 128:
      if constexpr (sizeof(R) == 4) return std::make_unique<SmallPlanImpl<V, R, 7, 1>>(tab, nmax, dev);
      break;
  }
  return nullptr;
}

// ---- DCT-0 / DST-0 rows (FunctionId::Dct / Dst, N/2 + 1 / N/2 - 1 cells,
// oracle.hpp:38-41): scalar cells.  A 128-row tile is contiguous in global
// memory (a multiple of 16 bytes), so one bulk copy brings it in; the odd
// row stride makes lane-per-row scalar accesses conflict-free.  The rows
// past the last full tile are read and written straight from global memory.
template <typename R> struct ScalarIO {
  R* p;
  __device__ __forceinline__ void ld(int c, R& a) const { a = p[c]; }
  __device__ __forceinline__ void st(int c, R a) const { p[c] = a; }
};
template <typename R> struct GScalarIO {
  const R* pi;   // may alias po (in-place rows)
  R* po;
  __device__ __forceinline__ void ld(int c, R& a) const { a = pi[c]; }
  __device__ __forceinline__ void st(int c, R a) const { po[c] = a; }
};

template <typename R, int LOGN, int F>
struct KCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int CELLS = F == 2 ? N / 2 + 1 : N / 2 - 1;
  static constexpr int NT = (N < 8 ? 8 : N) / 4;
  static constexpr int T = 128;
  static constexpr uint32_t TILEB = static_cast<uint32_t>(T) * CELLS * sizeof(R);
  static constexpr size_t SMEM = TILEB + 16;
  static_assert(TILEB % 16 == 0, "bulk copies move multiples of 16 bytes");
};

template <int V, typename R, int LOGN, int F>
__global__ void __launch_bounds__(128)
k_scalar(const R* __restrict__ in, R* __restrict__ out, size_t rows,
         const __grid_constant__ TabP<R, KCfg<R, LOGN, F>::NT> tp) {
  using C = KCfg<R, LOGN, F>;
  using G = SmallGen<V, F, LOGN, R>;
  extern __shared__ __align__(128) unsigned char sm[];
  R* tile_s = reinterpret_cast<R*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::TILEB);
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;
  const size_t full = rows / C::T;
  for (size_t tile = blockIdx.x; tile < full; tile += gridDim.x) {
    const R* src = in + tile * C::T * C::CELLS;
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(s_u32(bar)), "r"(C::TILEB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(s_u32(tile_s)), "l"(src), "r"(C::TILEB), "r"(s_u32(bar)) : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(s_u32(bar)), "r"(parity) : "memory");
    parity ^= 1;
    ScalarIO<R> io{tile_s + tid * C::CELLS};
    G::template run<Arith<R>>(io, tp.v);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(out + tile * C::T * C::CELLS), "r"(s_u32(tile_s)), "r"(C::TILEB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (blockIdx.x == gridDim.x - 1) {   // rows past the last full tile
    const size_t row = full * C::T + tid;
    if (row < rows) {
      GScalarIO<R> io{in + row * C::CELLS, out + row * C::CELLS};
      G::template run<Arith<R>>(io, tp.v);
    }
  }
}

template <int V, typename R, int LOGN, int F>
class ScalarPlanImpl final : public FastPlan {
  using C = KCfg<R, LOGN, F>;

 public:
  ScalarPlanImpl(const void* tab, uint32_t nmax, int device) {
    cudaError_t e = fetch_table(tp_.v, C::NT, tab, nmax);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    auto f0 = k_scalar<V, R, LOGN, F>;
    if (C::SMEM > 48 * 1024) {
      e = cudaFuncSetAttribute(f0, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
      if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f0, C::T, C::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    grid_cap_ = std::max(1, per_sm) * sms;
    launches = 1;
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    if (inverse) throw std::invalid_argument("the inverse is defined for CDFT plans only");
    const size_t full = rows / C::T;
    const unsigned grid = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(full, grid_cap_)));
    k_scalar<V, R, LOGN, F><<<grid, C::T, C::SMEM, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                         tp_);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }

 private:
  TabP<R, C::NT> tp_{};
  int grid_cap_ = 148;
};

template <int V, typename R>
std::unique_ptr<FastPlan> make_small_dctdst(int fn, size_t n, const void* tab, uint32_t nmax, int dev) {
#define AMQFT_SCALAR_CASE(LG)                                                                         \
  case (1 << LG):                                                                                     \
    if (fn == AMQFT_FN_DCT) return std::make_unique<ScalarPlanImpl<V, R, LG, 2>>(tab, nmax, dev);     \
    if (LG >= 3) return std::make_unique<ScalarPlanImpl<V, R, (LG >= 3 ? LG : 3), 3>>(tab, nmax, dev); \
    break;
  switch (n) {
    AMQFT_SCALAR_CASE(2)
    AMQFT_SCALAR_CASE(3)
    AMQFT_SCALAR_CASE(4)
    AMQFT_SCALAR_CASE(5)
    AMQFT_SCALAR_CASE(6)
    AMQFT_SCALAR_CASE(7)
    case 256:
      if constexpr (sizeof(R) == 4) {
        if (fn == AMQFT_FN_DCT) return std::make_unique<ScalarPlanImpl<V, R, 8, 2>>(tab, nmax, dev);
        return std::make_unique<ScalarPlanImpl<V, R, 8, 3>>(tab, nmax, dev);
      }
      break;
  }
#undef AMQFT_SCALAR_CASE
  return nullptr;
}

}  // namespace smallk
}  // namespace amqft_b200
