// fourstep.cu -- large-N CDFT (N = N1 * N2 >= 2^20) as a four-step
// decomposition whose two DFT passes are the fused AM-QFT kernel
// (fast_kernel.cuh) on rows of length N1 and N2 (BASELINE config 4:
// N = 2^24 = 4096 x 4096; SURVEY §8(d) C4, §8(e) C5 local passes).
//
//   n = N2 n1 + n2,  k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_n2 w_N2^(n2 k2) [ w_N^(n2 k1) sum_n1 x[N2 n1 + n2] w_N1^(n1 k1) ]
//
//   1. transpose   x as [n1][n2] -> A[n2][n1]            (re/im swap for the inverse)
//   2. AM-QFT      N2 rows of length N1, in place         (fused kernel, variant v)
//   3. twiddle + transpose  A[n2][k1] w_N^(n2 k1) -> B[k1][n2]
//   4. AM-QFT      N1 rows of length N2                   (fused kernel, variant v)
//   5. transpose   Z[k1][k2] -> X[k2][k1] = natural order (swap + 1/N for the inverse)
//
// The AM-QFT recursion itself is not preserved across the split (the
// sub-transforms are), so this path is "fast order" only (fp32, and fp64
// for config 3's large sizes); its accuracy is checked against the fp64
// oracle of the same variant.  Sub-transforms: the fused kernel (N1, N2 >=
// 1024) or the small-CDFT kernels (<= 512 fp32 / 256 fp64).
// Twiddles w_N^j = exp(-2 pi i j / N): TRIG_TABLE = two half-size tables
// w^(jh B) and w^(jl) (B = 2^ceil(lg N / 2)) multiplied in fp64;
// TRIG_ONTHEFLY = sincospi of the exact integer phase 2 (j mod N) / N per
// element: sincospif for fp32 plans (no table reads: the lane-scattered
// table lookups were the slow part of the twiddle passes), fp64 sincospi
// for fp64 plans.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fast.cuh"
#include <cstdlib>

#include "fourstep.cuh"
#include "slab.cuh"

namespace amqft_b200 {

namespace {

constexpr int TD = 32;   // transpose tile
constexpr int TR = 8;    // rows of threads per tile

// out[r][c] (C1 x R1 per matrix) = in[c][r] (R1 x C1), one matrix per
// blockIdx.z.  MODE 0: plain; 1: twiddle by w_N^(r c) (r = row of out, c =
// column of out); SWAP: exchange re/im of the input; scale multiplies the
// result.  (A swap on both sides of a transform is the swap-trick inverse.)
template <typename R> struct C2;
template <> struct C2<float> { using T = float2; static __device__ __forceinline__ T mk(float a, float b) { return make_float2(a, b); } };
template <> struct C2<double> { using T = double2; static __device__ __forceinline__ T mk(double a, double b) { return make_double2(a, b); } };

template <int MODE, bool SWAP, typename R = float>
__global__ void __launch_bounds__(TD * TR) k_transpose(const typename C2<R>::T* __restrict__ in,
                                                      typename C2<R>::T* __restrict__ out,
                                                      int R1, int C1, R scale,
                                                      const double2* __restrict__ twh,
                                                      const double2* __restrict__ twl, int logb,
                                                      int logn, int onthefly) {
  using V2 = typename C2<R>::T;
  __shared__ V2 tile[TD][TD + 1];
  const size_t mat = static_cast<size_t>(blockIdx.z) * R1 * C1;
  const int c0 = blockIdx.x * TD, r0 = blockIdx.y * TD;
#pragma unroll
  for (int j = 0; j < TD; j += TR) {
    const int r = r0 + threadIdx.y + j, c = c0 + threadIdx.x;
    V2 v = in[mat + static_cast<size_t>(r) * C1 + c];
    if (SWAP) v = C2<R>::mk(v.y, v.x);
    tile[threadIdx.y + j][threadIdx.x] = v;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < TD; j += TR) {
    const int orow = c0 + threadIdx.y + j;   // row of out = column of in
    const int ocol = r0 + threadIdx.x;
    V2 v = tile[threadIdx.x][threadIdx.y + j];
    if (MODE == 1) {
      // w_N^(orow * ocol): j = (orow * ocol) mod N
      const unsigned long long jj =
          (static_cast<unsigned long long>(orow) * static_cast<unsigned long long>(ocol)) &
          ((1ull << logn) - 1ull);
      R fr, fi;
      if constexpr (sizeof(R) == 4) {
        if (onthefly) {   // fp32 plans: sincospif of the exact integer phase (no table reads)
          float sn, cs;
          sincospif(static_cast<float>(static_cast<double>(jj) * (2.0 / static_cast<double>(1ull << logn))), &sn,
                    &cs);
          fr = cs;
          fi = -sn;
        } else {
          const double2 a = twh[jj >> logb], b = twl[jj & ((1ull << logb) - 1ull)];
          fr = static_cast<R>(a.x * b.x - a.y * b.y);
          fi = static_cast<R>(a.x * b.y + a.y * b.x);
        }
      } else {
        double wr, wi;
        if (onthefly) {
          double s, c;
          sincospi(static_cast<double>(jj) * 2.0 / static_cast<double>(1ull << logn), &s, &c);
          wr = c;
          wi = -s;
        } else {
          const double2 a = twh[jj >> logb], b = twl[jj & ((1ull << logb) - 1ull)];
          wr = a.x * b.x - a.y * b.y;
          wi = a.x * b.y + a.y * b.x;
        }
        fr = static_cast<R>(wr);
        fi = static_cast<R>(wi);
      }
      v = C2<R>::mk(v.x * fr - v.y * fi, v.x * fi + v.y * fr);
    }
    v.x *= scale;
    v.y *= scale;
    out[mat + static_cast<size_t>(orow) * R1 + ocol] = v;
  }
}

// Element-wise variant for matrices with a side below the 32-wide tile
// (four-step splits with a sub-size of 2..16): one thread per output
// element, same twiddle/swap/scale semantics.
template <int MODE, bool SWAP, typename R>
__global__ void __launch_bounds__(256) k_transpose_small(const typename C2<R>::T* __restrict__ in,
                                                        typename C2<R>::T* __restrict__ out, size_t mats,
                                                        int R1, int C1, R scale, const double2* __restrict__ twh,
                                                        const double2* __restrict__ twl, int logb, int logn,
                                                        int onthefly) {
  using V2 = typename C2<R>::T;
  const size_t per = static_cast<size_t>(R1) * C1, total = mats * per;
  for (size_t i = threadIdx.x + static_cast<size_t>(blockIdx.x) * blockDim.x; i < total;
       i += static_cast<size_t>(blockDim.x) * gridDim.x) {
    const size_t mat = i / per;
    const int e = static_cast<int>(i - mat * per);
    const int orow = e / R1, ocol = e - orow * R1;        // out is C1 x R1
    V2 v = in[mat * per + static_cast<size_t>(ocol) * C1 + orow];
    if (SWAP) v = C2<R>::mk(v.y, v.x);
    if (MODE == 1) {
      const unsigned long long jj =
          (static_cast<unsigned long long>(orow) * static_cast<unsigned long long>(ocol)) & ((1ull << logn) - 1ull);
      double wr, wi;
      if (onthefly) {
        double sn, cs;
        sincospi(static_cast<double>(jj) * 2.0 / static_cast<double>(1ull << logn), &sn, &cs);
        wr = cs;
        wi = -sn;
      } else {
        const double2 a = twh[jj >> logb], b = twl[jj & ((1ull << logb) - 1ull)];
        wr = a.x * b.x - a.y * b.y;
        wi = a.x * b.y + a.y * b.x;
      }
      const R fr = static_cast<R>(wr), fi = static_cast<R>(wi);
      v = C2<R>::mk(v.x * fr - v.y * fi, v.x * fi + v.y * fr);
    }
    out[i] = C2<R>::mk(v.x * scale, v.y * scale);
  }
}

template <int MODE, bool SWAP, typename R = float>
void launch_t(const typename C2<R>::T* in, typename C2<R>::T* out, size_t mats, int R1, int C1, R scale,
              const double2* twh, const double2* twl, int logb, int logn, int onthefly, cudaStream_t st) {
  if (R1 % TD || C1 % TD) {
    const size_t total = mats * static_cast<size_t>(R1) * C1;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 32));
    k_transpose_small<MODE, SWAP, R><<<grid, 256, 0, st>>>(in, out, mats, R1, C1, scale, twh, twl, logb, logn,
                                                           onthefly);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("k_transpose_small: ") + cudaGetErrorString(e));
    return;
  }
  // grid.z is limited to 65535: loop over chunks of matrices
  for (size_t m0 = 0; m0 < mats; m0 += 65535) {
    const unsigned nz = static_cast<unsigned>(std::min<size_t>(65535, mats - m0));
    const dim3 grid(C1 / TD, R1 / TD, nz), block(TD, TR);
    const size_t off = m0 * static_cast<size_t>(R1) * C1;
    k_transpose<MODE, SWAP, R><<<grid, block, 0, st>>>(in + off, out + off, R1, C1, scale, twh, twl, logb, logn,
                                                        onthefly);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("k_transpose: ") + cudaGetErrorString(e));
}

// Three-factor four-step, last pass: U[mat][k1][jb][jc] (dims A, B, C) ->
// Y[mat][jc][jb][k1], i.e. for every (mat, jb) the A x C matrix of rows k1
// (stride B C) transposed into rows jc (stride B A); 32 x 32 tiles.
// SWAP / scale: the swap-trick inverse's second half.
template <bool SWAP, typename R>
__global__ void __launch_bounds__(TD * TR) k_transpose3(const typename C2<R>::T* __restrict__ in,
                                                       typename C2<R>::T* __restrict__ out, int A, int B, int Cc,
                                                       R scale) {
  using V2 = typename C2<R>::T;
  __shared__ V2 tile[TD][TD + 1];
  const size_t z = blockIdx.z;                    // mat * B + jb
  const size_t mat = z / B, jb = z - mat * B;
  const int c0 = blockIdx.x * TD, r0 = blockIdx.y * TD;   // jc block, k1 block
  const size_t base_in = mat * size_t(A) * B * Cc + jb * Cc;
  const size_t base_out = mat * size_t(A) * B * Cc + jb * A;
#pragma unroll
  for (int j = 0; j < TD; j += TR) {
    const int k1 = r0 + threadIdx.y + j, jc = c0 + threadIdx.x;
    V2 v = in[base_in + size_t(k1) * B * Cc + jc];
    if (SWAP) v = C2<R>::mk(v.y, v.x);
    tile[threadIdx.y + j][threadIdx.x] = v;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < TD; j += TR) {
    const int jc = c0 + threadIdx.y + j, k1 = r0 + threadIdx.x;
    const V2 v = tile[threadIdx.x][threadIdx.y + j];
    out[base_out + size_t(jc) * B * A + k1] = C2<R>::mk(v.x * scale, v.y * scale);
  }
}

template <bool SWAP, typename R>
void launch_t3(const typename C2<R>::T* in, typename C2<R>::T* out, size_t mats, int A, int B, int Cc, R scale,
               cudaStream_t st) {
  // grid.z <= 65535: chunks of whole matrices (a multiple of B slices)
  const size_t zs = mats * B, step = (65535 / static_cast<size_t>(B)) * B;
  for (size_t z0 = 0; z0 < zs; z0 += step) {
    const unsigned nz = static_cast<unsigned>(std::min<size_t>(step, zs - z0));
    const size_t off = (z0 / B) * size_t(A) * B * Cc;
    k_transpose3<SWAP, R><<<dim3(Cc / TD, A / TD, nz), dim3(TD, TR), 0, st>>>(in + off, out + off, A, B, Cc, scale);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("k_transpose3: ") + cudaGetErrorString(e));
}

// Distributed four-step, one rank's half-way step: rows n2 = row0 + r
// (r < rows) of length N1 (already transformed over n1) are multiplied by
// w_N^(n2 k1) and scattered by k1-slab: destination q receives the
// columns k1 in [q N1/P, (q+1) N1/P) at dst[q] + src * rows * (N1/P),
// laid out [r][k1 - q N1/P].  dst[] are device pointers: the local send
// buffer slots (then an all-to-all) or the peers' receive buffers mapped
// over NVLink (the transfer is the kernel's own stores).
constexpr int kMaxParts = 64;
struct DstPtrs {
  float2* p[kMaxParts];
};

// Each thread takes 4 consecutive k1 of one row (two 16-byte loads and
// stores; w = n1 / nparts is a multiple of 4, so they share a slab) and
// one twiddle evaluation: w^(n2 (k1 + e)) = w^(n2 k1) (w^n2)^e in fp64.
__device__ __forceinline__ void scatter_tw(unsigned long long jj, int logn, const double2* __restrict__ twh,
                                           const double2* __restrict__ twl, int logb, int onthefly, double& wr,
                                           double& wi) {
  jj &= (1ull << logn) - 1ull;
  if (onthefly) {   // fp32 data: sincospif of the exact integer phase (as the fp32 four-step)
    float sn, cs;
    sincospif(static_cast<float>(static_cast<double>(jj) * (2.0 / static_cast<double>(1ull << logn))), &sn, &cs);
    wr = cs;
    wi = -sn;
  } else {
    const double2 a = twh[jj >> logb], b = twl[jj & ((1ull << logb) - 1ull)];
    wr = a.x * b.x - a.y * b.y;
    wi = a.x * b.y + a.y * b.x;
  }
}

__global__ void __launch_bounds__(256) k_twiddle_scatter(const float2* __restrict__ in, const DstPtrs dst,
                                                         int rows, int n1, int logn, long long row0, int src,
                                                         int nparts, const double2* __restrict__ twh,
                                                         const double2* __restrict__ twl, int logb, int onthefly) {
  const int w = n1 / nparts;
  const long long total = static_cast<long long>(rows) * (n1 / 4);
  for (long long i = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; i < total;
       i += static_cast<long long>(blockDim.x) * gridDim.x) {
    const int r = static_cast<int>(i / (n1 / 4)), k1 = 4 * static_cast<int>(i % (n1 / 4));
    const unsigned long long n2 = static_cast<unsigned long long>(row0 + r);
    double cr, ci, sr, si;
    scatter_tw(n2 * static_cast<unsigned long long>(k1), logn, twh, twl, logb, onthefly, cr, ci);
    scatter_tw(n2, logn, twh, twl, logb, onthefly, sr, si);
    const float4* src4 = reinterpret_cast<const float4*>(in + static_cast<long long>(r) * n1 + k1);
    const float4 u0 = src4[0], u1 = src4[1];
    const float v[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float fr = static_cast<float>(cr), fi = static_cast<float>(ci);
      o[2 * e] = v[2 * e] * fr - v[2 * e + 1] * fi;
      o[2 * e + 1] = v[2 * e] * fi + v[2 * e + 1] * fr;
      const double tr = cr * sr - ci * si, ti = cr * si + ci * sr;
      cr = tr;
      ci = ti;
    }
    const int q = k1 / w, kl = k1 - q * w;
    float4* d4 = reinterpret_cast<float4*>(dst.p[q] + (static_cast<long long>(src) * rows + r) * w + kl);
    d4[0] = make_float4(o[0], o[1], o[2], o[3]);
    d4[1] = make_float4(o[4], o[5], o[6], o[7]);
  }
}

// The same scatter for rows left in a column-mode four-step's transposed
// order in[r][ka][kb] = row value at k1 = ka + A kb (A x B, B = n1 / A):
// the four-step's final transpose folded in.  32 x 32 tiles (ka, kb) per
// row: reads coalesced along kb, writes along ka (consecutive k1, one
// slab when w is a multiple of 32); per thread 4 (8 on 64-wide tiles) elements
// kb + 8 j share one twiddle evaluation and a recurrence (step w^(8 A n2)).
template <int KB>   // kb per tile: 32, or 64 (8 elements per twiddle evaluation) where n1 / A allows
__global__ void __launch_bounds__(256) k_twiddle_scatter_t(const float2* __restrict__ in, const DstPtrs dst,
                                                           int rows, int n1, int A, int logn, long long row0,
                                                           int src, int nparts, const double2* __restrict__ twh,
                                                           const double2* __restrict__ twl, int logb, int onthefly) {
  __shared__ float2 tile[KB][33];   // [kb][ka]
  const int B = n1 / A, w = n1 / nparts;
  const int r = blockIdx.z;
  const int kb0 = blockIdx.x * KB, ka0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const float2* row = in + static_cast<long long>(r) * n1;
#pragma unroll
  for (int h = 0; h < KB; h += 32)
#pragma unroll
    for (int j = 0; j < 32; j += 8)
      tile[h + tx][ty + j] = row[static_cast<long long>(ka0 + ty + j) * B + kb0 + h + tx];
  __syncthreads();
  const unsigned long long n2 = static_cast<unsigned long long>(row0 + r);
  const int ka = ka0 + tx;
  double cr, ci, sr, si;
  scatter_tw(n2 * static_cast<unsigned long long>(ka + A * (kb0 + ty)), logn, twh, twl, logb, onthefly, cr, ci);
  scatter_tw(n2 * static_cast<unsigned long long>(8 * A), logn, twh, twl, logb, onthefly, sr, si);
#pragma unroll
  for (int j = 0; j < KB; j += 8) {
    const int kb = kb0 + ty + j;
    const float2 v = tile[ty + j][tx];
    const float fr = static_cast<float>(cr), fi = static_cast<float>(ci);
    const int k1 = ka + A * kb;
    const int q = k1 / w, kl = k1 - q * w;
    dst.p[q][(static_cast<long long>(src) * rows + r) * w + kl] =
        make_float2(v.x * fr - v.y * fi, v.x * fi + v.y * fr);
    const double t0 = cr * sr - ci * si, t1 = cr * si + ci * sr;
    cr = t0;
    ci = t1;
  }
}

// The scatter and the exchange-side transpose in one kernel ("direct" mode):
// element (n2, k1) of the local rows goes straight to its place in the
// destination rank's [n1 / parts][n2_total] rows, dst[k1 / w][(k1 % w)
// n2_total + n2], times w_N^(n2 k1) -- into the peers' mapped buffers, or the
// rank's own when there is one part.  The rows come in the column-mode
// four-step's transposed order in[r][ka][kb], k1 = ka + A kb (A = 1: plain
// rows).  32 x 32 tiles (r, kb) for a fixed ka: reads coalesced along kb,
// writes along n2; per thread 4 elements kb + 8 j share one twiddle
// evaluation and a recurrence (step w^(8 A n2)).
template <int KB>   // kb per tile: 32, or 64 (8 elements per twiddle evaluation) where n1 / A allows
__global__ void __launch_bounds__(256) k_twiddle_scatter_direct(const float2* __restrict__ in, const DstPtrs dst,
                                                                int n1, int A, int logn, long long row0,
                                                                long long n2_total, int nparts,
                                                                const double2* __restrict__ twh,
                                                                const double2* __restrict__ twl, int logb,
                                                                int onthefly) {
  __shared__ float2 tile[KB][33];
  const int B = n1 / A, w = n1 / nparts;
  const int ka = blockIdx.z;
  const int kb0 = blockIdx.x * KB, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  // tile[kb][r]: rows read along kb (coalesced), 32 kb per pass
#pragma unroll
  for (int h = 0; h < KB; h += 32)
#pragma unroll
    for (int j = 0; j < 32; j += 8)
      tile[h + tx][ty + j] =
          in[static_cast<long long>(r0 + ty + j) * n1 + static_cast<long long>(ka) * B + kb0 + h + tx];
  __syncthreads();
  const unsigned long long n2 = static_cast<unsigned long long>(row0 + r0 + tx);
  double cr, ci, sr, si;
  scatter_tw(n2 * static_cast<unsigned long long>(ka + A * (kb0 + ty)), logn, twh, twl, logb, onthefly, cr, ci);
  scatter_tw(n2 * static_cast<unsigned long long>(8 * A), logn, twh, twl, logb, onthefly, sr, si);
#pragma unroll
  for (int j = 0; j < KB; j += 8) {
    const int kb = kb0 + ty + j;
    const float2 v = tile[ty + j][tx];
    const float fr = static_cast<float>(cr), fi = static_cast<float>(ci);
    const int k1 = ka + A * kb;
    const int q = k1 / w, kl = k1 - q * w;
    dst.p[q][static_cast<long long>(kl) * n2_total + static_cast<long long>(n2)] =
        make_float2(v.x * fr - v.y * fi, v.x * fi + v.y * fr);
    const double t0 = cr * sr - ci * si, t1 = cr * si + ci * sr;
    cr = t0;
    ci = t1;
  }
}

int lg2(size_t v) {
  int l = 0;
  while ((size_t(1) << l) < v) ++l;
  return l;
}

// Split N = N1 N2 over covered sub-sizes (both >= 32 from N = 2^10 on, for
// the tiled transposes; below that the element-wise transpose), and the
// column mode where N1 is a one-thread-per-row size,
// minimising the two DFT passes' and the transposes' time by the measured HBM
// throughput of each sub-size (B200, TB/s; tools/sweep_c3.py,
// tools/prof_fast.py).
double sub_tbs(int dtype, int lg, int variant, bool col = false) {
  static const double f32[14] = {0, 5.0, 5.0, 5.0, 5.0, 5.0, 5.0, 3.9, 1.78, 1.26, 1.72, 2.43, 3.17, 2.09};
  static const double f64[13] = {0, 5.5, 5.5, 5.5, 5.5, 5.5, 5.4, 2.94, 2.06, 0.0, 2.27, 2.68, 2.88};
  // fp32 rows through the fp64 instance (variants 5-8, fast.cuh): half the fp64 row bytes
  static const double mixed[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1.13, 1.34, 1.44};
  // in-shared-memory four-step (tile_kernel.cuh): fp32 N = 16 .. 65536, all variants
  static const double tile[17] = {0, 0, 0, 0, 5.18, 6.5, 5.78, 6.25, 5.85, 6.3, 6.2, 5.5, 5.63, 5.75, 5.09, 3.76, 3.03};
  if (!col && dtype == AMQFT_F32 && lg >= 4 && lg <= 16) {
    amqft_plan_desc d{};
    d.function = AMQFT_FN_CDFT;
    d.dtype = dtype;
    d.n = size_t(1) << lg;
    d.variant = variant;
    if (tile_covers(d)) return tile[lg];
  }
  // fp64 (variants 1-4 to 2^15, 5-8 to 2^8: fast.cu tile_covers)
  static const double tile64[16] = {0, 0, 0, 0, 0, 0, 5.97, 6.36, 5.59, 5.68, 5.48, 6.11, 5.26, 5.04, 3.85, 3.01};
  if (!col && dtype == AMQFT_F64 && lg >= 6 && lg <= 15) {
    amqft_plan_desc d{};
    d.function = AMQFT_FN_CDFT;
    d.dtype = dtype;
    d.n = size_t(1) << lg;
    d.variant = variant;
    if (tile_covers(d)) return tile64[lg];
  }
  if (dtype == AMQFT_F32 && lg < 13 && f32_needs_f64_compute(variant, size_t(1) << lg)) return mixed[lg];
  if (dtype == AMQFT_F32) return lg < 14 ? f32[lg] : 0.0;
  return lg < 13 ? f64[lg] : 0.0;
}

// Column mode: the first pass runs the one-thread-per-row kernel straight
// on the columns of x (coalesced: a warp's lanes take consecutive columns)
// with the twiddle fused into its stores, so transposes 1 and 2 vanish.
bool col_capable(int dtype, int lg) { return lg >= 1 && lg <= (dtype == AMQFT_F32 ? 6 : 5); }

bool fourstep_split(int dtype, size_t n, int variant, size_t* n1, size_t* n2, bool* col = nullptr) {
  constexpr double kTransposeTBs = 6.9;   // measured k_transpose (B200)
  const int lg = lg2(n);
  double best = 0.0;
  for (int l1 = 1; l1 < lg; ++l1) {
    const int l2 = lg - l1;
    if (!fast_sub_covered(dtype, size_t(1) << l1, variant) || !fast_sub_covered(dtype, size_t(1) << l2, variant))
      continue;
    const double b = sub_tbs(dtype, l2, variant);
    for (int c = 0; c < 2; ++c) {
      if (c == 1 && !col_capable(dtype, l1)) continue;
      const double a = sub_tbs(dtype, l1, variant, c == 1);
      if (a <= 0.0 || b <= 0.0) continue;
      // tiled transposes need both sides >= 32 from N = 2^10 on (column
      // mode: only the last transpose, N1 x N2)
      if (c == 0 && (l1 < 5 || l2 < 5) && lg >= 10) continue;
      if (c == 1 && (l1 < 5 || l2 < 5) && lg >= 10) continue;
      const double cost = 1.0 / a + 1.0 / b + (c ? 1.0 : 3.0) / kTransposeTBs;
      if (best == 0.0 || cost < best - 1e-9) {
        best = cost;
        *n1 = size_t(1) << l1;
        *n2 = size_t(1) << l2;
        if (col) *col = c == 1;
      }
    }
  }
  return best > 0.0;
}

// Three-factor mode: N = A B C, A and B one-thread-per-row sizes (column
// passes, coalesced, twiddles fused into their stores), C a single-kernel
// row size, and one 3D transpose: 4 passes.  Chosen when cheaper than the
// best two-factor plan by the same throughput model.
bool fourstep_split3(int dtype, size_t n, int variant, size_t* a, size_t* b, size_t* c, double* cost) {
  constexpr double kTransposeTBs = 6.9;
  const int lg = lg2(n);
  double best = 0.0;
  // column factors up to 64 (one thread per column): with the per-column
  // twiddle recurrence the 64-point column pass moves 4.3 TB/s (N = 2^24 as
  // 64 x 64 x 4096: 0.262 ms vs 0.335 ms for the two-factor 4096 x 4096)
  for (int la = 5; la <= 6; ++la)
    for (int lb = 1; lb <= 6; ++lb) {
      const int lc = lg - la - lb;
      if (lc < 5 || !col_capable(dtype, la) || !col_capable(dtype, lb)) continue;
      if (!fast_sub_covered(dtype, size_t(1) << lc, variant)) continue;
      const double ta = sub_tbs(dtype, la, variant, true), tb = sub_tbs(dtype, lb, variant, true),
                   tc = sub_tbs(dtype, lc, variant);
      if (ta <= 0.0 || tb <= 0.0 || tc <= 0.0) continue;
      const double cst = 1.0 / ta + 1.0 / tb + 1.0 / tc + 1.0 / kTransposeTBs;
      if (best == 0.0 || cst < best - 1e-9) {
        best = cst;
        *a = size_t(1) << la;
        *b = size_t(1) << lb;
        *c = size_t(1) << lc;
      }
    }
  if (cost) *cost = best;
  return best > 0.0;
}

double fourstep_cost2(int dtype, int variant, size_t n1, size_t n2, bool col) {
  return 1.0 / sub_tbs(dtype, lg2(n1), variant, col) + 1.0 / sub_tbs(dtype, lg2(n2), variant) + (col ? 1.0 : 3.0) / 6.9;
}

// The factors a four-step plan runs: two-factor (n1 x n2, column mode or
// three transposes) or three-factor (a x b x c), by the same cost model
// the plan uses.
struct FourStepShape {
  bool ok = false, col = false, three = false;
  size_t n1 = 0, n2 = 0, nb = 0;   // three-factor: n1 = A, nb = B, n2 = C
};

FourStepShape fourstep_shape(int dtype, int variant, size_t n) {
  FourStepShape s;
  const bool two = fourstep_split(dtype, n, variant, &s.n1, &s.n2, &s.col);
  double c3 = 0.0;
  size_t a3 = 0, b3 = 0, cc3 = 0;
  s.three = fourstep_split3(dtype, n, variant, &a3, &b3, &cc3, &c3) &&
            (!two || c3 < fourstep_cost2(dtype, variant, s.n1, s.n2, s.col) - 1e-9);
  if (s.three) {
    s.n1 = a3;
    s.nb = b3;
    s.n2 = cc3;
    s.col = true;
  }
  s.ok = two || s.three;
  return s;
}

template <typename R>
class FourStepPlan final : public FastPlan {
  using V2 = typename C2<R>::T;

 public:
  FourStepPlan(int variant, size_t n, size_t batch, int trig_mode, const void* tab, uint32_t nmax, int dev,
               const void* tab64)
      : n_(n), batch_(batch), onthefly_(trig_mode == AMQFT_TRIG_ONTHEFLY) {
    logn_ = lg2(n);
    const int dtype = sizeof(R) == 8 ? AMQFT_F64 : AMQFT_F32;
    const FourStepShape sh = fourstep_shape(dtype, variant, n);
    if (!sh.ok) throw std::invalid_argument("four-step: no covered split");
    n1_ = sh.n1;
    n2_ = sh.n2;
    nb_ = sh.nb;
    col_ = sh.col;
    three_ = sh.three;
    if (three_) {   // p1_: A columns, pb_: B columns, p2_: C rows
      pb_ = make_fast_sub(variant, nb_, dtype, tab, nmax, dev, tab64, true);
      if (!pb_) throw std::invalid_argument("four-step: no kernel for the middle factor");
    }
    p1_ = make_fast_sub(variant, n1_, dtype, tab, nmax, dev, tab64, col_);
    p2_ = make_fast_sub(variant, n2_, dtype, tab, nmax, dev, tab64);
    if (!p1_ || !p2_) throw std::invalid_argument("four-step: no fused kernel for the sub-transform sizes");
    // half-size twiddle tables: w^(jh B), w^(jl), long double -> double
    logb_ = (logn_ + 1) / 2;
    const size_t B = size_t(1) << logb_, NH = n >> logb_;
    std::vector<double2> th(NH), tl(B);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (size_t j = 0; j < NH; ++j) {
      const long double a = two_pi * static_cast<long double>(j << logb_) / static_cast<long double>(n);
      th[j] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    for (size_t j = 0; j < B; ++j) {
      const long double a = two_pi * static_cast<long double>(j) / static_cast<long double>(n);
      tl[j] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    check(cudaMalloc(&twh_, NH * sizeof(double2)), "cudaMalloc twiddles");
    check(cudaMalloc(&twl_, B * sizeof(double2)), "cudaMalloc twiddles");
    check(cudaMemcpy(twh_, th.data(), NH * sizeof(double2), cudaMemcpyHostToDevice), "cudaMemcpy");
    check(cudaMemcpy(twl_, tl.data(), B * sizeof(double2), cudaMemcpyHostToDevice), "cudaMemcpy");
    check(cudaMalloc(&scratch_, batch_ * n_ * sizeof(V2)), "cudaMalloc four-step scratch");
    if (three_) check(cudaMalloc(&scratch2_, batch_ * n_ * sizeof(V2)), "cudaMalloc four-step scratch");
    launches = three_ ? 4 : (col_ ? 1 + p1_->launches + p2_->launches : 3 + p1_->launches + p2_->launches);
  }
  size_t transposed_factor() const override { return (col_ && !three_) ? n1_ : 0; }
  void exec_transposed(const void* in, void* out, size_t rows, cudaStream_t st) override {
    if (!col_ || three_) throw std::invalid_argument("transposed output needs a column-mode four-step");
    ColTwiddle tw;
    tw.hi = twh_;
    tw.lo = twl_;
    tw.logb = logb_;
    tw.logn = logn_;
    tw.onthefly = onthefly_ ? 1 : 0;
    if (!p1_->exec_columns(in, scratch_, rows, n2_, 0, tw, st))
      throw std::runtime_error("four-step: sub-plan has no column mode");
    p2_->exec(scratch_, out, rows * n1_, 0, st);
  }
  ~FourStepPlan() override {
    if (scratch2_) cudaFree(scratch2_);
    if (twh_) cudaFree(twh_);
    if (twl_) cudaFree(twl_);
    if (scratch_) cudaFree(scratch_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    if (rows > batch_) throw std::invalid_argument("rows exceed the plan batch");
    const V2* x = static_cast<const V2*>(in);
    V2* y = static_cast<V2*>(out);
    V2* s = scratch_;
    const int R1 = static_cast<int>(n1_), C1 = static_cast<int>(n2_);
    if (three_) {
      // x [a][b][c] (dims A, B, C): columns over a (length A, stride B C),
      // times w_N^((b C + c) ka) -> s [ka][b][c]
      ColTwiddle tw;
      tw.hi = twh_;
      tw.lo = twl_;
      tw.logb = logb_;
      tw.logn = logn_;
      tw.onthefly = onthefly_ ? 1 : 0;
      if (!p1_->exec_columns(x, s, rows, nb_ * n2_, inverse, tw, st))
        throw std::runtime_error("four-step: sub-plan has no column mode");
      // rows ka of length M = B C: columns over b (stride C), times
      // w_M^(c kb) = w_N^(A c kb) -> s2 [ka][kb][c]
      tw.mul = n1_;
      if (!pb_->exec_columns(s, scratch2_, rows * n1_, n2_, 0, tw, st))
        throw std::runtime_error("four-step: sub-plan has no column mode");
      // rows of length C, in place: s2 [ka][kb][kc] = X[ka + A (kb + B kc)]
      p2_->exec(scratch2_, scratch2_, rows * n1_ * nb_, 0, st);
      // s2 [ka][kb][kc] -> y [kc][kb][ka]
      if (inverse)
        launch_t3<true, R>(scratch2_, y, rows, R1, static_cast<int>(nb_), C1, R(1) / static_cast<R>(n_), st);
      else
        launch_t3<false, R>(scratch2_, y, rows, R1, static_cast<int>(nb_), C1, R(1), st);
      return;
    }
    if (col_) {
      // 1+2+3. columns of x [n1][n2] -> s [k1][n2], times w^(n2 k1)
      ColTwiddle tw;
      tw.hi = twh_;
      tw.lo = twl_;
      tw.logb = logb_;
      tw.logn = logn_;
      tw.onthefly = onthefly_ ? 1 : 0;
      if (!p1_->exec_columns(x, s, rows, n2_, inverse, tw, st))
        throw std::runtime_error("four-step: sub-plan has no column mode");
      // 4. rows of length N2, in place: s [k1][k2]
      p2_->exec(s, s, rows * n1_, 0, st);
      // 5. s [k1][k2] -> y [k2][k1]
      if (inverse)
        launch_t<0, true, R>(s, y, rows, R1, C1, R(1) / static_cast<R>(n_), nullptr, nullptr, 0, logn_, 0, st);
      else
        launch_t<0, false, R>(s, y, rows, R1, C1, R(1), nullptr, nullptr, 0, logn_, 0, st);
      return;
    }
    // 1. x [n1][n2] -> s [n2][n1]
    if (inverse)
      launch_t<0, true, R>(x, s, rows, R1, C1, R(1), nullptr, nullptr, 0, logn_, 0, st);
    else
      launch_t<0, false, R>(x, s, rows, R1, C1, R(1), nullptr, nullptr, 0, logn_, 0, st);
    // 2. rows of length N1
    p1_->exec(s, s, rows * n2_, 0, st);
    // 3. s [n2][k1] * w^(n2 k1) -> y [k1][n2]
    launch_t<1, false, R>(s, y, rows, C1, R1, R(1), twh_, twl_, logb_, logn_, onthefly_ ? 1 : 0, st);
    // 4. rows of length N2: y -> s [k1][k2]
    p2_->exec(y, s, rows * n1_, 0, st);
    // 5. s [k1][k2] -> y [k2][k1]
    if (inverse)
      launch_t<0, true, R>(s, y, rows, R1, C1, R(1) / static_cast<R>(n_), nullptr, nullptr, 0, logn_, 0, st);
    else
      launch_t<0, false, R>(s, y, rows, R1, C1, R(1), nullptr, nullptr, 0, logn_, 0, st);
  }

 private:
  static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
  size_t n_, batch_, n1_ = 0, n2_ = 0;
  int logn_ = 0, logb_ = 0;
  bool onthefly_;
  bool col_ = false;
  bool three_ = false;   // N = A B C: two column passes, rows, one 3D transpose
  size_t nb_ = 0;
  std::unique_ptr<FastPlan> pb_;
  V2* scratch2_ = nullptr;
  std::unique_ptr<FastPlan> p1_, p2_;
  double2* twh_ = nullptr;
  double2* twl_ = nullptr;
  V2* scratch_ = nullptr;
};

}  // namespace

// Half-size twiddle tables for w_N (fp64, from long double).
struct Twiddles {
  double2* hi = nullptr;
  double2* lo = nullptr;
  int logb = 0, logn = 0;
  explicit Twiddles(size_t n) {
    logn = lg2(n);
    logb = (logn + 1) / 2;
    const size_t B = size_t(1) << logb, NH = n >> logb;
    std::vector<double2> th(NH), tl(B);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (size_t j = 0; j < NH; ++j) {
      const long double a = two_pi * static_cast<long double>(j << logb) / static_cast<long double>(n);
      th[j] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    for (size_t j = 0; j < B; ++j) {
      const long double a = two_pi * static_cast<long double>(j) / static_cast<long double>(n);
      tl[j] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    if (cudaMalloc(&hi, NH * sizeof(double2)) != cudaSuccess || cudaMalloc(&lo, B * sizeof(double2)) != cudaSuccess)
      throw std::runtime_error("cudaMalloc twiddles");
    cudaMemcpy(hi, th.data(), NH * sizeof(double2), cudaMemcpyHostToDevice);
    cudaMemcpy(lo, tl.data(), B * sizeof(double2), cudaMemcpyHostToDevice);
  }
  ~Twiddles() {
    if (hi) cudaFree(hi);
    if (lo) cudaFree(lo);
  }
};

void dist_twiddle_scatter(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                          int src, int nparts, int trig_mode, cudaStream_t st) {
  static thread_local std::unique_ptr<Twiddles> tw;
  static thread_local int tw_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!tw || (size_t(1) << tw->logn) != n || tw_dev != dev) {
    tw.reset(new Twiddles(n));
    tw_dev = dev;
  }
  if (nparts < 1 || nparts > kMaxParts || n1 % nparts || (n1 / nparts) % 4)
    throw std::invalid_argument("twiddle_scatter: bad part count (n1 / parts must be a multiple of 4)");
  DstPtrs dp{};
  for (int q = 0; q < nparts; ++q) dp.p[q] = static_cast<float2*>(d_dst[q]);
  const long long total = static_cast<long long>(rows) * static_cast<long long>(n1 / 4);
  const unsigned grid = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 148LL * 16));
  k_twiddle_scatter<<<grid, 256, 0, st>>>(static_cast<const float2*>(in), dp,
                                          static_cast<int>(rows), static_cast<int>(n1), tw->logn,
                                          static_cast<long long>(row0), src, nparts, tw->hi, tw->lo, tw->logb,
                                          trig_mode == AMQFT_TRIG_ONTHEFLY ? 1 : 0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("k_twiddle_scatter: ") + cudaGetErrorString(e));
}

void dist_twiddle_scatter_t(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                            int src, int nparts, int trig_mode, size_t a, cudaStream_t st) {
  static thread_local std::unique_ptr<Twiddles> tw;
  static thread_local int tw_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!tw || (size_t(1) << tw->logn) != n || tw_dev != dev) {
    tw.reset(new Twiddles(n));
    tw_dev = dev;
  }
  if (nparts < 1 || nparts > kMaxParts || n1 % nparts || (n1 / nparts) % 32)
    throw std::invalid_argument("twiddle_scatter_t: n1 / parts must be a multiple of 32");
  if (a == 0 || a % 32 || n1 % a || (n1 / a) % 32 || rows > 65535)
    throw std::invalid_argument("twiddle_scatter_t: A and n1 / A must be multiples of 32, rows <= 65535");
  DstPtrs dp{};
  for (int q = 0; q < nparts; ++q) dp.p[q] = static_cast<float2*>(d_dst[q]);
  const bool wide = (n1 / a) % 64 == 0;
  const dim3 grid(static_cast<unsigned>(n1 / a / (wide ? 64 : 32)), static_cast<unsigned>(a / 32),
                  static_cast<unsigned>(rows));
  auto kern = wide ? k_twiddle_scatter_t<64> : k_twiddle_scatter_t<32>;
  kern<<<grid, dim3(32, 8), 0, st>>>(static_cast<const float2*>(in), dp, static_cast<int>(rows), static_cast<int>(n1),
                                      static_cast<int>(a), tw->logn, static_cast<long long>(row0), src, nparts,
                                      tw->hi, tw->lo, tw->logb, trig_mode == AMQFT_TRIG_ONTHEFLY ? 1 : 0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("k_twiddle_scatter_t: ") + cudaGetErrorString(e));
}

void dist_twiddle_scatter_direct(const void* in, void* const* d_dst, size_t rows, size_t n1, size_t n, size_t row0,
                                 int nparts, int trig_mode, size_t a, cudaStream_t st) {
  static thread_local std::unique_ptr<Twiddles> tw;
  static thread_local int tw_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!tw || (size_t(1) << tw->logn) != n || tw_dev != dev) {
    tw.reset(new Twiddles(n));
    tw_dev = dev;
  }
  if (a == 0) a = 1;   // plain rows
  if (nparts < 1 || nparts > kMaxParts || n1 % nparts)
    throw std::invalid_argument("twiddle_scatter_direct: n1 must divide over the parts");
  if (n1 % a || (n1 / a) % 32 || rows % 32 || a > 65535 || rows / 32 > 65535)
    throw std::invalid_argument("twiddle_scatter_direct: n1 / A and rows must be multiples of 32");
  DstPtrs dp{};
  for (int q = 0; q < nparts; ++q) dp.p[q] = static_cast<float2*>(d_dst[q]);
  const bool wide = (n1 / a) % 64 == 0;
  const dim3 grid(static_cast<unsigned>(n1 / a / (wide ? 64 : 32)), static_cast<unsigned>(rows / 32),
                  static_cast<unsigned>(a));
  auto kern = wide ? k_twiddle_scatter_direct<64> : k_twiddle_scatter_direct<32>;
  kern<<<grid, dim3(32, 8), 0, st>>>(static_cast<const float2*>(in), dp, static_cast<int>(n1), static_cast<int>(a),
                                      tw->logn, static_cast<long long>(row0), static_cast<long long>(n / n1), nparts,
                                      tw->hi, tw->lo, tw->logb, trig_mode == AMQFT_TRIG_ONTHEFLY ? 1 : 0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("k_twiddle_scatter_direct: ") + cudaGetErrorString(e));
}

void transpose_c64(const void* in, void* out, size_t mats, size_t r, size_t c, cudaStream_t st) {
  if (r % TD || c % TD) throw std::invalid_argument("transpose: dimensions must be multiples of 32");
  launch_t<0, false>(static_cast<const float2*>(in), static_cast<float2*>(out), mats, static_cast<int>(r),
                     static_cast<int>(c), 1.0f, nullptr, nullptr, 0, 0, 0, st);
}

// ---- Column-slab plans (slab_kernel.cuh): N = L1 L2 in two passes, N = L1
// L2 L3 in three, L in {128, 256, 512, 1024}, natural order in and out and
// no transpose kernel.  Measured against the column / row / transpose
// four-step above (B200, GB/s on algorithmic bytes): see fourstep_slab_shape.
struct SlabShape {
  int passes = 0;
  size_t len[3] = {0, 0, 0};
};

// Balanced factors, the largest first.  Two passes for 2^14 .. 2^20, three
// for 2^21 .. 2^30.
SlabShape slab_factors(size_t n, int dtype) {
  SlabShape s;
  const int lg = lg2(n);
  if ((size_t(1) << lg) != n) return s;
  // fp32 has 2048- and 4096-point slab passes (64-point factors, 8- / 4-column slabs): two passes
  // for 2^21 .. 2^23 (measured 1875 / 1745 / 1717 GB/s against 1686 / 1603 / 1614 for the best
  // alternative; 2^24 as 4096 x 4096 loses to three 256-point passes, 1492 against 1694)
  const bool two_long = dtype == AMQFT_F32 && lg >= 21 && lg <= 23;
  if ((lg >= 14 && lg <= 20) || two_long) {
    s.passes = 2;
    s.len[0] = size_t(1) << ((lg + 1) / 2);
    s.len[1] = size_t(1) << (lg / 2);
  } else if (lg >= 21 && lg <= 30) {
    s.passes = 3;
    const int a = (lg + 2) / 3, b = (lg - a + 1) / 2, c = lg - a - b;
    s.len[0] = size_t(1) << a;
    s.len[1] = size_t(1) << b;
    s.len[2] = size_t(1) << c;
  }
  return s;
}

// Where the slab plan replaces the column / row / transpose four-step.
// AMQFT_AB_SLAB=none|all overrides (A/B measurements).
thread_local bool g_prefer_transposable = false;

SlabShape fourstep_slab_shape(const amqft_plan_desc& d) {
  SlabShape none;
  if (d.function != AMQFT_FN_CDFT || g_prefer_transposable) return none;
  const SlabShape s = slab_factors(d.n, d.dtype);
  if (!s.passes) return none;
  if (const char* e = std::getenv("AMQFT_AB_SLAB")) {
    if (e[0] == 'n') return none;
    if (e[0] == 'a') return s;
  }
  const int lg = lg2(d.n);
  // one-pass tile kernels own N <= 2^16 (fp32) / 2^15 (fp64 variants 1-4)
  amqft_plan_desc t = d;
  t.order = AMQFT_ORDER_FAST;
  if (tile_covers(t)) return none;
  // measured (B200, v4, GB/s on algorithmic bytes, slab against column + tile rows + transpose;
  // tools/slab_ab.sh): fp32 two passes 2^17-2^20 2553 / 2467 / 2178 / 2016 against 2083 / 2077 / 1970 /
  // 1893; two long passes 2^21-2^23 (slab_factors); three passes 2^24-2^26 1676 / 1522 / 1640 against
  // 1453 / 1396 / 1356.
  // fp64: 2^16 2804 against 2156, 2^19 / 2^20 1813 / 1890 against 1759 / 1565, 2^21-2^24 1603 / 1676 /
  // 1770 / 1837 against 1587 / 1512 / 1493 / 1366; 2^17 / 2^18 lose (1936 / 1608 against 2023 / 1982).
  // fp64 variants 5-8 have no one-pass tile rows above N = 256 (fast.cu tile_covers), so the older plan
  // runs on the whole-DAG kernels: slab 2^14 / 2^15 / 2^17 / 2^18 2642 / 2863 / 1979 / 1642 against 1605 /
  // 1581 / 1622 / 1575 (v6)
  if (d.dtype == AMQFT_F64 && d.variant >= 5) return lg >= 14 ? s : none;
  if (d.dtype == AMQFT_F64) return (lg == 16 || lg == 19 || lg >= 20) ? s : none;
  return lg >= 17 ? s : none;
}

template <typename R>
class SlabPlan final : public FastPlan {
  using V2 = typename C2<R>::T;

 public:
  SlabPlan(int variant, size_t n, size_t batch, int trig_mode, const void* tab, uint32_t nmax, int dev,
           const SlabShape& sh)
      : n_(n), batch_(batch), sh_(sh), tws_(n) {
    const int dtype = sizeof(R) == 8 ? AMQFT_F64 : AMQFT_F32;
    for (int i = 0; i < sh.passes; ++i) {
      pass_[i] = make_slab_pass_rt<R>(variant, sh.len[i], tab, nmax, dev);
      if (!pass_[i]) throw std::invalid_argument("slab four-step: no kernel for a factor");
    }
    (void)dtype;
    ColTwiddle tw;
    tw.hi = tws_.hi;
    tw.lo = tws_.lo;
    tw.logb = tws_.logb;
    tw.logn = tws_.logn;
    tw.onthefly = trig_mode == AMQFT_TRIG_ONTHEFLY ? 1 : 0;
    const size_t L1 = sh.len[0], L2 = sh.len[1], L3 = sh.len[2];
    using slabk::SlabPass;
    if (sh.passes == 2) {
      // pass 1: columns n2 of x [n1][n2] -> Y [n2][k1], times w_N^(n2 k1)
      SlabPass& a = p_[0];
      a.in_row = a.out_row = n;
      a.cols = a.qin = a.qout = static_cast<unsigned>(L2);
      a.sj_in = L2;
      a.transposing = 1;
      a.sj_out = 1;
      a.sw_out = L1;
      a.twiddle = 1;
      a.tw = tw;
      // pass 2: columns k1 of Y [n2][k1] -> X [k2][k1]
      SlabPass& b = p_[1];
      b.in_row = b.out_row = n;
      b.cols = b.qin = b.qout = static_cast<unsigned>(L1);
      b.sj_in = b.sj_out = L1;
    } else {
      const size_t M = L2 * L3;
      // pass 1: columns m = L3 n2 + n3 of x [n1][m] -> Y1 [n2][n3][k1], times w_N^(m k1)
      SlabPass& a = p_[0];
      a.in_row = a.out_row = n;
      a.cols = a.qin = a.qout = static_cast<unsigned>(M);
      a.sj_in = M;
      a.transposing = 1;
      a.sj_out = 1;
      a.sw_out = L1;
      a.twiddle = 1;
      a.tw = tw;
      // pass 2: over n2 for the columns (n3, k1) -> Y2 [n3][k2][k1], times w_M^(n3 k2) = w_N^(L1 n3 k2)
      SlabPass& b = p_[1];
      b.in_row = b.out_row = n;
      b.cols = b.qin = static_cast<unsigned>(L3 * L1);
      b.sj_in = L3 * L1;
      b.qout = static_cast<unsigned>(L1);
      b.qo = L2 * L1;
      b.sj_out = L1;
      b.twiddle = 1;
      b.tdiv = static_cast<unsigned>(L1);
      b.tw = tw;
      b.tw.mul = L1;
      // pass 3: over n3 for the columns (k2, k1), in place -> X [k3][k2][k1]
      SlabPass& c = p_[2];
      c.in_row = c.out_row = n;
      c.cols = c.qin = c.qout = static_cast<unsigned>(L2 * L1);
      c.sj_in = c.sj_out = L2 * L1;
    }
    if (cudaMalloc(&scratch_, batch_ * n_ * sizeof(V2)) != cudaSuccess)
      throw std::runtime_error("cudaMalloc slab four-step scratch");
    launches = sh.passes;
  }
  ~SlabPlan() override {
    if (scratch_) cudaFree(scratch_);
  }
  void exec(const void* in, void* out, size_t rows, int inverse, cudaStream_t st) override {
    if (rows > batch_) throw std::invalid_argument("rows exceed the plan batch");
    const bool inv = inverse != 0;
    const R scale = R(1) / static_cast<R>(n_);
    const bool alias = in == out;
    if (sh_.passes == 2) {
      void* mid = alias ? static_cast<void*>(scratch_) : out;
      pass_[0]->run(in, mid, rows, p_[0], inv, false, R(1), st);
      pass_[1]->run(mid, out, rows, p_[1], false, inv, scale, st);
      return;
    }
    // three passes: in -> a -> b -> out with a != in, b != a; the last pass may run in place
    void* a = alias ? static_cast<void*>(scratch_) : out;
    void* b = alias ? out : static_cast<void*>(scratch_);
    pass_[0]->run(in, a, rows, p_[0], inv, false, R(1), st);
    pass_[1]->run(a, b, rows, p_[1], false, false, R(1), st);
    pass_[2]->run(b, out, rows, p_[2], false, inv, scale, st);
  }

 private:
  size_t n_, batch_;
  SlabShape sh_;
  Twiddles tws_;
  std::unique_ptr<slabk::SlabPassExec<R>> pass_[3];
  slabk::SlabPass p_[3];
  V2* scratch_ = nullptr;
};

void fourstep_prefer_transposable(bool on) { g_prefer_transposable = on; }

bool fourstep_covers(const amqft_plan_desc& d) {
  if (d.function != AMQFT_FN_CDFT || (d.order != AMQFT_ORDER_FAST && d.order != AMQFT_ORDER_FAST_DAG)) return false;
  if ((d.n & (d.n - 1)) != 0 || d.n > (size_t(1) << 26)) return false;
  // one fused / small / tile kernel does it (FAST_DAG plans: the whole-DAG kernels only)
  if (fast_sub_covered(d.dtype, d.n, d.variant, d.order != AMQFT_ORDER_FAST_DAG)) return false;
  return fourstep_slab_shape(d).passes > 0 || fourstep_shape(d.dtype, d.variant, d.n).ok;
}

OpCount fourstep_op_counts(const amqft_plan_desc& d) {
  // Two-factor: N2 sub-transforms of length N1, N1 of length N2 (the
  // reference DAG of each), plus one complex twiddle multiply per element
  // (4 muls + 2 adds).  Three-factor A x B x C: B C of length A, A C of
  // length B, A B of length C, and two twiddle passes.
  if (const SlabShape ss = fourstep_slab_shape(d); ss.passes) {
    // per pass N / L columns of the two-factor length-L schedule (tile_op_counts), one twiddle
    // multiply per element between passes
    OpCount c;
    for (int i = 0; i < ss.passes; ++i) {
      amqft_plan_desc t = d;
      t.n = ss.len[i];
      const OpCount f = tile_op_counts(t);
      const uint64_t cols = d.n / ss.len[i];
      c.adds += cols * f.adds;
      c.muls += cols * f.muls;
      c.bt += cols * f.bt;
    }
    c.adds += static_cast<uint64_t>(ss.passes - 1) * 2 * d.n;
    c.muls += static_cast<uint64_t>(ss.passes - 1) * 4 * d.n;
    return c;
  }
  const FourStepShape sh = fourstep_shape(d.dtype, d.variant, d.n);
  OpCount c;
  if (sh.three) {
    const size_t a = sh.n1, b = sh.nb, cc = sh.n2;
    const OpCount ca = fast_sub_op_counts(d.variant, a, d.dtype, true),
                  cb = fast_sub_op_counts(d.variant, b, d.dtype, true), ccc = fast_sub_op_counts(d.variant, cc, d.dtype);
    c.adds = b * cc * ca.adds + a * cc * cb.adds + a * b * ccc.adds + 2 * 2 * d.n;
    c.muls = b * cc * ca.muls + a * cc * cb.muls + a * b * ccc.muls + 2 * 4 * d.n;
    c.bt = b * cc * ca.bt + a * cc * cb.bt + a * b * ccc.bt;
    return c;
  }
  const size_t n1 = sh.n1, n2 = sh.n2;
  const OpCount c1 = fast_sub_op_counts(d.variant, n1, d.dtype, sh.col), c2 = fast_sub_op_counts(d.variant, n2, d.dtype);
  c.adds = n2 * c1.adds + n1 * c2.adds + 2 * d.n;
  c.muls = n2 * c1.muls + n1 * c2.muls + 4 * d.n;
  c.bt = n2 * c1.bt + n1 * c2.bt;
  return c;
}

amqft_status fourstep_factors(const amqft_plan_desc& d, size_t* f3) {
  if (const SlabShape ss = fourstep_slab_shape(d); ss.passes) {
    f3[0] = ss.len[0];
    f3[1] = ss.passes == 3 ? ss.len[1] : 1;
    f3[2] = ss.passes == 3 ? ss.len[2] : ss.len[1];
    return AMQFT_OK;
  }
  const FourStepShape sh = fourstep_shape(d.dtype, d.variant, d.n);
  if (!sh.ok) return AMQFT_EINVAL;
  f3[0] = sh.n1;
  f3[1] = sh.three ? sh.nb : 1;
  f3[2] = sh.n2;
  return AMQFT_OK;
}

std::unique_ptr<FastPlan> make_fourstep_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax,
                                             const void* d_trig64) {
  if (!fourstep_covers(d)) return nullptr;
  if (const SlabShape ss = fourstep_slab_shape(d); ss.passes) {
    if (d.dtype == AMQFT_F64)
      return std::make_unique<SlabPlan<double>>(d.variant, d.n, d.batch, d.trig_mode, d_trig, nmax, d.device, ss);
    return std::make_unique<SlabPlan<float>>(d.variant, d.n, d.batch, d.trig_mode, d_trig, nmax, d.device, ss);
  }
  if (d.dtype == AMQFT_F64)
    return std::make_unique<FourStepPlan<double>>(d.variant, d.n, d.batch, d.trig_mode, d_trig, nmax, d.device,
                                                   d_trig64);
  return std::make_unique<FourStepPlan<float>>(d.variant, d.n, d.batch, d.trig_mode, d_trig, nmax, d.device,
                                                d_trig64);
}

}  // namespace amqft_b200
