// inverse.cu -- inverses of the real transforms (the
// reference has no inverse at all), defined on top of the forward AM-QFT
// DCT-0 / DST-0 like the CDFT swap trick: only exact scalings by powers of
// two and one butterfly are added, so each inverse is bitwise defined by the
// forward transform of the same variant.
//
// With A the DCT-0 matrix cos(2 pi k m / N), k, m = 0..N/2 (no endpoint
// weights) and W = diag(1/2, 1, .., 1, 1/2): the weighted
// DCT-I T = A W satisfies T T = (N/4) I, so
//   DCT-0^-1(C) = (4/N) W A (W C)                       (two exact weightings)
// The DST-0 matrix B = sin(2 pi k m / N), k, m = 1..N/2-1, satisfies
// B B = (N/4) I:
//   DST-0^-1(S) = (4/N) B S
// RDFT (packed spectrum P, signal.hpp:122-124; SplitReal, elaborations.cpp:
// 185-208): C(k) = P[k] (k <= N/2), S(k) = P[N-k] are the DCT-0 / DST-0 of
// c(m) = x[m] + x[N-m] and s(m) = x[m] - x[N-m], so
//   x[0] = c(0), x[N/2] = c(N/2), x[m] = (c(m) + s(m)) / 2, x[N-m] = (c(m) - s(m)) / 2.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "generic.cuh"
#include "inverse.cuh"

namespace amqft_b200 {
namespace {

inline unsigned grid_for(size_t total) {
  return static_cast<unsigned>(std::min<size_t>((total + 255) / 256, size_t(148) * 32));
}

inline void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// out[r][i] = in[r][i] * (endpoint ? s_end : s_mid)   (DCT-0 rows; DST-0 rows: s_end = s_mid)
template <typename R>
__global__ void __launch_bounds__(256) k_weight(const R* __restrict__ in, R* __restrict__ out, size_t rows,
                                                uint32_t cells, R s_mid, R s_end) {
  using A = Arith<R>;
  const size_t total = rows * cells;
  for (size_t i = threadIdx.x + blockIdx.x * size_t(blockDim.x); i < total; i += size_t(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i % cells);
    out[i] = A::mul(in[i], (c == 0 || c == cells - 1) ? s_end : s_mid);
  }
}

// packed RDFT spectrum -> W C (N/2 + 1 cells) and S (N/2 - 1 cells)
template <typename R>
__global__ void __launch_bounds__(256) k_rdft_split(const R* __restrict__ in, R* __restrict__ cw, R* __restrict__ s,
                                                    size_t rows, uint32_t n) {
  using A = Arith<R>;
  const uint32_t h = n / 2;
  const size_t total = rows * n;
  for (size_t i = threadIdx.x + blockIdx.x * size_t(blockDim.x); i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t r = i / n;
    const uint32_t k = static_cast<uint32_t>(i - r * n);
    const R v = in[i];
    if (k <= h) cw[r * (h + 1) + k] = (k == 0 || k == h) ? A::mul(v, R(0.5)) : v;
    else s[r * (h - 1) + (n - k - 1)] = v;           // S(k') at k' = n - k, cell k' - 1
  }
}

// c = (4/N) W DCT(W C), s = (4/N) DST(S) -> x
template <typename R>
__global__ void __launch_bounds__(256) k_rdft_combine(const R* __restrict__ cc, const R* __restrict__ ss,
                                                      R* __restrict__ out, size_t rows, uint32_t n, R sc) {
  using A = Arith<R>;
  const uint32_t h = n / 2;
  const size_t total = rows * (h + 1);
  for (size_t i = threadIdx.x + blockIdx.x * size_t(blockDim.x); i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t r = i / (h + 1);
    const uint32_t m = static_cast<uint32_t>(i - r * (h + 1));
    R* x = out + r * n;
    if (m == 0 || m == h) {
      x[m] = A::mul(A::mul(cc[i], sc), R(0.5));
      continue;
    }
    const R c = A::mul(cc[i], sc), s = A::mul(ss[r * (h - 1) + m - 1], sc);
    x[m] = A::mul(A::add(c, s), R(0.5));
    x[n - m] = A::mul(A::sub(c, s), R(0.5));
  }
}

template <typename R>
void weight_t(const void* in, void* out, size_t rows, size_t cells, double s_mid, double s_end, cudaStream_t st) {
  const size_t total = rows * cells;
  if (!total) return;
  k_weight<R><<<grid_for(total), 256, 0, st>>>(static_cast<const R*>(in), static_cast<R*>(out), rows,
                                                static_cast<uint32_t>(cells), static_cast<R>(s_mid),
                                                static_cast<R>(s_end));
  check_launch("k_weight");
}

}  // namespace

void inv_weight(int dtype_f64, const void* in, void* out, size_t rows, size_t cells, double s_mid, double s_end,
                cudaStream_t st) {
  if (dtype_f64) weight_t<double>(in, out, rows, cells, s_mid, s_end, st);
  else weight_t<float>(in, out, rows, cells, s_mid, s_end, st);
}

void inv_rdft_split(int dtype_f64, const void* in, void* cw, void* s, size_t rows, size_t n, cudaStream_t st) {
  const size_t total = rows * n;
  if (dtype_f64)
    k_rdft_split<double><<<grid_for(total), 256, 0, st>>>(static_cast<const double*>(in), static_cast<double*>(cw),
                                                           static_cast<double*>(s), rows, static_cast<uint32_t>(n));
  else
    k_rdft_split<float><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(in), static_cast<float*>(cw),
                                                          static_cast<float*>(s), rows, static_cast<uint32_t>(n));
  check_launch("k_rdft_split");
}

void inv_rdft_combine(int dtype_f64, const void* cc, const void* ss, void* out, size_t rows, size_t n, double sc,
                      cudaStream_t st) {
  const size_t total = rows * (n / 2 + 1);
  if (dtype_f64)
    k_rdft_combine<double><<<grid_for(total), 256, 0, st>>>(static_cast<const double*>(cc),
                                                             static_cast<const double*>(ss),
                                                             static_cast<double*>(out), rows,
                                                             static_cast<uint32_t>(n), sc);
  else
    k_rdft_combine<float><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(cc),
                                                            static_cast<const float*>(ss), static_cast<float*>(out),
                                                            rows, static_cast<uint32_t>(n),
                                                            static_cast<float>(sc));
  check_launch("k_rdft_combine");
}

// fp32 rows <-> fp64 working rows of a plan that computes in fp64
// (fast.cuh f32_needs_f64_compute): widening is exact, narrowing rounds once.
template <typename S, typename D>
__global__ void __launch_bounds__(256) k_convert(const S* __restrict__ in, D* __restrict__ out, size_t total) {
  for (size_t i = threadIdx.x + blockIdx.x * size_t(blockDim.x); i < total; i += size_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<D>(in[i]);
}

void convert_rows(int to_f64, const void* in, void* out, size_t total, cudaStream_t st) {
  if (to_f64)
    k_convert<float, double><<<grid_for(total), 256, 0, st>>>(static_cast<const float*>(in),
                                                               static_cast<double*>(out), total);
  else
    k_convert<double, float><<<grid_for(total), 256, 0, st>>>(static_cast<const double*>(in),
                                                               static_cast<float*>(out), total);
  check_launch("k_convert");
}

}  // namespace amqft_b200
