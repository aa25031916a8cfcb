// verify.cu -- direct evaluation of selected DFT bins on the device.
//
// The verification utility behind the CLI's verify / accuracy commands
// (cli.cpp) and the large-N spot checks (bench.py config 5, tests).  It is
// not a transform path: O(N) work per bin, X[k] = sum_n x[n] w_N^((n k) mod N)
// with the phase reduced exactly in integers before any rounding (the
// reference's naive-DFT discipline, src/oracle.cpp:30-35).
//
//   amqft_direct_bins           fp64: twiddles by sincospi of the reduced
//                               phase, fp64 sums; any N (config 5: 2^30),
//                               any strided / slab layout of the samples.
//   amqft_direct_bins_extended  the extended-precision reference the CLI
//                               grades against (src/oracle.cpp:155-158:
//                               long double twiddle table, compensated
//                               long double sums): the same long double
//                               twiddles, carried exactly as double-double,
//                               products and sums in double-double.
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amqft_b200.h"

namespace amqft_b200 {
void set_last_error(const std::string& m);
}

namespace {

using amqft_b200::set_last_error;

struct DD {
  double hi, lo;
};

__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return DD{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ DD quick_two_sum(double a, double b) {
  const double s = a + b;
  return DD{s, b - (s - a)};
}
// accurate double-double addition
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
// double x double-double
__device__ __forceinline__ DD dd_mul(double a, DD b) {
  const double p = a * b.hi;
  double e = fma(a, b.hi, -p);
  e = fma(a, b.lo, e);
  return quick_two_sum(p, e);
}
__device__ __forceinline__ DD dd_neg(DD a) { return DD{-a.hi, -a.lo}; }

// One thread per bin; the samples stream through shared memory in tiles.
// tab[4 r] = {cos hi, cos lo, sin hi, sin lo} of 2 pi r / n.
template <typename T>
__global__ void k_bins_dd(const T* __restrict__ x, size_t n, const unsigned long long* __restrict__ bins,
                          size_t nb, const double* __restrict__ tab, int reverse, double* __restrict__ out) {
  constexpr int TILE = 512;
  __shared__ double2 xs[TILE];
  const size_t b = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const bool live = b < nb;
  const unsigned long long k = live ? bins[b] % n : 0;
  DD re{0.0, 0.0}, im{0.0, 0.0};
  // phase of the first sample in walking order, then +-k per step (mod n)
  unsigned long long r = reverse ? ((n - 1) % n) * k % n : 0;
  const unsigned long long step = reverse ? (n - k) % n : k;
  for (size_t t0 = 0; t0 < n; t0 += TILE) {
    __syncthreads();
    for (int i = threadIdx.x; i < TILE && t0 + i < n; i += blockDim.x) {
      const size_t m = reverse ? n - 1 - (t0 + i) : t0 + i;
      xs[i] = make_double2(static_cast<double>(x[2 * m]), static_cast<double>(x[2 * m + 1]));
    }
    __syncthreads();
    const int cnt = static_cast<int>(n - t0 < TILE ? n - t0 : TILE);
    if (live)
      for (int i = 0; i < cnt; ++i) {
        const double2 v = xs[i];
        const double2 c = *reinterpret_cast<const double2*>(tab + 4 * r);
        const double2 s = *reinterpret_cast<const double2*>(tab + 4 * r + 2);
        const DD C{c.x, c.y}, S{s.x, s.y};
        // (xr + i xi)(cos - i sin)
        re = dd_add(re, dd_mul(v.x, C));
        re = dd_add(re, dd_mul(v.y, S));
        im = dd_add(im, dd_mul(v.y, C));
        im = dd_add(im, dd_neg(dd_mul(v.x, S)));
        r += step;
        if (r >= n) r -= n;
      }
  }
  if (live) {
    out[4 * b + 0] = re.hi;
    out[4 * b + 1] = re.lo;
    out[4 * b + 2] = im.hi;
    out[4 * b + 3] = im.lo;
  }
}

// fp64 mode.  Sample e of the buffer (row e / row_len, column e % row_len)
// is x[m], m = row0 + row + stride * column (a plain signal: row0 = 0,
// rows = 1, stride = 1; config 5's column slab: row0 = first column,
// stride = n2).  Up to KB bins per pass; block partials are combined with
// fp64 atomics.
constexpr int KB = 8;
template <typename T>
__global__ void k_bins_f64(const T* __restrict__ x, size_t total, size_t row_len, size_t row0, size_t stride,
                           size_t n, const unsigned long long* __restrict__ bins, int nb, double* __restrict__ acc) {
  double sr[KB], si[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) sr[j] = si[j] = 0.0;
  unsigned long long kk[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) kk[j] = j < nb ? bins[j] % n : 0;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t row = e / row_len, col = e - row * row_len;
    const unsigned long long m = (row0 + row + stride * col) % n;
    const double xr = static_cast<double>(x[2 * e]), xi = static_cast<double>(x[2 * e + 1]);
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j >= nb) break;
      // exact reduction: m, k < n <= 2^32 -> m k < 2^64
      const unsigned long long ph = (m * kk[j]) % n;
      double s, c;
      sincospi(2.0 * static_cast<double>(ph) / static_cast<double>(n), &s, &c);
      sr[j] = fma(xr, c, fma(xi, s, sr[j]));
      si[j] = fma(xi, c, fma(-xr, s, si[j]));
    }
  }
  __shared__ double red[32][2 * KB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    for (int o = 16; o; o >>= 1) {
      sr[j] += __shfl_down_sync(0xffffffffu, sr[j], o);
      si[j] += __shfl_down_sync(0xffffffffu, si[j], o);
    }
    if (lane == 0) {
      red[warp][2 * j] = sr[j];
      red[warp][2 * j + 1] = si[j];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * nb) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    atomicAdd(acc + threadIdx.x, s);
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Long double twiddles of the reference's angle table (src/oracle.cpp:17-27),
// carried exactly as double-double.  Cached per n (tables are immutable).
const double* dd_table(size_t n) {
  static std::mutex mu;
  static std::vector<std::pair<size_t, double*>> cache;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t key = n * 64 + static_cast<size_t>(dev);
  for (auto& e : cache)
    if (e.first == key) return e.second;
  std::vector<double> t(4 * n);
  const long double step = 2.0L * 3.141592653589793238462643383279502884L / static_cast<long double>(n);
  for (size_t m = 0; m < n; ++m) {
    const long double a = step * static_cast<long double>(m);
    const long double c = cosl(a), s = sinl(a);
    t[4 * m] = static_cast<double>(c);
    t[4 * m + 1] = static_cast<double>(c - static_cast<long double>(t[4 * m]));
    t[4 * m + 2] = static_cast<double>(s);
    t[4 * m + 3] = static_cast<double>(s - static_cast<long double>(t[4 * m + 2]));
  }
  double* d = nullptr;
  ck(cudaMalloc(&d, t.size() * sizeof(double)), "cudaMalloc twiddle table");
  ck(cudaMemcpy(d, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
  cache.emplace_back(key, d);
  return d;
}

amqft_status fail(amqft_status s, const std::string& m) {
  set_last_error(m);
  return s;
}

}  // namespace

extern "C" {

amqft_status amqft_direct_bins(const void* d_x, int dtype, size_t rows, size_t row_len, size_t row0, size_t stride,
                               size_t n, const uint64_t* bins, size_t nbins, double* out, void* stream) {
  if (!d_x || !bins || !out || n == 0 || rows == 0 || row_len == 0)
    return fail(AMQFT_EINVAL, "direct bins: null buffer or empty shape");
  if (dtype != AMQFT_F32 && dtype != AMQFT_F64) return fail(AMQFT_EINVAL, "direct bins: dtype must be F32 or F64");
  if (n > (size_t(1) << 32)) return fail(AMQFT_EINVAL, "direct bins: n above 2^32");
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long* dbins = nullptr;
    double* dacc = nullptr;
    ck(cudaMalloc(&dbins, nbins * sizeof(unsigned long long)), "cudaMalloc");
    ck(cudaMalloc(&dacc, 2 * nbins * sizeof(double)), "cudaMalloc");
    ck(cudaMemcpyAsync(dbins, bins, nbins * sizeof(unsigned long long), cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaMemsetAsync(dacc, 0, 2 * nbins * sizeof(double), st), "memset");
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t total = rows * row_len;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, static_cast<size_t>(sms) * 8));
    for (size_t b0 = 0; b0 < nbins; b0 += KB) {
      const int nb = static_cast<int>(std::min<size_t>(KB, nbins - b0));
      if (dtype == AMQFT_F32)
        k_bins_f64<float><<<grid, 256, 0, st>>>(static_cast<const float*>(d_x), total, row_len, row0, stride, n,
                                                 dbins + b0, nb, dacc + 2 * b0);
      else
        k_bins_f64<double><<<grid, 256, 0, st>>>(static_cast<const double*>(d_x), total, row_len, row0, stride, n,
                                                  dbins + b0, nb, dacc + 2 * b0);
      ck(cudaGetLastError(), "k_bins_f64 launch");
    }
    ck(cudaMemcpyAsync(out, dacc, 2 * nbins * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    cudaFree(dbins);
    cudaFree(dacc);
    return AMQFT_OK;
  } catch (const std::exception& e) {
    return fail(AMQFT_ECUDA, e.what());
  }
}

amqft_status amqft_direct_bins_extended(const double* x, size_t n, const uint64_t* bins, size_t nbins, int reverse,
                                        double* out) {
  if (!x || !bins || !out || n == 0) return fail(AMQFT_EINVAL, "direct bins: null buffer or n = 0");
  if (n > (size_t(1) << 22)) return fail(AMQFT_EINVAL, "extended direct bins: n above 2^22 (O(n) table)");
  try {
    const double* tab = dd_table(n);
    double *dx = nullptr, *dout = nullptr;
    unsigned long long* dbins = nullptr;
    ck(cudaMalloc(&dx, 2 * n * sizeof(double)), "cudaMalloc");
    ck(cudaMalloc(&dbins, nbins * sizeof(unsigned long long)), "cudaMalloc");
    ck(cudaMalloc(&dout, 4 * nbins * sizeof(double)), "cudaMalloc");
    ck(cudaMemcpy(dx, x, 2 * n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(dbins, bins, nbins * sizeof(unsigned long long), cudaMemcpyHostToDevice), "H2D");
    const unsigned grid = static_cast<unsigned>((nbins + 255) / 256);
    k_bins_dd<double><<<grid, 256>>>(dx, n, dbins, nbins, tab, reverse, dout);
    ck(cudaGetLastError(), "k_bins_dd launch");
    ck(cudaMemcpy(out, dout, 4 * nbins * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    cudaFree(dx);
    cudaFree(dbins);
    cudaFree(dout);
    return AMQFT_OK;
  } catch (const std::exception& e) {
    return fail(AMQFT_ECUDA, e.what());
  }
}

}  // extern "C"
