// phase_timing.cu -- DIAGNOSTIC build of the fused kernel with per-phase
// clock64() accounting (CTA 0).  Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -shared -Xcompiler -fPIC \
//        -o tools/libphase_timing.so tools/phase_timing.cu
#define AMQFT_PHASE_TIMING
#include <cstdio>
#ifndef AMQFT_FAST_MINB
#define AMQFT_FAST_MINB 2
#endif
#include "../paper_1404_1810_b200/csrc/fast_kernel.cuh"

using namespace amqft_b200::fastk;

template <int V, int LOGN>
static int run_v(const float* in, float* out, size_t rows, const float* tab, int nmax,
                 unsigned long long* cyc, int grid) {
  using C = Cfg<V, float, LOGN, 6>;
  auto fn = k_fast<V, float, LOGN, 6, false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BLOCK);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::NTB, C::SMEM_BLOCK);
  if (grid <= 0) grid = 148 * (per_sm > 0 ? per_sm : 1);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  unsigned long long zz[16][16] = {{0}};
  cudaMemcpyToSymbol(g_warp_work, zz, sizeof(zz));
  float* ltab = nullptr;
  cudaMalloc(&ltab, sizeof(float) * C::H);
  k_level_table<float><<<8, 256>>>(tab, ltab, C::H, C::LT, nmax);
  TabParam<float, C::N / 4> tp;
  cudaMemcpy(tp.v, tab, sizeof(tp.v), cudaMemcpyDeviceToHost);
  fn<<<grid, C::NTB, C::SMEM_BLOCK>>>(in, out, rows, tp, ltab, nmax, 1.0f / C::N);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(cyc, g_phase_cycles, sizeof(z));
  cudaFree(ltab);
  unsigned long long ww[16][16];
  cudaMemcpyFromSymbol(ww, g_warp_work, sizeof(ww));
  for (int p = 0; p < 6; ++p) {
    printf("  phase %d warp work:", p);
    for (int w = 0; w < C::NTB / 32; ++w) printf(" %6llu", ww[p][w] / (rows / (grid * C::RPC)));
    printf("\n");
  }
  printf("  (grid %d, %d rows per CTA iteration)\n", grid, C::RPC);
  cyc[15] = (unsigned long long)grid * C::RPC;
  return (int)cudaGetLastError();
}

extern "C" int pt_run(int v, const float* in, float* out, size_t rows, const float* tab,
                      int nmax, unsigned long long* cyc, int grid) {
  // nmax is the transform size (table built for Nmax = N)
  switch (v * 100 + nmax / 1024) {
    case 101: return run_v<1, 10>(in, out, rows, tab, nmax, cyc, grid);
    case 104: return run_v<1, 12>(in, out, rows, tab, nmax, cyc, grid);
    case 201: return run_v<2, 10>(in, out, rows, tab, nmax, cyc, grid);
    case 202: return run_v<2, 11>(in, out, rows, tab, nmax, cyc, grid);
    case 204: return run_v<2, 12>(in, out, rows, tab, nmax, cyc, grid);
    case 401: return run_v<4, 10>(in, out, rows, tab, nmax, cyc, grid);
    case 402: return run_v<4, 11>(in, out, rows, tab, nmax, cyc, grid);
    case 404: return run_v<4, 12>(in, out, rows, tab, nmax, cyc, grid);
    case 408: return run_v<4, 13>(in, out, rows, tab, nmax, cyc, grid);
  }
  return -1;
}
