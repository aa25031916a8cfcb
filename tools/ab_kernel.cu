// ab_kernel.cu -- DIAGNOSTIC: the fused kernel built with alternative
// compile-time options (-D...), timed with CUDA events on its own stream.
// Not part of the product library.  tools/ab_kernel.py drives it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -shared -Xcompiler -fPIC -DAMQFT_TMA_STORE=0 -o tools/ab_X.so tools/ab_kernel.cu
#include <cstdio>
#include "../paper_1404_1810_b200/csrc/fast_kernel.cuh"

using namespace amqft_b200::fastk;

template <int V>
static float run_v(const float* in, float* out, size_t rows, const float* tab, int nmax, int reps) {
  using C = Cfg<V, float, 12, 6>;
  auto fn = k_fast<V, float, 12, 6, false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BLOCK);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::NTB, C::SMEM_BLOCK);
  const size_t units = (rows + C::RPC - 1) / C::RPC;
  const unsigned grid = (unsigned)std::min<size_t>(units, 148 * (size_t)(per_sm > 0 ? per_sm : 1));
  float* ltab = nullptr;
  cudaMalloc(&ltab, sizeof(float) * C::H);
  k_level_table<float><<<8, 256>>>(tab, ltab, C::H, C::LT, nmax);
  TabParam<float, C::N / 4> tp;
  cudaMemcpy(tp.v, tab, sizeof(tp.v), cudaMemcpyDeviceToHost);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    fn<<<grid, C::NTB, C::SMEM_BLOCK>>>(in, out, rows, tp, ltab, nmax, 1.0f / 4096);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  cudaFree(ltab);
  return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}

extern "C" float ab_run(int v, const float* in, float* out, size_t rows, const float* tab, int nmax,
                        int reps) {
  switch (v) {
    case 1: return run_v<1>(in, out, rows, tab, nmax, reps);
    case 2: return run_v<2>(in, out, rows, tab, nmax, reps);
    case 3: return run_v<3>(in, out, rows, tab, nmax, reps);
    case 4: return run_v<4>(in, out, rows, tab, nmax, reps);
    case 5: return run_v<5>(in, out, rows, tab, nmax, reps);
    case 6: return run_v<6>(in, out, rows, tab, nmax, reps);
    case 7: return run_v<7>(in, out, rows, tab, nmax, reps);
    case 8: return run_v<8>(in, out, rows, tab, nmax, reps);
  }
  return -1.0f;
}
