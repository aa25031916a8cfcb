// Microbenchmark (diagnostic): issue / pipe throughput of FADD vs FADD2
// (packed fp32 on sm_100a) with 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* o, int it) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
  const float b = 1.0001f;
  for (int i = 0; i < it; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] * b + 0.5f;   // FFMA
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* o, int it) {
  unsigned long long a[8];
  for (int j = 0; j < 8; ++j) {
    float2 v = make_float2(threadIdx.x * 0.001f + j, j * 0.5f);
    a[j] = *reinterpret_cast<unsigned long long*>(&v);
  }
  float2 bb = make_float2(1.0001f, 1.0002f), cc = make_float2(0.5f, 0.25f);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bb), c = *reinterpret_cast<unsigned long long*>(&cc);
  for (int i = 0; i < it; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(b), "l"(c));
  float s = 0;
  for (int j = 0; j < 8; ++j) { float2 v = *reinterpret_cast<float2*>(&a[j]); s += v.x + v.y; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int it = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k1<<<148 * 8, 256>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms1; cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0); k2<<<148 * 8, 256>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    double f1 = 148.0 * 8 * 256 * it * 8 * 2, f2 = f1 * 2;
    printf("FFMA : %.3f ms  %.1f TFLOP/s   FFMA2: %.3f ms  %.1f TFLOP/s\n", ms1, f1 / ms1 / 1e9, ms2, f2 / ms2 / 1e9);
  }
  return 0;
}
