// inverse.cuh -- element-wise kernels of the RDFT / DCT-0 / DST-0 inverses
// (inverse.cu); the transforms themselves are the plans' forward paths.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace amqft_b200 {
void inv_weight(int dtype_f64, const void* in, void* out, size_t rows, size_t cells, double s_mid, double s_end,
                cudaStream_t st);
void inv_rdft_split(int dtype_f64, const void* in, void* cw, void* s, size_t rows, size_t n, cudaStream_t st);
void inv_rdft_combine(int dtype_f64, const void* cc, const void* ss, void* out, size_t rows, size_t n, double sc,
                      cudaStream_t st);
// fp32 <-> fp64 rows (total elements): to_f64 = 1 widens, 0 narrows.
void convert_rows(int to_f64, const void* in, void* out, size_t total, cudaStream_t st);
}  // namespace amqft_b200
