/*
 * amqft_b200.h -- C ABI of the B200 AM-QFT library (libamqft_b200.so).
 *
 * Drop-in boundary for the reference's transform entry point
 *   SignalBuffer amqft::execute(VariantId, FunctionId, const SignalBuffer&,
 *                               const TrigSource&, OpMeter*)
 *   (/root/reference/proj/include/amqft/variants.hpp:148-153,
 *    src/variants.cpp:404-442)
 * and its constant-table plugin
 *   TrigTable(VariantId, max_periodization, TrigMode)
 *   (include/amqft/variants.hpp:111-141, src/variants.cpp:248-299).
 * The C++ header amqft_b200.hpp keeps the reference names on top of this.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are caller-owned and
 *    must stay valid until the stream work completes.  `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Cell layout per transform is the reference SignalBuffer layout
 *    (include/amqft/signal.hpp:110-146): CDFT = 2N interleaved re/im reals,
 *    RDFT = N reals (packed spectrum Re S(j), j <= N/2, then Im S(j)),
 *    DCT = N/2+1, DST = N/2-1, restricted types per their stored ranges.
 *    Batches are row-major: row r starts at r * cells.
 *  - Transforms are unnormalised forward sums with kernel e^{-2 pi i nk/N}
 *    (src/oracle.cpp:69-84).  amqft_exec_inverse is builder-defined (the
 *    reference has none): CDFT x = swap(DFT(swap(X))) / N; DCT-0
 *    x = (4/N) W DCT(W C), W = diag(1/2, 1, .., 1, 1/2); DST-0
 *    x = (4/N) DST(S); RDFT through those two on the split packed spectrum
 *    (csrc/inverse.cu).  Only exact power-of-two scalings and one butterfly
 *    are added to the forward transforms.
 *  - Errors mirror the reference's std::invalid_argument cases
 *    (variants.cpp:404-421, signal.cpp:138-147) as AMQFT_EINVAL;
 *    amqft_last_error() returns the message (thread-local).
 *  - There is no CPU fallback: without a usable CUDA device every exec
 *    call returns AMQFT_ECUDA.
 */
#ifndef AMQFT_B200_H
#define AMQFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AMQFT_OK = 0,
  AMQFT_EINVAL = 1, /* reference: std::invalid_argument */
  AMQFT_ECUDA = 2,
  AMQFT_ENCCL = 3,
  AMQFT_ENOMEM = 4
} amqft_status;

/* FunctionId, same order as include/amqft/variants.hpp:55-66. */
typedef enum {
  AMQFT_FN_CDFT = 0,
  AMQFT_FN_RDFT = 1,
  AMQFT_FN_DCT = 2,
  AMQFT_FN_DST = 3,
  AMQFT_FN_DCT_ODD_TIME = 4,
  AMQFT_FN_DST_ODD_TIME = 5,
  AMQFT_FN_DCT_ODD_HARM = 6,
  AMQFT_FN_DST_ODD_HARM = 7,
  AMQFT_FN_DCT_ODD_ODD = 8,
  AMQFT_FN_DST_ODD_ODD = 9
} amqft_function;

typedef enum { AMQFT_F32 = 0, AMQFT_F64 = 1 } amqft_dtype;

/* TrigMode (variants.hpp:108): TABLE = Precomputed (host long-double
 * constants, bitwise the reference's); ONTHEFLY = computed on the device
 * with sincospi in the plan's dtype (close to, not bitwise, the table). */
typedef enum { AMQFT_TRIG_TABLE = 0, AMQFT_TRIG_ONTHEFLY = 1 } amqft_trig_mode;

/* Execution order.  EXACT: every node's operations in the reference's
 * operand order and association, no FMA contraction, serial M1/M3/M5/M7
 * recurrences -> bitwise equal to amqft::execute in F64.  FAST: the fastest
 * kernels that keep the result within the tolerance against the CPU
 * reference of the same variant (1e-5 log2 n in F32, 1e-12 in F64): CDFT
 * rows of n = 16 .. 65536 (F64: 64 .. 32768 for variants 1-4, 64 .. 256 for
 * 5-8) run as two or three register-resident AM-QFT factors of <= 64 points
 * in one pass over HBM (the four-step inside shared memory: the AM-QFT DAG is
 * kept inside each factor), larger n as a multi-pass four-step; everything
 * else on the specialised whole-DAG kernels.  FAST_DAG: FAST without the
 * split inside shared memory -- the fused / cooperative / one-thread-per-row
 * kernels run the whole length-n reference DAG (recurrences may be evaluated
 * as parallel scans in F32; the F64 instances are bitwise amqft::execute up
 * to n = 4096), the multi-pass four-step above them. */
typedef enum { AMQFT_ORDER_EXACT = 0, AMQFT_ORDER_FAST = 1, AMQFT_ORDER_FAST_DAG = 2 } amqft_order;

typedef struct amqft_plan_s* amqft_plan;

typedef struct {
  int variant;          /* 1..8 (VariantId) */
  int function;         /* amqft_function */
  size_t n;             /* periodization, power of two >= the function base */
  size_t batch;         /* rows per exec call */
  int dtype;            /* amqft_dtype */
  int trig_mode;        /* amqft_trig_mode */
  int order;            /* amqft_order */
  int device;           /* CUDA device ordinal */
  size_t table_max_n;   /* TrigTable max periodization; 0 = max(n, 8) */
  int corrupt_constants;/* TrigTable::corrupt_for_testing (variants.cpp:301) */
} amqft_plan_desc;

/* Plan lifecycle.  Creation compiles the schedule, uploads it and the
 * constant table, and allocates every workspace the device entry points
 * use (four-step scratch, the real inverses' scratch and sub-plans, fp64
 * working rows): amqft_exec_forward / _inverse / _rows allocate nothing and
 * are stream-ordered (CUDA-graph capturable).  amqft_exec_host_rows creates
 * its pipeline slots and streams on its first call (serialised per plan).
 *
 * fp32 plans of variants 5-8 at n >= 512 that keep the whole DAG (EXACT and
 * FAST_DAG orders, RDFT / DCT / DST rows) compute in fp64 (their fp32
 * recursion amplifies rounding beyond 1e-5 log2 n): fp32 rows in and out,
 * the reference's fp64 DAG inside.  FAST CDFT plans split n into factors of
 * <= 64 points, which are stable in fp32 for every variant. */
amqft_status amqft_plan_create(amqft_plan* out, const amqft_plan_desc* desc);
amqft_status amqft_plan_destroy(amqft_plan plan);

/* Plan creation with caller-supplied constants (the TrigSource plugin,
 * elaborations.hpp:90-98): `constants` in the TrigTable::constants layout
 * (variants.cpp:289-299) for Nmax = desc->table_max_n (0: max(n, 8)): the
 * slots f(2 pi p / Nmax), p = 1 .. Nmax/4 - 1, then the base constant;
 * count must be Nmax / 4.  desc->corrupt_constants is ignored (the values
 * are taken as given). */
amqft_status amqft_plan_create_with_constants(amqft_plan* out, const amqft_plan_desc* desc,
                                              const double* constants, size_t count);

/* Cells per row of the plan's operand (cell_count, signal.cpp:254-258). */
size_t amqft_plan_cells(amqft_plan plan);

/* Forward transform of `plan->batch` rows: d_in -> d_out (may alias).
 * Fast-order plans (fused, four-step and small-CDFT kernels) need 16-byte
 * aligned device buffers (TMA bulk copies, 16-byte vectors): AMQFT_EINVAL
 * otherwise.  Exact-order plans take any alignment of the dtype. */
amqft_status amqft_exec_forward(amqft_plan plan, const void* d_in, void* d_out,
                                void* stream);

/* Inverse of `batch` rows: CDFT (swap trick), RDFT / DCT / DST (n >= 4);
 * AMQFT_EINVAL for the odd-function plans. */
amqft_status amqft_exec_inverse(amqft_plan plan, const void* d_in, void* d_out,
                                void* stream);

/* Forward / inverse with an explicit row count <= plan batch. */
amqft_status amqft_exec_rows(amqft_plan plan, const void* d_in, void* d_out,
                             size_t rows, int inverse, void* stream);

/* Forward / inverse of `rows` rows between HOST buffers (any row count; the
 * batch streams through three device slots as an H2D | transform | D2H
 * pipeline on the plan's own streams).  Stream-ordered: `stream` waits for
 * the last download.  Pass pinned host memory for asynchronous copies.
 * Replaces the reference's per-signal loop over execute (accuracy.cpp:67-74,
 * cli.cpp:155-174) for host-resident batches. */
amqft_status amqft_exec_host_rows(amqft_plan plan, const void* h_in, void* h_out,
                                  size_t rows, int inverse, void* stream);

/* Convenience mirror of amqft::execute: one signal, HOST buffers (upload,
 * run on the device, download, synchronise).  meter3 (nullable) receives
 * {adds, muls, binary translations} of the executed schedule. */
amqft_status amqft_execute_host(int variant, int function, size_t n,
                                const double* in, double* out, int trig_mode,
                                size_t table_max_n, int corrupt_constants,
                                uint64_t* meter3);

/* amqft::execute(v, f, input, trig, meter) for an arbitrary TrigSource:
 * as amqft_execute_host with the constants given in the TrigTable layout at
 * Nmax = 4 * count (amqft_plan_create_with_constants).  The C++ execute
 * (include/amqft_b200.hpp) collects them from the caller's TrigSource. */
amqft_status amqft_execute_host_constants(int variant, int function, size_t n, const double* in,
                                          double* out, const double* constants, size_t count,
                                          uint64_t* meter3);

/* Inverse CDFT of one host spectrum (swap trick, exact fp64 order). */
amqft_status amqft_execute_host_inverse(int variant, size_t n, const double* in, double* out);

/* ---- Distributed four-step (BASELINE config 5), fp32
 * complex.  One transform of length n = n1 * n2 over nparts ranks: rank p
 * holds rows n2 in [p n2/P, (p+1) n2/P) of length n1 (x[n2_total * n1_idx +
 * n2] gathered by column), transforms them (a length-n1 plan), then
 * amqft_dist_twiddle_scatter multiplies by w_n^(n2 k1) and scatters the
 * k1-slab of destination q to d_dst[q] at offset src_rank * rows * n1/P
 * ([row][k1 - q n1/P]).  d_dst (a HOST array of nparts device pointers) is
 * either the local send buffer's slots (followed by an all-to-all, e.g.
 * NCCL) or the peers' receive buffers mapped over NVLink (no collective:
 * the kernel's stores are the exchange).  After the exchange each rank
 * transposes [n2][n1/P] -> [n1/P][n2] (amqft_transpose_c64) and runs a
 * length-n2 plan; its output is X[k1 + n1 k2] for its k1-slab.  Replaces
 * nothing in the reference (single-process only, variants.cpp:404). */
amqft_status amqft_dist_twiddle_scatter(const void* d_rows, void* const* d_dst, size_t rows,
                                        size_t n1, size_t n, size_t row0, int src_rank,
                                        int nparts, int trig_mode, void* stream);

/* Distributed four-step with the local four-step's final transpose folded
 * into the scatter (config 5): for a column-mode four-step plan (path 3),
 * amqft_plan_transposed_factor gives its column factor A (0 otherwise) and
 * amqft_exec_rows_transposed leaves each row as out[r][ka][kb] = X[ka + A kb];
 * amqft_dist_twiddle_scatter_t is amqft_dist_twiddle_scatter for rows in
 * that order (A and n1/A multiples of 32, n1/nparts a multiple of 32).
 * Replaces nothing in the reference (it has no distributed path). */
/* The scatter and the exchange-side transpose in one kernel: element
 * (n2, k1) of the local rows goes straight to its place in the destination
 * rank's [n1 / nparts][n / n1] rows -- d_dst[q] is rank q's row buffer, mapped
 * into this process (CUDA IPC / a registered window), or the rank's own with
 * one part -- times w_N^(n2 k1); the length-n2 plan then runs on those rows
 * with no transpose in between.  a: the local plan's transposed factor (rows
 * in amqft_exec_rows_transposed order), or 0 for plain rows; rows and
 * n1 / max(a, 1) multiples of 32.  Config 5 on one B200: one pass less. */
amqft_status amqft_dist_twiddle_scatter_direct(const void* d_rows, void* const* d_dst, size_t rows, size_t n1,
                                               size_t n, size_t row0, int nparts, int trig_mode, size_t a,
                                               void* stream);
amqft_status amqft_plan_transposed_factor(amqft_plan plan, size_t* a);
/* amqft_plan_create for a caller that will use amqft_exec_rows_transposed:
 * among the four-step plans it prefers the column-mode one that has a
 * transposed output (the column-slab plans, measured a little faster as
 * stand-alone transforms at some sizes, have none).  The distributed
 * four-step creates its local length-n1 plan with it (config 5 on one B200:
 * 15.7 ms against 16.1 ms with a slab plan and the plain scatter). */
amqft_status amqft_plan_create_transposable(amqft_plan* out, const amqft_plan_desc* desc);
amqft_status amqft_exec_rows_transposed(amqft_plan plan, const void* d_in, void* d_out, size_t rows,
                                        void* stream);
amqft_status amqft_dist_twiddle_scatter_t(const void* d_rows, void* const* d_dst, size_t rows, size_t n1,
                                          size_t n, size_t row0, int src_rank, int nparts, int trig_mode,
                                          size_t a, void* stream);

/* ---- Verification (not a transform path): direct O(N)-per-bin DFT bins
 * X[k] = sum_n x[n] w_N^((n k) mod N), the phase reduced exactly in
 * integers first (the reference naive DFT's discipline, src/oracle.cpp:30-35).
 *
 * amqft_direct_bins: fp64 twiddles (sincospi of the reduced phase) and fp64
 * sums, for spot checks of huge transforms (config 5, N = 2^30).  d_x is a
 * device buffer of rows x row_len interleaved complex samples (dtype F32 or
 * F64); sample (r, c) is x[(row0 + r + stride c) mod n] (a plain signal:
 * rows = 1, row0 = 0, stride = 1).  bins: host array; out: host, {re, im}
 * per bin.  Synchronises `stream`.
 *
 * amqft_direct_bins_extended: the extended-precision reference
 * (src/oracle.cpp:155-158 computes it with long double twiddles and
 * compensated long double sums): the same long double twiddles carried
 * exactly as double-double, double-double products and sums.  x: host,
 * n interleaved fp64 complex samples (n <= 2^22); reverse = 1 sums in
 * descending n (the reference's self-gauge, oracle.cpp:160-163); out:
 * host, {re hi, re lo, im hi, im lo} per bin. */
amqft_status amqft_direct_bins(const void* d_x, int dtype, size_t rows, size_t row_len, size_t row0,
                               size_t stride, size_t n, const uint64_t* bins, size_t nbins, double* out,
                               void* stream);
amqft_status amqft_direct_bins_extended(const double* x, size_t n, const uint64_t* bins, size_t nbins,
                                        int reverse, double* out);

/* ---- Distributed four-step plan (config 5): one plan per rank, owning its
 * NCCL communicator (NCCL is loaded at run time).  n = n1 n2; rank p passes
 * its column slab [n2/P][2 n1] (x[n2 i1 + i2] for i2 in its slab, interleaved
 * fp32; overwritten) and receives [n1/P][2 n2] = X[k1 + n1 k2] for its
 * k1-slab.  The exchange is grouped ncclSend / ncclRecv on `stream`
 * (AMQFT_ENCCL on NCCL failures).  amqft_dist_unique_id (rank 0) makes the
 * id every rank passes to amqft_dist_plan_create (the caller broadcasts
 * it); id128 may be NULL for nparts = 1 (no communicator, no exchange).
 * Replaces nothing in the reference (it is single-process,
 * src/variants.cpp:404). */
typedef struct amqft_dist_plan_s* amqft_dist_plan;
amqft_status amqft_dist_unique_id(void* id128);
amqft_status amqft_dist_plan_create(amqft_dist_plan* out, int variant, size_t n, int nparts, int rank,
                                    int device, int trig_mode, const void* id128);
amqft_status amqft_dist_plan_shape(amqft_dist_plan plan, size_t* n1, size_t* n2, size_t* rows_in,
                                   size_t* rows_out);
amqft_status amqft_dist_exec_forward(amqft_dist_plan plan, void* d_in, void* d_out, void* stream);
amqft_status amqft_dist_plan_destroy(amqft_dist_plan plan);

/* Batched transpose of complex fp32 matrices: mats x [r][c] -> [c][r];
 * r and c multiples of 32. */
amqft_status amqft_transpose_c64(const void* d_in, void* d_out, size_t mats, size_t r,
                                 size_t c, void* stream);

/* Arithmetic performed per row by the compiled schedule (OpMeter,
 * include/amqft/opmeter.hpp:13-29): {adds, muls, binary translations}. */
amqft_status amqft_plan_op_counts(amqft_plan plan, uint64_t* out3);

/* Which kernel path the plan uses: 0 generic single-CTA schedule,
 * 1 generic multi-pass, 2 fused fast kernel, 3 four-step, 4 small-CDFT /
 * cooperative kernels, 5 fp32 rows through an fp64 plan (widen, fp64
 * plan, narrow).  Number of kernel launches per exec call in *launches. */
amqft_status amqft_plan_path(amqft_plan plan, int* path, int* launches);

/* Four-step plans (path 3): the factors f3 = {A, B, C} with n = A B C
 * (two-factor plans: B = 1, n = A C; A is the column / first factor).
 * AMQFT_EINVAL for other paths. */
amqft_status amqft_plan_fourstep_factors(amqft_plan plan, size_t* f3);

/* Serialise the compiled schedule for host-side inspection (tests):
 * writes up to cap 16-byte elaboration records {op,lens,flags,am,n,off,aux}
 * of program `prog` (0 = root) and returns the record count in *count;
 * stage boundaries (pairs begin,end) go to stages (cap2 pairs). */
amqft_status amqft_plan_dump(amqft_plan plan, int prog, void* records,
                             size_t cap, size_t* count, uint32_t* stages,
                             size_t cap2, size_t* nstages);

/* Host-only schedule compilation (no device needed): compiles (variant,
 * function, n) for a CTA capacity of `capacity_cells` and serialises the
 * single-CTA stage program as amqft_plan_dump does.  Returns AMQFT_EINVAL
 * for requests the reference rejects.  ops3 (nullable) receives the
 * schedule's {adds, muls, binary translations}. */
amqft_status amqft_schedule_dump(int variant, int function, size_t n,
                                 size_t capacity_cells, void* records,
                                 size_t cap, size_t* count, uint32_t* stages,
                                 size_t cap2, size_t* nstages, uint64_t* ops3);

/* Device synchronisation helper and error text. */
amqft_status amqft_device_synchronize(int device);
const char* amqft_last_error(void);
const char* amqft_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AMQFT_B200_H */
