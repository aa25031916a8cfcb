// fast.cu -- dispatcher of the fused CDFT kernels (kernel: fast_kernel.cuh;
// per-variant instances: fast_v1.cu .. fast_v8.cu).
#include "fast.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "fourstep.cuh"
#include "slab.cuh"
#include "gen/small_ops.cuh"

namespace amqft_b200 {
namespace fastk {
// instances: fast_v<V>.cu (CDFT rows), fast_rv<V>.cu (RDFT rows)
template <int V, typename R, bool RD, typename IO = R>
std::unique_ptr<FastPlan> make_sized(size_t n, const void* tab, uint32_t nmax, int dev);

template <int V, typename R, typename IO = R>
std::unique_ptr<FastPlan> make_cluster(size_t n, const void* tab, uint32_t nmax, int dev);

template <int V, typename R, typename IO = R>
std::unique_ptr<FastPlan> make_for_variant(int kind, size_t n, const void* tab, uint32_t nmax, int dev) {
  return kind == 1 ? make_sized<V, R, true, IO>(n, tab, nmax, dev) : make_sized<V, R, false, IO>(n, tab, nmax, dev);
}
}  // namespace fastk

// kind 0: CDFT rows; 1: RDFT rows
template <typename R>
std::unique_ptr<FastPlan> make_fast_typed(int v, int kind, size_t n, const void* tab, uint32_t nmax, int dev) {
  using namespace fastk;
  switch (v) {
    case 1: return make_for_variant<1, R>(kind, n, tab, nmax, dev);
    case 2: return make_for_variant<2, R>(kind, n, tab, nmax, dev);
    case 3: return make_for_variant<3, R>(kind, n, tab, nmax, dev);
    case 4: return make_for_variant<4, R>(kind, n, tab, nmax, dev);
    case 5: return make_for_variant<5, R>(kind, n, tab, nmax, dev);
    case 6: return make_for_variant<6, R>(kind, n, tab, nmax, dev);
    case 7: return make_for_variant<7, R>(kind, n, tab, nmax, dev);
    case 8: return make_for_variant<8, R>(kind, n, tab, nmax, dev);
  }
  return nullptr;
}

// fp32 rows, fp64 arithmetic (variants 5-8, N = 1024-4096): the fused
// kernel's fp64 instance with fp32 loads/stores, on the plan's fp64 copy of
// its constant table.
std::unique_ptr<FastPlan> make_fast_mixed(int v, int kind, size_t n, const void* tab64, uint32_t nmax, int dev) {
  using namespace fastk;
  if (n < 1024 || n > 4096 || !tab64) return nullptr;
  switch (v) {
    case 5: return make_for_variant<5, double, float>(kind, n, tab64, nmax, dev);
    case 6: return make_for_variant<6, double, float>(kind, n, tab64, nmax, dev);
    case 7: return make_for_variant<7, double, float>(kind, n, tab64, nmax, dev);
    case 8: return make_for_variant<8, double, float>(kind, n, tab64, nmax, dev);
  }
  return nullptr;
}


// Cluster four-step (fast_kernel.cuh, k_fast<..., P>): CDFT N = P * 4096
// as P fused rows on one cluster of P CTAs, one pass over HBM.  fp32, and
// fp32 rows computed in fp64 for variants 5-8.  Measured (B200,
// profiles/r02_cluster_ab.log): 1.55-1.85 TB/s at N = 2^13 / 2^14, 1.3 /
// 0.77 TB/s at 2^15 / 2^16 (the per-row DSMEM exchange makes a cluster run in
// lockstep with its slowest CTA, and 16-CTA clusters leave a quarter of the
// SMs idle).  The in-shared-memory four-step (tile_kernel.cuh) now runs N <=
// 2^14 in one pass at 5.1-5.7 TB/s and the multi-pass four-step built on it
// 2^15 / 2^16 at 2.0 TB/s, so no plan picks the cluster kernel by default;
// AMQFT_AB_CLUSTER=all selects it (A/B measurements and its tests).
bool uses_cluster(const amqft_plan_desc& d) {
  if (d.function != AMQFT_FN_CDFT || d.dtype != AMQFT_F32) return false;
  if (d.n < 8192 || d.n > 65536 || (d.n & (d.n - 1))) return false;
  if (const char* e = std::getenv("AMQFT_AB_CLUSTER")) return e[0] == 'a';
  return false;
}

template <typename R, typename IO = R>
std::unique_ptr<FastPlan> make_cluster_typed(int v, size_t n, const void* tab, uint32_t nmax, int dev) {
  using namespace fastk;
  switch (v) {
    case 1: if constexpr (std::is_same<R, IO>::value) return make_cluster<1, R, IO>(n, tab, nmax, dev); break;
    case 2: if constexpr (std::is_same<R, IO>::value) return make_cluster<2, R, IO>(n, tab, nmax, dev); break;
    case 3: if constexpr (std::is_same<R, IO>::value) return make_cluster<3, R, IO>(n, tab, nmax, dev); break;
    case 4: if constexpr (std::is_same<R, IO>::value) return make_cluster<4, R, IO>(n, tab, nmax, dev); break;
    case 5: return make_cluster<5, R, IO>(n, tab, nmax, dev);
    case 6: return make_cluster<6, R, IO>(n, tab, nmax, dev);
    case 7: return make_cluster<7, R, IO>(n, tab, nmax, dev);
    case 8: return make_cluster<8, R, IO>(n, tab, nmax, dev);
  }
  return nullptr;
}

std::unique_ptr<FastPlan> make_fast_plan(const amqft_plan_desc& d, const void* d_trig,
                                         uint32_t nmax, const void* d_trig64) {
  if (d.function != AMQFT_FN_CDFT && d.function != AMQFT_FN_RDFT) return nullptr;
  if (uses_cluster(d)) {
    if (f32_needs_f64_compute(d.variant, d.n))
      return d_trig64 ? make_cluster_typed<double, float>(d.variant, d.n, d_trig64, nmax, d.device) : nullptr;
    return make_cluster_typed<float>(d.variant, d.n, d_trig, nmax, d.device);
  }
  // AM constants: both trig modes read the plan's host-built table, whose
  // values are bitwise the reference's on-the-fly long double values
  // (variants_test.cpp:267-277); the mode matters only for four-step twiddles
  const int kind = d.function == AMQFT_FN_RDFT ? 1 : 0;
  if (d.dtype == AMQFT_F32 && f32_needs_f64_compute(d.variant, d.n))
    return make_fast_mixed(d.variant, kind, d.n, d_trig64, nmax, d.device);
  if (d.dtype == AMQFT_F32) return make_fast_typed<float>(d.variant, kind, d.n, d_trig, nmax, d.device);
  return make_fast_typed<double>(d.variant, kind, d.n, d_trig, nmax, d.device);
}

namespace tilek {
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile(size_t n, const void* tab, uint32_t nmax, int dev);
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile_rdft(size_t n, const void* tab, uint32_t nmax, int dev);
template <int V, typename R>
std::unique_ptr<FastPlan> make_tile_dctdst(int fn, size_t n, const void* tab, uint32_t nmax, int dev);
// the split of tile_kernel.cuh make_tile: N1 (phase A) x N2 (phase B) [x N3
// (phase C); n3 = 1: two factors].  fp32: 4 x 4, 4 x 8, 8 x 8, 8 x 16, 16 x
// 16, 16 x 32, 32 x 32, 64 x 32, 64 x 64, then 32 x 16 x 16, 32 x 16 x 32, 32
// x 32 x 32, 32 x 32 x 64; fp64 the same up to 32 x 32, then 8 x 16 x 16, 16 x
// 16 x 16, 32 x 16 x 16, 32 x 16 x 32, 32 x 32 x 32
static void tile_split(int dtype, size_t n, size_t* n1, size_t* n2, size_t* n3) {
  int lg = 0;
  for (size_t t = n; t > 1; t >>= 1) ++lg;
  *n3 = 1;
  const int three_from = dtype == AMQFT_F64 ? 11 : 13;
  if (lg >= three_from) {
    static const int f32s[4][3] = {{32, 16, 16}, {32, 16, 32}, {32, 32, 32}, {32, 32, 64}};
    static const int f64s[5][3] = {{8, 16, 16}, {16, 16, 16}, {32, 16, 16}, {32, 16, 32}, {32, 32, 32}};
    const int* f = dtype == AMQFT_F64 ? f64s[lg - 11] : f32s[lg - 13];
    *n1 = f[0];
    *n2 = f[1];
    *n3 = f[2];
    return;
  }
  *n1 = size_t(1) << (lg == 11 ? 6 : lg / 2);
  *n2 = n / *n1;
}
}  // namespace tilek

// RDFT rows on the two-factor kernel (tile_kernel.cuh make_tile_rdft), at the sizes where it beats
// the whole-DAG RDFT kernels or only the generic interpreter is left: fp32 N = 256 .. 4096 (measured
// 5467 / 4642 / 5367 / 5084 GB/s at 256 .. 2048 against 57 / 53 on the generic interpreter and 1770 /
// 2349 on the fused kernel; the one-thread-per-row kernel runs N <= 128 at 5 TB/s, the fused kernel
// 8192), fp64 N = 128 .. 1024 under the same tolerance rule as the CDFT rows.
bool tile_rdft_covers(const amqft_plan_desc& d) {
  if (d.function != AMQFT_FN_RDFT || d.order != AMQFT_ORDER_FAST || (d.n & (d.n - 1))) return false;
  if (const char* e = std::getenv("AMQFT_AB_TILE"))
    if (e[0] == 'n') return false;
  if (d.dtype == AMQFT_F64) return d.n >= 128 && d.n <= (d.variant >= 5 ? 256u : 1024u);
  return d.n >= 256 && d.n <= 4096;
}

// DCT-0 / DST-0 rows on the two-factor kernel (make_tile_dctdst): above the scalar small kernels'
// sizes (fp32 N <= 256, fp64 <= 128), where only the generic interpreter was left.
bool tile_dctdst_covers(const amqft_plan_desc& d) {
  if ((d.function != AMQFT_FN_DCT && d.function != AMQFT_FN_DST) || d.order != AMQFT_ORDER_FAST) return false;
  if (d.n & (d.n - 1)) return false;
  if (const char* e = std::getenv("AMQFT_AB_TILE"))
    if (e[0] == 'n') return false;
  if (d.dtype == AMQFT_F64) return d.n >= 256 && d.n <= (d.variant >= 5 ? 256u : 1024u);
  return d.n >= 512 && d.n <= 4096;
}

bool tile_covers(const amqft_plan_desc& d) {
  if (d.function != AMQFT_FN_CDFT || d.order == AMQFT_ORDER_FAST_DAG) return false;
  if (d.n < 16 || (d.n & (d.n - 1))) return false;
  size_t lo = 16, hi = 65536;
  if (d.dtype == AMQFT_F64) {
    // fp64: factors <= 32 points reach N = 2^15.  The result must stay
    // within 1e-12 of the CPU reference of the same variant: variants 1-4
    // do at every size (both ~1e-15 from the DFT); the reference's own
    // variants 5-8 drift from the DFT (4e-14 at N = 256, 1e-10 at 1024,
    // SURVEY 0), so from N = 512 their plans keep the reference DAG (the
    // fused kernel's fp64 instance, bitwise).
    hi = d.variant >= 5 ? 256 : 32768;
    lo = 64;   // N = 16, 32: the one-thread-per-row kernel is 3-6 % faster (and bitwise)
  }
  if (const char* e = std::getenv("AMQFT_AB_TILE")) {
    if (e[0] == 'n') return false;
    // A/B measurements: AMQFT_AB_TILE=lo,hi restricts the sizes it takes
    unsigned long a = 0, b = 0;
    if (std::sscanf(e, "%lu,%lu", &a, &b) == 2) lo = std::max<size_t>(lo, a), hi = std::min<size_t>(hi, b);
  }
  return d.n >= lo && d.n <= hi;
}

template <typename R>
static std::unique_ptr<FastPlan> make_tile_typed(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax) {
  using namespace tilek;
  if (d.function == AMQFT_FN_RDFT) {
    switch (d.variant) {
      case 1: return make_tile_rdft<1, R>(d.n, d_trig, nmax, d.device);
      case 2: return make_tile_rdft<2, R>(d.n, d_trig, nmax, d.device);
      case 3: return make_tile_rdft<3, R>(d.n, d_trig, nmax, d.device);
      case 4: return make_tile_rdft<4, R>(d.n, d_trig, nmax, d.device);
      case 5: return make_tile_rdft<5, R>(d.n, d_trig, nmax, d.device);
      case 6: return make_tile_rdft<6, R>(d.n, d_trig, nmax, d.device);
      case 7: return make_tile_rdft<7, R>(d.n, d_trig, nmax, d.device);
      case 8: return make_tile_rdft<8, R>(d.n, d_trig, nmax, d.device);
    }
    return nullptr;
  }
  if (d.function == AMQFT_FN_DCT || d.function == AMQFT_FN_DST) {
    switch (d.variant) {
      case 1: return make_tile_dctdst<1, R>(d.function, d.n, d_trig, nmax, d.device);
      case 2: return make_tile_dctdst<2, R>(d.function, d.n, d_trig, nmax, d.device);
      case 3: return make_tile_dctdst<3, R>(d.function, d.n, d_trig, nmax, d.device);
      case 4: return make_tile_dctdst<4, R>(d.function, d.n, d_trig, nmax, d.device);
      case 5: return make_tile_dctdst<5, R>(d.function, d.n, d_trig, nmax, d.device);
      case 6: return make_tile_dctdst<6, R>(d.function, d.n, d_trig, nmax, d.device);
      case 7: return make_tile_dctdst<7, R>(d.function, d.n, d_trig, nmax, d.device);
      case 8: return make_tile_dctdst<8, R>(d.function, d.n, d_trig, nmax, d.device);
    }
    return nullptr;
  }
  switch (d.variant) {
    case 1: return make_tile<1, R>(d.n, d_trig, nmax, d.device);
    case 2: return make_tile<2, R>(d.n, d_trig, nmax, d.device);
    case 3: return make_tile<3, R>(d.n, d_trig, nmax, d.device);
    case 4: return make_tile<4, R>(d.n, d_trig, nmax, d.device);
    case 5: return make_tile<5, R>(d.n, d_trig, nmax, d.device);
    case 6: return make_tile<6, R>(d.n, d_trig, nmax, d.device);
    case 7: return make_tile<7, R>(d.n, d_trig, nmax, d.device);
    case 8: return make_tile<8, R>(d.n, d_trig, nmax, d.device);
  }
  return nullptr;
}

std::unique_ptr<FastPlan> make_tile_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax) {
  if (!tile_covers(d) && !tile_rdft_covers(d) && !tile_dctdst_covers(d)) return nullptr;
  return d.dtype == AMQFT_F64 ? make_tile_typed<double>(d, d_trig, nmax) : make_tile_typed<float>(d, d_trig, nmax);
}

namespace slabk {
template <int V, typename R>
std::unique_ptr<SlabPassExec<R>> make_slab_pass(size_t len, const void* tab, uint32_t nmax, int dev);
}  // namespace slabk

template <typename R>
std::unique_ptr<slabk::SlabPassExec<R>> make_slab_pass_rt(int variant, size_t len, const void* tab, uint32_t nmax,
                                                          int dev) {
  using namespace slabk;
  switch (variant) {
    case 1: return make_slab_pass<1, R>(len, tab, nmax, dev);
    case 2: return make_slab_pass<2, R>(len, tab, nmax, dev);
    case 3: return make_slab_pass<3, R>(len, tab, nmax, dev);
    case 4: return make_slab_pass<4, R>(len, tab, nmax, dev);
    case 5: return make_slab_pass<5, R>(len, tab, nmax, dev);
    case 6: return make_slab_pass<6, R>(len, tab, nmax, dev);
    case 7: return make_slab_pass<7, R>(len, tab, nmax, dev);
    case 8: return make_slab_pass<8, R>(len, tab, nmax, dev);
  }
  return nullptr;
}
template std::unique_ptr<slabk::SlabPassExec<float>> make_slab_pass_rt<float>(int, size_t, const void*, uint32_t, int);
template std::unique_ptr<slabk::SlabPassExec<double>> make_slab_pass_rt<double>(int, size_t, const void*, uint32_t, int);

namespace smallk {
bool small_ops_n(int v, size_t n, bool f64, OpCount* o, int fn = AMQFT_FN_CDFT);
}

OpCount tile_op_counts(const amqft_plan_desc& d) {
  // N2 sub-transforms of length N1 and N1 of length N2 (the reference DAG of
  // each: the traced schedule's meter) plus one complex twiddle multiply
  // per element (4 muls + 2 adds), as the four-step's accounting
  size_t n1, n2, n3;
  tilek::tile_split(d.dtype, d.n, &n1, &n2, &n3);
  const bool f64 = d.dtype == AMQFT_F64;
  OpCount c1, c2, c3, c;
  smallk::small_ops_n(d.variant, n1, f64, &c1, AMQFT_FN_CDFT);
  smallk::small_ops_n(d.variant, n2, f64, &c2, AMQFT_FN_CDFT);
  if (n3 > 1) {   // three factors, two twiddle passes
    smallk::small_ops_n(d.variant, n3, f64, &c3, AMQFT_FN_CDFT);
    c.adds = n2 * n3 * c1.adds + n1 * n3 * c2.adds + n1 * n2 * c3.adds + 2 * 2 * d.n;
    c.muls = n2 * n3 * c1.muls + n1 * n3 * c2.muls + n1 * n2 * c3.muls + 2 * 4 * d.n;
    c.bt = n2 * n3 * c1.bt + n1 * n3 * c2.bt + n1 * n2 * c3.bt;
    return c;
  }
  c.adds = n2 * c1.adds + n1 * c2.adds + 2 * d.n;
  c.muls = n2 * c1.muls + n1 * c2.muls + 4 * d.n;
  c.bt = n2 * c1.bt + n1 * c2.bt;
  return c;
}

namespace smallk {
template <int V, typename R>
std::unique_ptr<FastPlan> make_small_sized(size_t n, const void* tab, uint32_t nmax, int dev);
template <int V, typename R>
std::unique_ptr<FastPlan> make_small_rdft(size_t n, const void* tab, uint32_t nmax, int dev);
template <int V, typename R>
std::unique_ptr<FastPlan> make_small_dctdst(int fn, size_t n, const void* tab, uint32_t nmax, int dev);

bool small_ops_n(int v, size_t n, bool f64, OpCount* o, int fn) {
  for (const SmallOps& e : kSmallOps)
    if (e.v == v && e.fn == fn && (size_t(1) << e.logn) == n && e.f64 == static_cast<int>(f64)) {
      o->adds = e.a;
      o->muls = e.m;
      o->bt = e.b;
      return true;
    }
  return false;
}
template <typename R>
std::unique_ptr<FastPlan> make_small_typed(int v, size_t n, const void* tab, uint32_t nmax, int dev, OpCount* o,
                                           int fn) {
  switch (v) {
#define AMQFT_SMALL_CASE(V) \
  case V: if (!small_ops_n(V, n, sizeof(R) == 8, o, fn)) return nullptr; \
    return fn == AMQFT_FN_RDFT ? make_small_rdft<V, R>(n, tab, nmax, dev)                                  \
         : fn == AMQFT_FN_CDFT ? make_small_sized<V, R>(n, tab, nmax, dev)                                 \
                               : make_small_dctdst<V, R>(fn, n, tab, nmax, dev);
    AMQFT_SMALL_CASE(1) AMQFT_SMALL_CASE(2) AMQFT_SMALL_CASE(3) AMQFT_SMALL_CASE(4)
    AMQFT_SMALL_CASE(5) AMQFT_SMALL_CASE(6) AMQFT_SMALL_CASE(7) AMQFT_SMALL_CASE(8)
#undef AMQFT_SMALL_CASE
  }
  return nullptr;
}
}  // namespace smallk

std::unique_ptr<FastPlan> make_small_plan(const amqft_plan_desc& d, const void* d_trig, uint32_t nmax,
                                          OpCount* ops) {
  if (d.function > AMQFT_FN_DST) return nullptr;   // AM constants from the table in both trig modes
  if (d.dtype == AMQFT_F32 && f32_needs_f64_compute(d.variant, d.n)) return nullptr;
  if (d.dtype == AMQFT_F32)
    return smallk::make_small_typed<float>(d.variant, d.n, d_trig, nmax, d.device, ops, d.function);
  return smallk::make_small_typed<double>(d.variant, d.n, d_trig, nmax, d.device, ops, d.function);
}

OpCount fast_op_counts(const amqft_plan_desc& d) {
  if (uses_cluster(d)) {
    // P rows of the 4096-point DAG, N/P radix-2 P-point DFTs (each
    // butterfly: one complex multiply, 4 muls + 2 adds, and 4 adds), and per
    // DFT P - 1 twiddle multiplies plus P - 2 for the twiddle powers
    // (4 muls + 2 adds each)
    amqft_plan_desc s = d;
    s.n = 4096;
    const OpCount r = fast_op_counts(s);
    const uint64_t P = d.n / 4096;
    uint64_t lgp = 0;
    for (uint64_t t = P; t > 1; t >>= 1) ++lgp;
    const uint64_t dfts = d.n / P, bfly = dfts * (P / 2) * lgp, tw = (2 * P - 3) * dfts;
    OpCount c;
    c.adds = P * r.adds + bfly * 6 + tw * 2;
    c.muls = P * r.muls + bfly * 4 + tw * 4;
    c.bt = P * r.bt;
    return c;
  }
  // The fused kernel executes exactly the reference DAG (fast_model.py):
  // the closed forms of metering.cpp:85-96.
  OpCount c;
  uint64_t lg = 0;
  for (size_t v = d.n; v > 1; v >>= 1) ++lg;
  const uint64_t n = d.n;
  c.adds = 3 * n * lg - 3 * n + 4;
  c.muls = n * lg - 3 * n + 4;
  c.bt = (d.variant % 2 == 1) ? n - 4 * lg + 4 : 0;
  if (d.function == AMQFT_FN_RDFT) {
    // CDFT = SplitComplex bwd (2N - 4 adds, elaborations_test.cpp:91-92) + 2 RDFT
    c.adds = (c.adds - (2 * n - 4)) / 2;
    c.muls /= 2;
    c.bt /= 2;
  }
  return c;
}

static amqft_plan_desc sub_desc(int variant, size_t n, int dtype) {
  amqft_plan_desc d{};
  d.variant = variant;
  d.function = AMQFT_FN_CDFT;
  d.n = n;
  d.batch = 1;
  d.dtype = dtype;
  d.trig_mode = AMQFT_TRIG_TABLE;
  d.order = AMQFT_ORDER_FAST;
  return d;
}

bool fast_sub_covered(int dtype, size_t n, int variant, bool allow_tile) {
  if (allow_tile && tile_covers(sub_desc(variant, n, dtype))) return true;   // fp32 16 .. 65536, every variant
  if (dtype == AMQFT_F32 && f32_needs_f64_compute(variant, n)) return n >= 1024 && n <= 4096;
  if (dtype == AMQFT_F32) return n >= 2 && n <= 8192;
  return n >= 2 && n <= 4096 && n != 512;
}

std::unique_ptr<FastPlan> make_fast_sub(int variant, size_t n, int dtype, const void* tab, uint32_t nmax, int dev,
                                        const void* tab64, bool columns) {
  amqft_plan_desc d{};
  d.variant = variant;
  d.function = AMQFT_FN_CDFT;
  d.n = n;
  d.batch = 1;
  d.dtype = dtype;
  d.trig_mode = AMQFT_TRIG_TABLE;
  d.order = AMQFT_ORDER_FAST;
  d.device = dev;
  std::unique_ptr<FastPlan> p;
  if (columns) {   // column mode: the one-thread-per-row kernel (N <= 64 fp32, 32 fp64)
    OpCount oc;
    return make_small_plan(d, tab, nmax, &oc);
  }
  p = make_tile_plan(d, tab, nmax);
  if (!p) p = make_fast_plan(d, tab, nmax, tab64);
  OpCount o;
  if (!p) p = make_small_plan(d, tab, nmax, &o);
  return p;
}

OpCount fast_sub_op_counts(int variant, size_t n, int dtype, bool columns) {
  amqft_plan_desc d{};
  d.variant = variant;
  d.function = AMQFT_FN_CDFT;
  d.n = n;
  d.dtype = dtype;
  OpCount o;
  if (!columns && tile_covers(sub_desc(variant, n, dtype))) return tile_op_counts(d);
  if (n >= 1024) return fast_op_counts(d);
  smallk::small_ops_n(variant, n, dtype == AMQFT_F64, &o);
  return o;
}

}  // namespace amqft_b200
