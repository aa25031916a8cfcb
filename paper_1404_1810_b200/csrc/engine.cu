// engine.cu -- plan objects, kernel launches and the C ABI (amqft_b200.h).
//
// Execution paths (chosen at plan creation, no runtime fallback):
//   path 0  generic single-CTA: one CTA per row runs the whole compiled
//           stage program out of shared memory (k_prog).
//   path 1  generic multi-pass: nodes whose operand exceeds the CTA
//           capacity run as grid-wide stages over two HBM arenas (k_stage),
//           the subtrees below as per-CTA jobs (k_prog).  This keeps the
//           reference recursion (and fp64 bitwise parity) at any N.
//   path 2  fused fast kernels (fast.cuh) for the CDFT hot path.
//   path 3  four-step over the fused kernel (fourstep.cuh), large N, fp32.
//   path 4  one thread per row (small_kernel.cuh), small CDFTs.
//   path 6  four-step inside one CTA's shared memory (tile_kernel.cuh),
//           fp32 CDFT N = 256 .. 4096, one pass over HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/amqft_b200.h"
#include "fast.cuh"
#include "fourstep.cuh"
#include "generic_exec.hpp"
#include "inverse.cuh"
#include "plan.hpp"
#include "trig.hpp"

using namespace amqft_b200;

namespace {

thread_local std::string g_err;

}  // namespace

namespace amqft_b200 {
void set_last_error(const std::string& m) { g_err = m; }
}  // namespace amqft_b200

namespace {

amqft_status set_err(amqft_status s, const std::string& m) {
  g_err = m;
  return s;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Every extern "C" entry point ends in `catch (...) { return from_exception(); }`:
// no C++ exception crosses the C ABI.  std::invalid_argument (the
// reference's error type, variants.cpp:404-421) -> EINVAL; allocation
// failures (host bad_alloc, cudaErrorMemoryAllocation) -> ENOMEM; any other
// error (CUDA launch/runtime) -> ECUDA.
amqft_status from_exception() {
  try {
    throw;
  } catch (const std::invalid_argument& e) {
    return set_err(AMQFT_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(AMQFT_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    const std::string m = e.what();
    if (m.find(cudaGetErrorString(cudaErrorMemoryAllocation)) != std::string::npos) {
      cudaGetLastError();   // clear the (non-sticky) allocation error
      return set_err(AMQFT_ENOMEM, m);
    }
    return set_err(AMQFT_ECUDA, m);
  } catch (...) {
    return set_err(AMQFT_ECUDA, "unknown exception");
  }
}

// Kernels and launchers live in generic_kernels.cuh (instantiated per dtype
// in generic_f32.cu / generic_f64.cu so the build parallelises).

}  // namespace

// ---------------------------------------------------------------------------
// Plan object.

struct amqft_plan_s {
  amqft_plan_desc d{};
  Compiled c;
  int path = 0;
  int T = 256, K = 1;
  size_t smem = 0;
  size_t capacity = 0;
  size_t esize = 8;
  uint32_t nmax = 8;
  // device arrays
  void* d_trig = nullptr;
  void* d_trig64 = nullptr;   // fp32 plans computing in fp64: the fp64 copy of the table
  EI* d_eis = nullptr;
  uint32_t* d_prefix = nullptr;
  Stage* d_stages = nullptr;
  ProgInfo* d_progs = nullptr;
  JobDev* d_jobs = nullptr;   // multi-pass jobs; for path 0 a single job
  uint32_t njobs = 0;
  EI* d_geis = nullptr;       // global EIs
  uint32_t* d_gprefix = nullptr;
  void* bufA = nullptr;
  void* bufB = nullptr;
  std::unique_ptr<FastPlan> fast;
  int launches = 0;
  int sms = 148;
  // fp32 rows computed by an fp64 plan (fast.cuh f32_needs_f64_compute,
  // path 5): widen into wide_in, run `wide`, narrow from wide_out
  amqft_plan_s* wide = nullptr;
  void* wide_in = nullptr;
  void* wide_out = nullptr;
  // host-buffer pipeline (amqft_exec_host_rows), created on its first call
  // (serialised by host_mu: one pipeline per plan)
  std::mutex host_mu;
  static constexpr int NSLOT = 3;
  void* slot[NSLOT] = {nullptr, nullptr, nullptr};
  size_t slot_rows = 0;
  cudaStream_t s_h2d = nullptr, s_run = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[NSLOT] = {}, ev_run[NSLOT] = {}, ev_d2h[NSLOT] = {}, ev_in = nullptr;
  // inverses of the real transforms (inverse.cu), created with the plan
  void* inv_a = nullptr;
  void* inv_b = nullptr;
  amqft_plan_s* inv_dct = nullptr;
  amqft_plan_s* inv_dst = nullptr;

  ~amqft_plan_s() {
    delete inv_dct;
    delete inv_dst;
    delete wide;
    if (inv_a) cudaFree(inv_a);
    if (inv_b) cudaFree(inv_b);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(d.device);
    for (void* p : {static_cast<void*>(d_trig), d_trig64, static_cast<void*>(d_eis),
                    static_cast<void*>(d_prefix), static_cast<void*>(d_stages),
                    static_cast<void*>(d_progs), static_cast<void*>(d_jobs),
                    static_cast<void*>(d_geis), static_cast<void*>(d_gprefix),
                    bufA, bufB, slot[0], slot[1], slot[2], wide_in, wide_out})
      if (p) cudaFree(p);
    for (cudaStream_t q : {s_h2d, s_run, s_d2h})
      if (q) cudaStreamDestroy(q);
    for (int k = 0; k < NSLOT; ++k)
      for (cudaEvent_t e : {ev_h2d[k], ev_run[k], ev_d2h[k]})
        if (e) cudaEventDestroy(e);
    if (ev_in) cudaEventDestroy(ev_in);
    fast.reset();
    cudaSetDevice(cur);
  }
};

namespace {

template <typename Tv>
Tv* upload(const std::vector<Tv>& v) {
  if (v.empty()) return nullptr;
  Tv* p = nullptr;
  ck(cudaMalloc(&p, v.size() * sizeof(Tv)), "cudaMalloc");
  ck(cudaMemcpy(p, v.data(), v.size() * sizeof(Tv), cudaMemcpyHostToDevice), "cudaMemcpy");
  return p;
}

int pick_k(uint32_t per_thread) {
  int k = 1;
  while (k < static_cast<int>(per_thread)) k *= 2;
  return k;
}

void build_generic(amqft_plan_s* P) {
  const Compiled& c = P->c;
  // Concatenate programs.
  std::vector<EI> eis;
  std::vector<uint32_t> prefix;
  std::vector<Stage> stages;
  std::vector<ProgInfo> infos;
  uint32_t max_items = 0, max_cells = 0;
  for (const SubProgram& sp : c.progs) {
    ProgInfo pi;
    pi.ei_base = static_cast<uint32_t>(eis.size());
    pi.stage_base = static_cast<uint32_t>(stages.size());
    pi.nstages = static_cast<uint32_t>(sp.stages.size());
    pi.cells = static_cast<uint32_t>(sp.cells);
    eis.insert(eis.end(), sp.eis.begin(), sp.eis.end());
    prefix.insert(prefix.end(), sp.prefix.begin(), sp.prefix.end());
    stages.insert(stages.end(), sp.stages.begin(), sp.stages.end());
    infos.push_back(pi);
    max_items = std::max(max_items, sp.max_items);
    max_cells = std::max(max_cells, static_cast<uint32_t>(sp.cells));
  }
  P->T = max_items > 1024 ? 512 : 256;
  P->K = pick_k((max_items + P->T - 1) / P->T);
  if (P->K > 32) throw std::invalid_argument("subtree too large for one CTA");
  P->smem = std::max<size_t>(16, max_cells * P->esize);
  P->d_eis = upload(eis);
  P->d_prefix = upload(prefix);
  P->d_stages = upload(stages);
  P->d_progs = upload(infos);
  std::vector<JobDev> jobs;
  if (c.single) {
    jobs.push_back(JobDev{0, 0, 0, 0});
  } else {
    for (const Job& j : c.jobs) jobs.push_back(JobDev{j.prog, j.off, j.src, j.dst});
    std::vector<uint32_t> gp(c.global_eis.size());
    for (const auto* sv : {&c.fwd_stages, &c.bwd_stages})
      for (const Stage& st : *sv) {
        uint32_t acc = 0;
        for (uint32_t k = st.ei_begin; k < st.ei_end; ++k) {
          gp[k] = acc;
          acc += ei_items(c.global_eis[k]);
        }
      }
    P->d_geis = upload(c.global_eis);
    P->d_gprefix = upload(gp);
    const size_t bytes = P->d.batch * c.cells * P->esize;
    ck(cudaMalloc(&P->bufA, bytes), "cudaMalloc arena A");
    ck(cudaMalloc(&P->bufB, bytes), "cudaMalloc arena B");
  }
  P->njobs = static_cast<uint32_t>(jobs.size());
  P->d_jobs = upload(jobs);
  P->launches = c.single ? 1
                         : static_cast<int>(2 + c.fwd_stages.size() + c.bwd_stages.size() + 1);
}

template <typename R>
void exec_generic(amqft_plan_s* P, const void* in, void* out, size_t rows,
                  int inverse, cudaStream_t st) {
  const Compiled& c = P->c;
  TrigRef trig{P->d_trig, P->nmax, static_cast<uint32_t>(modulation_kind(P->d.variant)),
               static_cast<uint32_t>(P->d.trig_mode == AMQFT_TRIG_ONTHEFLY)};
  const double scale = 1.0 / static_cast<double>(P->d.n);
  const size_t sms = static_cast<size_t>(P->sms);
  const int swap = inverse ? 1 : 0;
  ProgLaunch L{};
  L.eis = P->d_eis;
  L.prefix = P->d_prefix;
  L.stages = P->d_stages;
  L.progs = P->d_progs;
  L.jobs = P->d_jobs;
  L.trig = trig;
  L.smem = P->smem;
  L.T = P->T;
  L.K = P->K;
  L.stream = st;
  L.arena = c.cells;
  L.rows = rows;
  if (c.single) {
    L.njobs = 1;
    L.srcA = in;
    L.dstA = out;
    L.swap_in = L.swap_out = swap;
    L.scale = scale;
    L.grid = static_cast<unsigned>(std::min<size_t>(rows, sms * 32));
    ck(launch_prog<R>(L), "k_prog launch");
    return;
  }
  void* A = P->bufA;
  void* B = P->bufB;
  const size_t total = rows * c.cells;
  const unsigned cgrid = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, sms * 64));
  ck(launch_copy<R>(in, c.root_src ? B : A, total, swap, 1.0, cgrid, st), "k_copy_rows");
  auto stage_run = [&](const Stage& s) {
    const size_t work = static_cast<size_t>(s.items) * rows;
    const unsigned g = static_cast<unsigned>(std::min<size_t>((work + 255) / 256, sms * 64));
    ck(launch_stage<R>(P->d_geis, P->d_gprefix, s, A, B, c.cells, rows, trig, g, st), "k_stage");
  };
  for (const Stage& s : c.fwd_stages) stage_run(s);
  L.njobs = P->njobs;
  L.srcA = A;
  L.srcB = B;
  L.dstA = A;
  L.dstB = B;
  L.swap_in = L.swap_out = 0;
  L.scale = 1.0;
  L.grid = static_cast<unsigned>(std::min<size_t>(rows * P->njobs, sms * 32));
  ck(launch_prog<R>(L), "k_prog jobs launch");
  for (const Stage& s : c.bwd_stages) stage_run(s);
  ck(launch_copy<R>(c.root_dst ? B : A, out, total, swap, scale, cgrid, st), "k_copy_rows");
}

bool inverse_defined(const amqft_plan_s* P) {
  return P->d.function == AMQFT_FN_CDFT ||
         ((P->d.function == AMQFT_FN_RDFT || P->d.function == AMQFT_FN_DCT || P->d.function == AMQFT_FN_DST) &&
          P->d.n >= 4);
}

// The real-transform inverses' scratch rows and DCT-0 / DST-0 sub-plans
// (inverse.cu) are made with the plan, so exec allocates nothing.
thread_local bool g_inverse_subplan = false;   // creating an inverse's own sub-plans

amqft_status create_plan(amqft_plan* out, const amqft_plan_desc* desc, const std::vector<double>* host_tab);

void prepare_inverse(amqft_plan_s* P, const std::vector<double>* host_tab) {
  if (g_inverse_subplan) return;   // the sub-plans only run forward
  if (!inverse_defined(P) || P->d.function == AMQFT_FN_CDFT || P->d.function == AMQFT_FN_DST) return;
  const size_t h = P->d.n / 2;
  if (P->d.function == AMQFT_FN_DCT) {
    ck(cudaMalloc(&P->inv_a, P->d.batch * P->c.cells * P->esize), "cudaMalloc inverse scratch");
    return;
  }
  auto sub = [&](int fn) -> amqft_plan_s* {
    amqft_plan_desc d = P->d;
    d.function = fn;
    amqft_plan q = nullptr;
    g_inverse_subplan = true;
    const amqft_status s = create_plan(&q, &d, host_tab);
    g_inverse_subplan = false;
    if (s == AMQFT_ENOMEM) throw CudaError(std::string("inverse sub-plan: ") + g_err);
    if (s != AMQFT_OK) throw std::runtime_error(std::string("inverse sub-plan: ") + g_err);
    return q;
  };
  P->inv_dct = sub(AMQFT_FN_DCT);
  P->inv_dst = sub(AMQFT_FN_DST);
  ck(cudaMalloc(&P->inv_a, P->d.batch * (h + 1) * P->esize), "cudaMalloc inverse scratch");
  ck(cudaMalloc(&P->inv_b, P->d.batch * (h - 1) * P->esize), "cudaMalloc inverse scratch");
}

amqft_status validate_desc(const amqft_plan_desc* d) {
  if (!d) return set_err(AMQFT_EINVAL, "null plan descriptor");
  if (d->variant < 1 || d->variant > 8) return set_err(AMQFT_EINVAL, "variant number must be in 1..8");
  if (d->function < 0 || d->function >= kNumFn) return set_err(AMQFT_EINVAL, "unknown function");
  if (d->dtype != AMQFT_F32 && d->dtype != AMQFT_F64) return set_err(AMQFT_EINVAL, "dtype must be F32 or F64");
  if (d->trig_mode != AMQFT_TRIG_TABLE && d->trig_mode != AMQFT_TRIG_ONTHEFLY)
    return set_err(AMQFT_EINVAL, "unknown trig mode");
  if (d->order != AMQFT_ORDER_EXACT && d->order != AMQFT_ORDER_FAST && d->order != AMQFT_ORDER_FAST_DAG)
    return set_err(AMQFT_EINVAL, "unknown execution order");
  if (d->batch == 0) return set_err(AMQFT_EINVAL, "batch must be >= 1");
  return AMQFT_OK;
}

}  // namespace

extern "C" {

const char* amqft_last_error(void) { return g_err.c_str(); }
const char* amqft_version(void) { return "amqft_b200 0.1 (sm_100a)"; }

}  // extern "C"

namespace {

// Plan creation.  host_tab (nullable): the caller's constants in the
// TrigTable::constants layout for Nmax = table_max_n (or max(n, 8)) --
// amqft_plan_create_with_constants, the C++ execute over an arbitrary
// TrigSource; otherwise the TrigTable values are built here.
amqft_status create_plan(amqft_plan* out, const amqft_plan_desc* desc, const std::vector<double>* host_tab) {
  if (!out) return set_err(AMQFT_EINVAL, "null plan pointer");
  *out = nullptr;
  const amqft_status vs = validate_desc(desc);
  if (vs != AMQFT_OK) return vs;
  std::unique_ptr<amqft_plan_s> P(new amqft_plan_s());
  P->d = *desc;
  try {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      return set_err(AMQFT_ECUDA, "no CUDA device: the AM-QFT library has no CPU path");
    if (desc->device < 0 || desc->device >= ndev)
      return set_err(AMQFT_EINVAL, "device ordinal out of range");
    ck(cudaSetDevice(desc->device), "cudaSetDevice");
    cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, desc->device);
    P->esize = desc->dtype == AMQFT_F64 ? 8 : 4;
    const size_t n = desc->n;
    const size_t tmax = desc->table_max_n ? desc->table_max_n : std::max<size_t>(n, 8);
    if (tmax < n || (tmax & (tmax - 1)) != 0 || tmax < 8)
      return set_err(AMQFT_EINVAL, "constant table needs a power-of-two max periodization >= max(n, 8)");
    P->nmax = static_cast<uint32_t>(tmax);
    // Constant table (TrigTable::constants layout), host long double.
    if (host_tab && host_tab->size() != tmax / 4)
      return set_err(AMQFT_EINVAL, "constant table must hold table_max_n / 4 values (slots, then the base constant)");
    const std::vector<double> tab =
        host_tab ? *host_tab : trig_table(desc->variant, tmax, desc->corrupt_constants != 0);
    if (desc->dtype == AMQFT_F64) {
      P->d_trig = upload(tab);
    } else {
      std::vector<float> tf(tab.begin(), tab.end());
      P->d_trig = upload(tf);
      if (f32_needs_f64_compute(desc->variant, n)) P->d_trig64 = upload(tab);
    }
    // Fast fused path where one exists for this request.
    if (desc->order == AMQFT_ORDER_FAST || desc->order == AMQFT_ORDER_FAST_DAG) {
      int fpath = 6;
      P->fast = make_tile_plan(*desc, P->d_trig, P->nmax);
      if (!P->fast) {
        P->fast = make_fast_plan(*desc, P->d_trig, P->nmax, P->d_trig64);
        fpath = 2;
      }
      OpCount small_ops{};
      if (!P->fast) {
        P->fast = make_small_plan(*desc, P->d_trig, P->nmax, &small_ops);
        if (P->fast) fpath = 4;
      }
      if (!P->fast && fourstep_covers(*desc)) {
        P->fast = make_fourstep_plan(*desc, P->d_trig, P->nmax, P->d_trig64);
        fpath = 3;
      }
      if (P->fast) {
        P->path = fpath;
        P->c.variant = desc->variant;
        P->c.fn = desc->function;
        P->c.n = n;
        P->c.cells = fn_cells(desc->function, n);
        P->c.ops = fpath == 6   ? tile_op_counts(*desc)
                   : fpath == 2 ? fast_op_counts(*desc)
                   : fpath == 4 ? small_ops
                                : fourstep_op_counts(*desc);
        P->launches = P->fast->launches;
        prepare_inverse(P.get(), host_tab);
        *out = P.release();
        return AMQFT_OK;
      }
    }
    if (desc->dtype == AMQFT_F32 && f32_needs_f64_compute(desc->variant, n)) {
      // fp32 rows through an fp64 plan of the same request (the generic
      // exact path, or the fp64 fast paths): the fp32 recursion of the
      // sine-family variants is unstable at this size (fast.cuh)
      amqft_plan_desc d64 = *desc;
      d64.dtype = AMQFT_F64;
      amqft_plan w = nullptr;
      const amqft_status s = create_plan(&w, &d64, host_tab);
      if (s != AMQFT_OK) return s;
      P->wide = w;
      P->c.variant = desc->variant;
      P->c.fn = desc->function;
      P->c.n = n;
      P->c.cells = w->c.cells;
      P->c.ops = w->c.ops;
      const size_t bytes = desc->batch * P->c.cells * sizeof(double);
      ck(cudaMalloc(&P->wide_in, bytes), "cudaMalloc fp64 working rows");
      ck(cudaMalloc(&P->wide_out, bytes), "cudaMalloc fp64 working rows");
      P->path = 5;
      P->launches = w->launches + 2;
      *out = P.release();
      return AMQFT_OK;
    }
    P->capacity = desc->dtype == AMQFT_F64 ? 8192 : 16384;
    P->c = compile(desc->variant, desc->function, n, P->capacity);
    P->path = P->c.single ? 0 : 1;
    build_generic(P.get());
    prepare_inverse(P.get(), host_tab);
  } catch (...) {
    return from_exception();
  }
  *out = P.release();
  return AMQFT_OK;
}

}  // namespace

extern "C" {

amqft_status amqft_plan_create(amqft_plan* out, const amqft_plan_desc* desc) {
  return create_plan(out, desc, nullptr);
}

amqft_status amqft_plan_create_transposable(amqft_plan* out, const amqft_plan_desc* desc) {
  fourstep_prefer_transposable(true);   // thread-local: read by the four-step's plan selection
  const amqft_status s = create_plan(out, desc, nullptr);
  fourstep_prefer_transposable(false);
  return s;
}

amqft_status amqft_plan_create_with_constants(amqft_plan* out, const amqft_plan_desc* desc,
                                              const double* constants, size_t count) {
  if (!constants) return set_err(AMQFT_EINVAL, "null constant table");
  try {
    const std::vector<double> tab(constants, constants + count);
    return create_plan(out, desc, &tab);
  } catch (...) {
    return from_exception();
  }
}

amqft_status amqft_plan_destroy(amqft_plan plan) {
  delete plan;
  return AMQFT_OK;
}

size_t amqft_plan_cells(amqft_plan plan) { return plan ? plan->c.cells : 0; }

namespace {

// Inverse RDFT / DCT-0 / DST-0 (inverse.cu): the plan's own forward DCT-0 /
// DST-0 between exact power-of-two weightings.
amqft_status exec_real_inverse(amqft_plan_s* P, const void* in, void* out, size_t rows, cudaStream_t st) {
  const int f64 = P->d.dtype == AMQFT_F64;
  const double n = static_cast<double>(P->d.n);
  if (P->d.function == AMQFT_FN_DST) {          // (4/N) DST-0(S)
    amqft_status s = amqft_exec_rows(P, in, out, rows, 0, st);
    if (s != AMQFT_OK) return s;
    inv_weight(f64, out, out, rows, P->c.cells, 4.0 / n, 4.0 / n, st);
    return AMQFT_OK;
  }
  if (P->d.function == AMQFT_FN_DCT) {          // (4/N) W DCT-0(W C)
    inv_weight(f64, in, P->inv_a, rows, P->c.cells, 1.0, 0.5, st);
    amqft_status s = amqft_exec_rows(P, P->inv_a, out, rows, 0, st);
    if (s != AMQFT_OK) return s;
    inv_weight(f64, out, out, rows, P->c.cells, 4.0 / n, 2.0 / n, st);
    return AMQFT_OK;
  }
  // RDFT: split the packed spectrum, DCT-0 and DST-0 inverses, butterfly
  inv_rdft_split(f64, in, P->inv_a, P->inv_b, rows, P->d.n, st);
  amqft_status s = amqft_exec_rows(P->inv_dct, P->inv_a, P->inv_a, rows, 0, st);
  if (s == AMQFT_OK) s = amqft_exec_rows(P->inv_dst, P->inv_b, P->inv_b, rows, 0, st);
  if (s != AMQFT_OK) return s;
  inv_rdft_combine(f64, P->inv_a, P->inv_b, out, rows, P->d.n, 4.0 / n, st);
  return AMQFT_OK;
}

}  // namespace

amqft_status amqft_exec_rows(amqft_plan P, const void* in, void* out, size_t rows,
                             int inverse, void* stream) {
  if (!P) return set_err(AMQFT_EINVAL, "null plan");
  if (rows > P->d.batch) return set_err(AMQFT_EINVAL, "rows exceed the plan batch");
  if (inverse && !inverse_defined(P))
    return set_err(AMQFT_EINVAL, "the inverse is defined for CDFT, and for RDFT / DCT / DST plans with n >= 4");
  if (P->wide) {   // fp32 rows, fp64 plan (path 5)
    if (rows == 0) return AMQFT_OK;
    if (!in || !out) return set_err(AMQFT_EINVAL, "null data pointer");
    try {
      ck(cudaSetDevice(P->d.device), "cudaSetDevice");
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      convert_rows(1, in, P->wide_in, rows * P->c.cells, st);
      const amqft_status s = amqft_exec_rows(P->wide, P->wide_in, P->wide_out, rows, inverse, stream);
      if (s != AMQFT_OK) return s;
      convert_rows(0, P->wide_out, out, rows * P->c.cells, st);
    } catch (...) {
      return from_exception();
    }
    return AMQFT_OK;
  }
  if (inverse && P->d.function != AMQFT_FN_CDFT) {
    if (rows == 0) return AMQFT_OK;
    if (!in || !out) return set_err(AMQFT_EINVAL, "null data pointer");
    try {
      ck(cudaSetDevice(P->d.device), "cudaSetDevice");
      return exec_real_inverse(P, in, out, rows, static_cast<cudaStream_t>(stream));
    } catch (...) {
      return from_exception();
    }
  }
  if (rows == 0) return AMQFT_OK;
  if (!in || !out) return set_err(AMQFT_EINVAL, "null data pointer");
  // the fused, four-step and small-CDFT kernels move rows with TMA bulk
  // copies and 16-byte vectors: their device buffers must be 16-byte aligned
  if (((P->path >= 2 && P->path <= 4) || P->path == 6) && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u))
    return set_err(AMQFT_EINVAL, "device buffers of fast-order plans must be 16-byte aligned");
  try {
    ck(cudaSetDevice(P->d.device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (P->path >= 2) {
      P->fast->exec(in, out, rows, inverse, st);
    } else if (P->d.dtype == AMQFT_F64) {
      exec_generic<double>(P, in, out, rows, inverse, st);
    } else {
      exec_generic<float>(P, in, out, rows, inverse, st);
    }
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

// Host buffers in, host buffers out: the batch moves through NSLOT device
// slots in chunks, as a three-stage pipeline (H2D copy engine | transform
// | D2H copy engine) on three streams ordered by events, so the two PCIe
// directions and the kernel overlap.  Stream-ordered with respect to
// `stream` (the caller's stream waits for the last D2H).  Host memory
// should be pinned for the copies to be asynchronous.
amqft_status amqft_exec_host_rows(amqft_plan P, const void* h_in, void* h_out, size_t rows,
                                  int inverse, void* stream) {
  if (!P) return set_err(AMQFT_EINVAL, "null plan");
  if (inverse && !inverse_defined(P))
    return set_err(AMQFT_EINVAL, "the inverse is defined for CDFT, and for RDFT / DCT / DST plans with n >= 4");
  if (rows == 0) return AMQFT_OK;
  if (!h_in || !h_out) return set_err(AMQFT_EINVAL, "null data pointer");
  try {
    std::lock_guard<std::mutex> lock(P->host_mu);
    ck(cudaSetDevice(P->d.device), "cudaSetDevice");
    const size_t row_bytes = P->c.cells * P->esize;
    if (!P->s_run) {
      // ~64 MiB per slot, at least one full wave of CTAs, at most the plan batch
      size_t r = std::max<size_t>(1, (size_t(64) << 20) / row_bytes);
      r = std::max<size_t>(r, std::min<size_t>(P->d.batch, 2 * static_cast<size_t>(P->sms)));
      P->slot_rows = std::min<size_t>(r, P->d.batch);
      for (int k = 0; k < amqft_plan_s::NSLOT; ++k) {
        ck(cudaMalloc(&P->slot[k], P->slot_rows * row_bytes), "cudaMalloc(host pipeline slot)");
        ck(cudaEventCreateWithFlags(&P->ev_h2d[k], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&P->ev_run[k], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&P->ev_d2h[k], cudaEventDisableTiming), "cudaEventCreate");
      }
      ck(cudaEventCreateWithFlags(&P->ev_in, cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaStreamCreateWithFlags(&P->s_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaStreamCreateWithFlags(&P->s_run, cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaStreamCreateWithFlags(&P->s_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
      for (int k = 0; k < amqft_plan_s::NSLOT; ++k) ck(cudaEventRecord(P->ev_d2h[k], P->s_d2h), "record");
    }
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    ck(cudaEventRecord(P->ev_in, caller), "cudaEventRecord");
    ck(cudaStreamWaitEvent(P->s_h2d, P->ev_in, 0), "wait");
    const char* hi = static_cast<const char*>(h_in);
    char* ho = static_cast<char*>(h_out);
    size_t chunk = 0;
    for (size_t r0 = 0; r0 < rows; r0 += P->slot_rows, ++chunk) {
      const size_t nr = std::min(P->slot_rows, rows - r0);
      const int k = static_cast<int>(chunk % amqft_plan_s::NSLOT);
      const size_t bytes = nr * row_bytes;
      ck(cudaStreamWaitEvent(P->s_h2d, P->ev_d2h[k], 0), "wait");           // slot free
      ck(cudaMemcpyAsync(P->slot[k], hi + r0 * row_bytes, bytes, cudaMemcpyHostToDevice, P->s_h2d),
         "cudaMemcpyAsync H2D");
      ck(cudaEventRecord(P->ev_h2d[k], P->s_h2d), "record");
      ck(cudaStreamWaitEvent(P->s_run, P->ev_h2d[k], 0), "wait");
      const amqft_status st = amqft_exec_rows(P, P->slot[k], P->slot[k], nr, inverse, P->s_run);
      if (st != AMQFT_OK) return st;
      ck(cudaEventRecord(P->ev_run[k], P->s_run), "record");
      ck(cudaStreamWaitEvent(P->s_d2h, P->ev_run[k], 0), "wait");
      ck(cudaMemcpyAsync(ho + r0 * row_bytes, P->slot[k], bytes, cudaMemcpyDeviceToHost, P->s_d2h),
         "cudaMemcpyAsync D2H");
      ck(cudaEventRecord(P->ev_d2h[k], P->s_d2h), "record");
    }
    const int last = static_cast<int>((chunk - 1) % amqft_plan_s::NSLOT);
    ck(cudaStreamWaitEvent(caller, P->ev_d2h[last], 0), "wait");
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_exec_forward(amqft_plan P, const void* in, void* out, void* stream) {
  return amqft_exec_rows(P, in, out, P ? P->d.batch : 0, 0, stream);
}

amqft_status amqft_exec_inverse(amqft_plan P, const void* in, void* out, void* stream) {
  return amqft_exec_rows(P, in, out, P ? P->d.batch : 0, 1, stream);
}

amqft_status amqft_dist_twiddle_scatter(const void* d_rows, void* const* d_dst, size_t rows, size_t n1,
                                        size_t n, size_t row0, int src_rank, int nparts, int trig_mode,
                                        void* stream) {
  if (!d_rows || !d_dst) return set_err(AMQFT_EINVAL, "null pointer");
  if (n == 0 || (n & (n - 1)) || n1 == 0 || (n1 & (n1 - 1)) || n % n1 || n > (size_t(1) << 40))
    return set_err(AMQFT_EINVAL, "n and n1 must be powers of two with n1 | n");
  if (src_rank < 0 || src_rank >= nparts) return set_err(AMQFT_EINVAL, "src_rank out of range");
  try {
    dist_twiddle_scatter(d_rows, d_dst, rows, n1, n, row0, src_rank, nparts, trig_mode,
                         static_cast<cudaStream_t>(stream));
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_dist_twiddle_scatter_direct(const void* d_rows, void* const* d_dst, size_t rows, size_t n1,
                                               size_t n, size_t row0, int nparts, int trig_mode, size_t a,
                                               void* stream) {
  if (!d_rows || !d_dst) return set_err(AMQFT_EINVAL, "null pointer");
  if (n == 0 || (n & (n - 1)) || n1 == 0 || (n1 & (n1 - 1)) || n % n1 || n > (size_t(1) << 40))
    return set_err(AMQFT_EINVAL, "n and n1 must be powers of two with n1 | n");
  try {
    dist_twiddle_scatter_direct(d_rows, d_dst, rows, n1, n, row0, nparts, trig_mode, a,
                                static_cast<cudaStream_t>(stream));
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_plan_transposed_factor(amqft_plan P, size_t* a) {
  if (!P || !a) return set_err(AMQFT_EINVAL, "null argument");
  *a = (P->path == 3 && P->fast) ? P->fast->transposed_factor() : 0;
  return AMQFT_OK;
}

amqft_status amqft_exec_rows_transposed(amqft_plan P, const void* in, void* out, size_t rows, void* stream) {
  if (!P) return set_err(AMQFT_EINVAL, "null plan");
  if (rows > P->d.batch) return set_err(AMQFT_EINVAL, "rows exceed the plan batch");
  if (P->path != 3 || !P->fast || P->fast->transposed_factor() == 0)
    return set_err(AMQFT_EINVAL, "transposed output needs a column-mode four-step plan");
  if (!in || !out) return set_err(AMQFT_EINVAL, "null data pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u)
    return set_err(AMQFT_EINVAL, "device buffers of fast-order plans must be 16-byte aligned");
  if (rows == 0) return AMQFT_OK;
  try {
    ck(cudaSetDevice(P->d.device), "cudaSetDevice");
    P->fast->exec_transposed(in, out, rows, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_dist_twiddle_scatter_t(const void* d_rows, void* const* d_dst, size_t rows, size_t n1,
                                          size_t n, size_t row0, int src_rank, int nparts, int trig_mode,
                                          size_t a, void* stream) {
  if (!d_rows || !d_dst) return set_err(AMQFT_EINVAL, "null pointer");
  if (n == 0 || (n & (n - 1)) || n1 == 0 || (n1 & (n1 - 1)) || n % n1 || n > (size_t(1) << 40))
    return set_err(AMQFT_EINVAL, "n and n1 must be powers of two with n1 | n");
  if (src_rank < 0 || src_rank >= nparts) return set_err(AMQFT_EINVAL, "src_rank out of range");
  try {
    dist_twiddle_scatter_t(d_rows, d_dst, rows, n1, n, row0, src_rank, nparts, trig_mode, a,
                           static_cast<cudaStream_t>(stream));
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_transpose_c64(const void* d_in, void* d_out, size_t mats, size_t r, size_t c,
                                 void* stream) {
  if (!d_in || !d_out) return set_err(AMQFT_EINVAL, "null pointer");
  try {
    transpose_c64(d_in, d_out, mats, r, c, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return from_exception();
  }
  return AMQFT_OK;
}

amqft_status amqft_plan_op_counts(amqft_plan P, uint64_t* out3) {
  if (!P || !out3) return set_err(AMQFT_EINVAL, "null argument");
  out3[0] = P->c.ops.adds;
  out3[1] = P->c.ops.muls;
  out3[2] = P->c.ops.bt;
  return AMQFT_OK;
}

amqft_status amqft_plan_path(amqft_plan P, int* path, int* launches) {
  if (!P) return set_err(AMQFT_EINVAL, "null plan");
  if (path) *path = P->path;
  if (launches) *launches = P->launches;
  return AMQFT_OK;
}

amqft_status amqft_plan_fourstep_factors(amqft_plan P, size_t* f3) {
  if (!P || !f3) return set_err(AMQFT_EINVAL, "null argument");
  if (P->path != 3) return set_err(AMQFT_EINVAL, "not a four-step plan");
  return fourstep_factors(P->d, f3);
}

amqft_status amqft_plan_dump(amqft_plan P, int prog, void* records, size_t cap,
                             size_t* count, uint32_t* stages, size_t cap2,
                             size_t* nstages) {
  if (!P) return set_err(AMQFT_EINVAL, "null plan");
  if (P->path >= 2) return set_err(AMQFT_EINVAL, "fused plans carry no stage program");
  if (prog < 0 || static_cast<size_t>(prog) >= P->c.progs.size())
    return set_err(AMQFT_EINVAL, "no such program");
  const SubProgram& sp = P->c.progs[prog];
  if (count) *count = sp.eis.size();
  if (records) std::memcpy(records, sp.eis.data(), std::min(cap, sp.eis.size()) * sizeof(EI));
  if (nstages) *nstages = sp.stages.size();
  if (stages)
    for (size_t s = 0; s < std::min(cap2, sp.stages.size()); ++s) {
      stages[2 * s] = sp.stages[s].ei_begin;
      stages[2 * s + 1] = sp.stages[s].ei_end;
    }
  return AMQFT_OK;
}

}  // extern "C"

namespace {

// One signal between host buffers on the current device, exact fp64 order.
amqft_status execute_host_impl(const amqft_plan_desc& d, const std::vector<double>* host_tab, const double* in,
                               double* out, int inverse, uint64_t* meter3) {
  amqft_plan P = nullptr;
  amqft_status s = create_plan(&P, &d, host_tab);
  if (s != AMQFT_OK) return s;
  const size_t bytes = P->c.cells * sizeof(double);
  void *din = nullptr, *dout = nullptr;
  try {
    ck(cudaMalloc(&din, bytes), "cudaMalloc");
    ck(cudaMalloc(&dout, bytes), "cudaMalloc");
    ck(cudaMemcpy(din, in, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    s = amqft_exec_rows(P, din, dout, 1, inverse, nullptr);
    if (s == AMQFT_OK) {
      ck(cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
      if (meter3) amqft_plan_op_counts(P, meter3);
    }
  } catch (...) {
    s = from_exception();
  }
  cudaFree(din);
  cudaFree(dout);
  amqft_plan_destroy(P);
  return s;
}

amqft_plan_desc host_desc(int variant, int function, size_t n) {
  amqft_plan_desc d{};
  d.variant = variant;
  d.function = function;
  d.n = n;
  d.batch = 1;
  d.dtype = AMQFT_F64;
  d.trig_mode = AMQFT_TRIG_TABLE;
  d.order = AMQFT_ORDER_EXACT;
  d.device = 0;
  cudaGetDevice(&d.device);
  return d;
}

}  // namespace

extern "C" {

amqft_status amqft_execute_host_constants(int variant, int function, size_t n, const double* in, double* out,
                                          const double* constants, size_t count, uint64_t* meter3) {
  if (!constants || !in || !out) return set_err(AMQFT_EINVAL, "null buffer");
  try {
    const std::vector<double> tab(constants, constants + count);
    amqft_plan_desc d = host_desc(variant, function, n);
    d.table_max_n = 4 * count;
    return execute_host_impl(d, &tab, in, out, 0, meter3);
  } catch (...) {
    return from_exception();
  }
}

amqft_status amqft_execute_host_inverse(int variant, size_t n, const double* in, double* out) {
  if (!in || !out) return set_err(AMQFT_EINVAL, "null buffer");
  return execute_host_impl(host_desc(variant, AMQFT_FN_CDFT, n), nullptr, in, out, 1, nullptr);
}

amqft_status amqft_execute_host(int variant, int function, size_t n, const double* in,
                                double* out, int trig_mode, size_t table_max_n,
                                int corrupt_constants, uint64_t* meter3) {
  amqft_plan_desc d = host_desc(variant, function, n);
  d.trig_mode = trig_mode;
  d.table_max_n = table_max_n;
  d.corrupt_constants = corrupt_constants;
  return execute_host_impl(d, nullptr, in, out, 0, meter3);
}

amqft_status amqft_device_synchronize(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return set_err(AMQFT_ECUDA, "cudaSetDevice failed");
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_err(AMQFT_ECUDA, cudaGetErrorString(e));
  return AMQFT_OK;
}

}  // extern "C"
