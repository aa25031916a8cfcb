// dist.cpp -- the distributed four-step behind the C ABI (BASELINE config 5;
// SURVEY §8(e)): one plan per rank owning its NCCL communicator, so a C /
// C++ caller (the reference is single-process, src/variants.cpp:404) has a
// route to one huge transform over P GPUs without Python.
//
// n = n1 n2, x viewed as M[n1][n2] = x[n2 i1 + i2].  Rank p holds the column
// slab i2 in [p n2/P, (p+1) n2/P) as rows of length n1 (interleaved fp32
// complex).  amqft_dist_exec_forward:
//   1. the rank's n2/P length-n1 AM-QFTs (a fused / four-step plan; a
//      column-mode four-step leaves its rows transposed and step 2 reads
//      them in that order);
//   2. one kernel: twiddle w_N^(i2 k1) and scatter by k1-slab into P send
//      slots;
//   3. the exchange: grouped ncclSend / ncclRecv, one slot to every rank
//      (the all-to-all transpose over NVLink);
//   4. transpose [n2][n1/P] -> [n1/P][n2];
//   5. the n1/P length-n2 AM-QFTs.
// The output of rank p is X[k1 + n1 k2] for k1 in [p n1/P, (p+1) n1/P) as
// rows k1 of length n2 (no second all-to-all).  Same layouts and kernels as
// paper_1404_1810_b200.dist.DistFourStep (which drives them over
// torch.distributed).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring a copy
// already loaded in the process, e.g. torch's) so the library has no link
// dependency on it; only amqft_dist_* need it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/amqft_b200.h"

namespace amqft_b200 {
void set_last_error(const std::string& m);
}

namespace {

using amqft_b200::set_last_error;

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      return fp != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") && sym(api.comm_init_rank, "ncclCommInitRank") &&
             sym(api.comm_destroy, "ncclCommDestroy") && sym(api.group_start, "ncclGroupStart") &&
             sym(api.group_end, "ncclGroupEnd") && sym(api.send, "ncclSend") && sym(api.recv, "ncclRecv") &&
             sym(api.error_string, "ncclGetErrorString");
    if (!api.ok) api.why = "libnccl.so.2 lacks a symbol the distributed plan needs";
  });
  return api;
}

amqft_status err(amqft_status s, const std::string& m) {
  set_last_error(m);
  return s;
}

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().error_string(r));
}
void cck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void ack(amqft_status s) {
  if (s != AMQFT_OK) throw std::runtime_error(amqft_last_error());
}

bool fast_f32_size(size_t n) { return n >= 2 && n <= (size_t(1) << 26) && (n & (n - 1)) == 0; }

}  // namespace

struct amqft_dist_plan_s {
  int nparts = 1, rank = 0, device = 0, trig = AMQFT_TRIG_TABLE;
  size_t n = 0, n1 = 0, n2 = 0, rows1 = 0, w = 0, a_t = 0;
  amqft_plan p1 = nullptr, p2 = nullptr;
  void *send = nullptr, *recv = nullptr, *b = nullptr;
  ncclComm_t comm = nullptr;

  ~amqft_dist_plan_s() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (comm) nccl().comm_destroy(comm);
    amqft_plan_destroy(p1);
    amqft_plan_destroy(p2);
    for (void* p : {send, recv, b})
      if (p) cudaFree(p);
    cudaSetDevice(cur);
  }
};

extern "C" {

amqft_status amqft_dist_unique_id(void* id128) {
  if (!id128) return err(AMQFT_EINVAL, "null id buffer");
  const Nccl& api = nccl();
  if (!api.ok) return err(AMQFT_ENCCL, api.why);
  ncclUniqueId id;
  const ncclResult_t r = api.get_unique_id(&id);
  if (r != ncclSuccess) return err(AMQFT_ENCCL, std::string("ncclGetUniqueId: ") + api.error_string(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof id);
  return AMQFT_OK;
}

amqft_status amqft_dist_plan_create(amqft_dist_plan* out, int variant, size_t n, int nparts, int rank, int device,
                                    int trig_mode, const void* id128) {
  if (!out) return err(AMQFT_EINVAL, "null plan pointer");
  *out = nullptr;
  if (nparts < 1 || rank < 0 || rank >= nparts) return err(AMQFT_EINVAL, "rank must lie in [0, nparts)");
  if (n == 0 || (n & (n - 1)) != 0) return err(AMQFT_EINVAL, "n must be a power of two");
  if (nparts > 1 && !id128) return err(AMQFT_EINVAL, "nparts > 1 needs an NCCL unique id (amqft_dist_unique_id)");
  auto P = std::make_unique<amqft_dist_plan_s>();
  P->nparts = nparts;
  P->rank = rank;
  P->device = device;
  P->trig = trig_mode;
  P->n = n;
  // split: n2 a fused-kernel size (the rows after the exchange), n1 any
  // fp32 fast-order size, both divisible by the ranks (dist.py dist_split)
  for (size_t n2 : {size_t(4096), size_t(8192), size_t(2048), size_t(1024)}) {
    const size_t n1 = n / n2;
    if (n1 * n2 == n && fast_f32_size(n1) && n1 % nparts == 0 && n2 % nparts == 0) {
      P->n1 = n1;
      P->n2 = n2;
      break;
    }
  }
  if (!P->n1) return err(AMQFT_EINVAL, "no distributed four-step split for this n and rank count");
  P->rows1 = P->n2 / nparts;
  P->w = P->n1 / nparts;
  try {
    cck(cudaSetDevice(device), "cudaSetDevice");
    amqft_plan_desc d{};
    d.variant = variant;
    d.function = AMQFT_FN_CDFT;
    d.dtype = AMQFT_F32;
    d.trig_mode = trig_mode;
    d.order = AMQFT_ORDER_FAST;
    d.device = device;
    d.n = P->n1;
    d.batch = P->rows1;
    ack(amqft_plan_create_transposable(&P->p1, &d));
    d.n = P->n2;
    d.batch = P->w;
    ack(amqft_plan_create(&P->p2, &d));
    size_t fa = 0;
    ack(amqft_plan_transposed_factor(P->p1, &fa));
    if (fa && fa % 32 == 0 && (P->n1 / fa) % 32 == 0 && P->w % 32 == 0 && P->rows1 <= 65535) P->a_t = fa;
    const size_t slot = P->rows1 * P->w * 2 * sizeof(float);
    cck(cudaMalloc(&P->send, slot * nparts), "cudaMalloc send slots");
    cck(cudaMalloc(&P->recv, slot * nparts), "cudaMalloc receive slots");
    cck(cudaMalloc(&P->b, slot * nparts), "cudaMalloc transposed rows");
    if (id128) {   // the communicator (a one-rank plan may still exchange through NCCL)
      const Nccl& api = nccl();
      if (!api.ok) return err(AMQFT_ENCCL, api.why);
      ncclUniqueId id;
      std::memcpy(&id, id128, sizeof id);
      nck(api.comm_init_rank(&P->comm, nparts, id, rank), "ncclCommInitRank");
    }
  } catch (const NcclError& e) {
    return err(AMQFT_ENCCL, e.what());
  } catch (const std::exception& e) {
    const std::string m = e.what();
    return err(m.find("out of memory") != std::string::npos ? AMQFT_ENOMEM : AMQFT_ECUDA, m);
  }
  *out = P.release();
  return AMQFT_OK;
}

amqft_status amqft_dist_plan_shape(amqft_dist_plan P, size_t* n1, size_t* n2, size_t* rows_in, size_t* rows_out) {
  if (!P) return err(AMQFT_EINVAL, "null plan");
  if (n1) *n1 = P->n1;
  if (n2) *n2 = P->n2;
  if (rows_in) *rows_in = P->rows1;
  if (rows_out) *rows_out = P->w;
  return AMQFT_OK;
}

amqft_status amqft_dist_exec_forward(amqft_dist_plan P, void* d_in, void* d_out, void* stream) {
  if (!P || !d_in || !d_out) return err(AMQFT_EINVAL, "null plan or buffer");
  try {
    cck(cudaSetDevice(P->device), "cudaSetDevice");
    const size_t slot = P->rows1 * P->w * 2 * sizeof(float);
    const int parts = P->nparts;
    // 1. local length-n1 transforms (in place)
    if (P->a_t)
      ack(amqft_exec_rows_transposed(P->p1, d_in, d_in, P->rows1, stream));
    else
      ack(amqft_exec_rows(P->p1, d_in, d_in, P->rows1, 0, stream));
    // one rank, no communicator: no exchange to make -- the scatter writes each value to its final
    // place in the row buffer (scatter + transpose in one kernel), then the length-n2 transforms
    const size_t a1 = P->a_t ? P->a_t : 1;
    if (!P->comm && parts == 1 && P->rows1 % 32 == 0 && (P->n1 / a1) % 32 == 0 && P->rows1 / 32 <= 65535) {
      void* rows[1] = {P->b};
      ack(amqft_dist_twiddle_scatter_direct(d_in, rows, P->rows1, P->n1, P->n, 0, 1, P->trig, P->a_t, stream));
      ack(amqft_exec_rows(P->p2, P->b, d_out, P->w, 0, stream));
      return AMQFT_OK;
    }
    // 2. twiddle + scatter by k1-slab: into the send slots, or with no
    //    communicator straight into the receive slots
    void* dst = P->comm ? P->send : P->recv;
    std::vector<void*> slots(parts);
    for (int q = 0; q < parts; ++q) slots[q] = static_cast<char*>(dst) + q * slot;
    const size_t row0 = static_cast<size_t>(P->rank) * P->rows1;
    if (P->a_t)
      ack(amqft_dist_twiddle_scatter_t(d_in, slots.data(), P->rows1, P->n1, P->n, row0, 0, parts, P->trig, P->a_t,
                                       stream));
    else
      ack(amqft_dist_twiddle_scatter(d_in, slots.data(), P->rows1, P->n1, P->n, row0, 0, parts, P->trig, stream));
    // 3. the exchange: slot q to rank q, rank q's slot for us into recv slot q
    if (P->comm) {
      const Nccl& api = nccl();
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      nck(api.group_start(), "ncclGroupStart");
      for (int q = 0; q < parts; ++q) {
        nck(api.send(static_cast<char*>(P->send) + q * slot, slot / sizeof(float), ncclFloat, q, P->comm, st),
            "ncclSend");
        nck(api.recv(static_cast<char*>(P->recv) + q * slot, slot / sizeof(float), ncclFloat, q, P->comm, st),
            "ncclRecv");
      }
      nck(api.group_end(), "ncclGroupEnd");
    }
    // 4. [n2][n1/P] -> [n1/P][n2];  5. length-n2 transforms
    ack(amqft_transpose_c64(P->recv, P->b, 1, P->n2, P->w, stream));
    ack(amqft_exec_rows(P->p2, P->b, d_out, P->w, 0, stream));
  } catch (const NcclError& e) {
    return err(AMQFT_ENCCL, e.what());
  } catch (const std::exception& e) {
    return err(AMQFT_ECUDA, e.what());
  }
  return AMQFT_OK;
}

amqft_status amqft_dist_plan_destroy(amqft_dist_plan P) {
  delete P;
  return AMQFT_OK;
}

}  // extern "C"
