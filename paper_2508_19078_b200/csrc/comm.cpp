// comm.cpp — C1: the statistics all-reduce across the GPUs of one box.
//
// Activation frequency = activated tokens / total tokens.  With
// the profiling tokens sharded over the GPUs (data parallel),
// the only exchange is the sum of the int64 histograms hist[L][E]: one
// ncclAllReduce(int64, sum), in place, over NVLink/NVSwitch.  Integer sums are
// exact and order-free, so the result equals the single-GPU histogram bit for
// bit.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"), preferring the
// copy torch already loaded into the process (RTLD_NOLOAD), so libflux never
// mixes two NCCL builds in one process.  Only types come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>

#include <mutex>

#include "internal.h"

struct flux_comm {
  ncclComm_t comm;
};

namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  bool ok = false;
};
NcclApi g_api;
std::once_flag g_once;

const NcclApi& api() {
  std::call_once(g_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_api.get_unique_id = (decltype(g_api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    g_api.comm_init_rank = (decltype(g_api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    g_api.all_reduce = (decltype(g_api.all_reduce))dlsym(h, "ncclAllReduce");
    g_api.comm_destroy = (decltype(g_api.comm_destroy))dlsym(h, "ncclCommDestroy");
    g_api.ok = g_api.get_unique_id && g_api.comm_init_rank && g_api.all_reduce && g_api.comm_destroy;
  });
  return g_api;
}
}  // namespace

extern "C" {

flux_status flux_comm_unique_id(void* out) {
  if (!out) return FLUX_E_INVALID;
  const NcclApi& a = api();
  if (!a.ok) return FLUX_E_NCCL;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return FLUX_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  __builtin_memcpy(out, &id, sizeof(id));
  return FLUX_OK;
}

flux_status flux_comm_init(flux_comm** out, const void* uid, int32_t nranks, int32_t rank) {
  if (!out || !uid || nranks < 1 || rank < 0 || rank >= nranks) return FLUX_E_INVALID;
  const NcclApi& a = api();
  if (!a.ok) return FLUX_E_NCCL;
  ncclUniqueId id;
  __builtin_memcpy(&id, uid, sizeof(id));
  flux_comm* c = (flux_comm*)calloc(1, sizeof(flux_comm));
  if (!c) return FLUX_E_INVALID;
  if (a.comm_init_rank(&c->comm, nranks, id, rank) != ncclSuccess) {
    free(c);
    return FLUX_E_NCCL;
  }
  *out = c;
  return FLUX_OK;
}

flux_status flux_reduce_stats(flux_comm* c, int64_t* hist, size_t count, void* stream) {
  if (!c || (!hist && count)) return FLUX_E_INVALID;
  if (count == 0) return FLUX_OK;
  const NcclApi& a = api();
  if (!a.ok) return FLUX_E_NCCL;
  if (a.all_reduce(hist, hist, count, ncclInt64, ncclSum, c->comm, (cudaStream_t)stream) != ncclSuccess)
    return FLUX_E_NCCL;
  return FLUX_OK;
}

flux_status flux_comm_destroy(flux_comm* c) {
  if (!c) return FLUX_OK;
  const NcclApi& a = api();
  flux_status st = FLUX_OK;
  if (a.ok && a.comm_destroy(c->comm) != ncclSuccess) st = FLUX_E_NCCL;
  free(c);
  return st;
}

}  // extern "C"
