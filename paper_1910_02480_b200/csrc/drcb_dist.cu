// drcb_dist.cu — NCCL plumbing for data-parallel training over NVLink /
// NVSwitch. libnccl.so.2 is opened at first use (dlopen), so the library has
// no link-time NCCL dependency and shares the process's NCCL instance with
// torch when torch already loaded it.
#include <dlfcn.h>
#include <mutex>
#include <nccl.h>

#include <cstring>
#include <string>

#include "drcb_internal.h"

namespace drcb {
namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;  // several host threads may build communicators
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (n.h) {
      n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
      n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(n.h, "ncclCommInitRank"));
      n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
      n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(n.h, "ncclCommDestroy"));
      n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
    }
  });
  if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_reduce || !n.comm_destroy)
    return nullptr;
  return &n;
}

int nccl_fail(ncclResult_t r, const char* where) {
  Nccl* n = nccl();
  std::string m = std::string(where) + ": " + (n && n->error_string ? n->error_string(r) : "nccl error");
  return fail(DRCB_ENCCL, m);
}

}  // namespace

// all-reduce (sum) on the caller's stream; comm == NULL is a no-op
int allreduce_sum(void* comm, void* buf, size_t count, int is_double, cudaStream_t st) {
  if (!comm) return 0;
  Nccl* n = nccl();
  if (!n) return fail(DRCB_ENCCL, "libnccl.so.2 not available");
  ncclResult_t r = n->all_reduce(buf, buf, count, is_double ? ncclFloat64 : ncclFloat32, ncclSum,
                                 static_cast<ncclComm_t>(comm), st);
  return r == ncclSuccess ? 0 : nccl_fail(r, "ncclAllReduce");
}

}  // namespace drcb

using namespace drcb;

extern "C" int drcb_nccl_unique_id(void* out128) {
  if (!out128) return fail(DRCB_ECONTRACT, "drcb_nccl_unique_id: null buffer");
  Nccl* n = nccl();
  if (!n) return fail(DRCB_ENCCL, "libnccl.so.2 not available");
  ncclUniqueId id;
  ncclResult_t r = n->get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

extern "C" int drcb_nccl_comm_create(const void* id128, int32_t world, int32_t rank, void** comm) {
  if (!id128 || !comm) return fail(DRCB_ECONTRACT, "drcb_nccl_comm_create: null argument");
  Nccl* n = nccl();
  if (!n) return fail(DRCB_ENCCL, "libnccl.so.2 not available");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = n->comm_init_rank(&c, world, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return 0;
}

extern "C" int drcb_nccl_comm_destroy(void* comm) {
  if (!comm) return 0;
  Nccl* n = nccl();
  if (!n) return fail(DRCB_ENCCL, "libnccl.so.2 not available");
  ncclResult_t r = n->comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? 0 : nccl_fail(r, "ncclCommDestroy");
}

extern "C" int drcb_allreduce_sum_f32(void* comm, float* buf, int64_t n, void* stream) {
  return allreduce_sum(comm, buf, size_t(n), 0, static_cast<cudaStream_t>(stream));
}
