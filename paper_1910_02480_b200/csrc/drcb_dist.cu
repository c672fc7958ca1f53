// drcb_dist.cu — NCCL plumbing for data-parallel training over NVLink /
// NVSwitch. libnccl.so.2 is opened at first use (dlopen), so the library has
// no link-time NCCL dependency and shares the process's NCCL instance with
// torch when torch already loaded it.
#include <dlfcn.h>
#include <condition_variable>
#include <mutex>
#include <vector>
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

// ---------------------------------------------------------------------------
// Loopback communicator: `world` ranks as host threads of ONE process (e.g.
// two half-batch trainers on one GPU). An all-reduce synchronises the
// calling rank's stream, meets the other ranks at a barrier, and rank 0 sums
// the buffers in rank order ((b0 + b1) + b2 ...) and writes the sum back to
// every rank: the SyncBN statistics and the gradient all-reduce of a
// data-parallel step, with the same reduction hooks NCCL serves, testable on
// a single GPU (and bit-identical on every rank).
struct Loopback {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void*> bufs;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // all ranks meet; the last to arrive runs `f` before releasing the others
  template <class F>
  void barrier(F&& f) {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      f();
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
struct LoopbackRank {
  Loopback* lb;
  int rank;
};

__global__ void k_add_f32(float* a, const float* b, int64_t n) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i] += b[i];
}
__global__ void k_add_f64(double* a, const double* b, int64_t n) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i] += b[i];
}

}  // namespace drcb

using namespace drcb;

extern "C" int drcb_loopback_create(int32_t world, void** out) {
  if (world < 1 || !out) return fail(DRCB_ECONTRACT, "drcb_loopback_create: bad arguments");
  Loopback* L = new Loopback();
  L->world = world;
  L->bufs.assign(world, nullptr);
  *out = L;
  return 0;
}

extern "C" int drcb_loopback_rank(void* lb, int32_t rank, void** ctx) {
  Loopback* L = static_cast<Loopback*>(lb);
  if (!L || !ctx || rank < 0 || rank >= L->world) return fail(DRCB_ECONTRACT, "drcb_loopback_rank: bad arguments");
  *ctx = new LoopbackRank{L, rank};
  return 0;
}

extern "C" void drcb_loopback_destroy(void* lb, void** ranks, int32_t n) {
  for (int i = 0; i < n; ++i) delete static_cast<LoopbackRank*>(ranks[i]);
  Loopback* L = static_cast<Loopback*>(lb);
  if (L && L->scratch) cudaFree(L->scratch);
  delete L;
}

// the DrcbReduceFn of a loopback rank (ctx from drcb_loopback_rank)
extern "C" int drcb_loopback_reduce(void* ctx, void* buf, int64_t count, int32_t is_double, void* stream) {
  LoopbackRank* R = static_cast<LoopbackRank*>(ctx);
  Loopback* L = R->lb;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(DRCB_ECUDA, "loopback: stream sync");
  const size_t bytes = size_t(count) * (is_double ? 8 : 4);
  int rc = 0;
  L->bufs[R->rank] = buf;
  L->barrier([&] {
    // the last rank in: sum in rank order into scratch, write back to every rank
    if (L->scratch_bytes < bytes) {
      if (L->scratch) cudaFree(L->scratch);
      L->scratch = nullptr;
      L->scratch_bytes = 0;
      if (cudaMalloc(&L->scratch, bytes) != cudaSuccess) {
        rc = fail(DRCB_ECUDA, "loopback: scratch");
        return;
      }
      L->scratch_bytes = bytes;
    }
    cudaMemcpy(L->scratch, L->bufs[0], bytes, cudaMemcpyDeviceToDevice);
    const unsigned nb = unsigned((count + 255) / 256);
    for (int r = 1; r < L->world; ++r) {
      if (is_double)
        k_add_f64<<<nb, 256>>>(static_cast<double*>(L->scratch), static_cast<const double*>(L->bufs[r]), count);
      else
        k_add_f32<<<nb, 256>>>(static_cast<float*>(L->scratch), static_cast<const float*>(L->bufs[r]), count);
    }
    for (int r = 0; r < L->world; ++r) cudaMemcpy(L->bufs[r], L->scratch, bytes, cudaMemcpyDeviceToDevice);
    if (cudaDeviceSynchronize() != cudaSuccess) rc = fail(DRCB_ECUDA, "loopback: reduce");
  });
  return rc;
}

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

// byte copy between any two addresses (host or device, cudaMemcpyDefault) on
// `stream`, synchronised: the host-staged reduction hooks move a device
// buffer to the host and back with it
extern "C" int drcb_copy_sync(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return 0;
  if (!dst || !src) return fail(DRCB_ECONTRACT, "drcb_copy_sync: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DRCB_CUDA(cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDefault, st));
  DRCB_CUDA(cudaStreamSynchronize(st));
  return 0;
}
