// drcb_internal.h — host-side handle types shared by the C-ABI translation
// units. Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <string>
#include <vector>

#include "../../include/drcb.h"
#include "drcb_scene.cuh"

namespace drcb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
void count_launch(int n = 1);
void keep_pool_memory();
int allreduce_sum(void* comm, void* buf, size_t count, int is_double, cudaStream_t st);

// Per-device launch state: kernel attributes and SM counts are
// properties of a device, and several host threads may launch on several
// devices. A flag word per kernel remembers which devices are set up; the
// attribute call is idempotent, so two threads racing on a first launch
// both set it and neither launches before its own call returned.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
struct DeviceFlags {
  std::atomic<uint64_t> bits{0};
  bool test(int dev) const { return (bits.load(std::memory_order_acquire) >> (dev & 63)) & 1; }
  void set(int dev) { bits.fetch_or(uint64_t(1) << (dev & 63), std::memory_order_release); }
};
// Programmatic dependent launch: the tensor-core and training kernels are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization and begin
// with pdl_wait() (griddepcontrol.wait: returns once the preceding kernel of
// the stream has completed and its writes are visible), so a kernel's launch
// and block scheduling overlap its predecessor's tail instead of following
// it. Every kernel launched this way waits before touching memory; a kernel
// launched plainly executes the wait as a no-op. DRCB_NO_PDL turns it off.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
inline bool pdl_enabled() {
  static const bool on = getenv("DRCB_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
template <class K>
inline void smem_attr_once(DeviceFlags& f, K kern, int bytes) {
  const int dev = current_device();
  if (!f.test(dev)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    f.set(dev);
  }
}
// SM count of the current device (cached per device)
inline int sm_count() {
  static std::atomic<int> cache[64];
  const int dev = current_device();
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

#define DRCB_CUDA(call)                                      \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return ::drcb::cuda_fail(_e, #call); \
  } while (0)

struct SceneStats {
  int64_t n_prims = 0, n_nodes = 0, n_leaves = 0, max_depth = 0, n_lights = 0, bytes = 0, n_refs = 0;
};

template <typename R>
int launch_pt_frame(const DevScene& S, const DevCamera& C, const DrcbRenderCfg& cfg, int spp,
                    int tile, R* image, int64_t* nonfinite, cudaStream_t st);
template <typename R>
int launch_reference_map(const DevScene& S, const DrcbRenderCfg& cfg, const R* pos, const R* nrm,
                         uint64_t key, int ref_spp, R* out, int64_t* nonfinite, cudaStream_t st);
}  // namespace drcb

struct DrcbScene {
  drcb::DevScene dev;          // device pointers (owned)
  std::vector<void*> allocs;   // device allocations to free
  drcb::SceneStats stats;
  int device = 0;
};

namespace drcb {
DevCamera make_camera(const DrcbCamera& c);

// stage launchers (drcb_render.cu)
template <typename R>
int launch_intersect(const DevScene& S, const R* O, const R* D, int64_t n, const R* tmin,
                     const R* tmax, int record, uint8_t* hit, R* t, int64_t* prim, int32_t* mat,
                     R* pos, R* nrm, cudaStream_t st);
// fp32 traversal of fp64 rays with fp64 near-tie refinement (DRCB_PREC_MIXED)
int launch_intersect_mixed(const DevScene& S, const double* O, const double* D, int64_t n,
                           const double* tmin, const double* tmax, int record, uint8_t* hit,
                           double* t, int64_t* prim, int32_t* mat, double* pos, double* nrm,
                           cudaStream_t st);
template <typename R>
int launch_primary_chain(const DevScene& S, const R* O, const R* D, int64_t n,
                         const DrcbGBuffer& gb, cudaStream_t st);
template <typename R>
int launch_li_direct(const DevScene& S, const DrcbRenderCfg& cfg, const R* O, const R* D,
                     const uint64_t* pix, const uint64_t* smp, int64_t n, int include_bg, R* L,
                     int64_t* nonfinite, cudaStream_t st);
template <typename R>
int launch_trace_radiance(const DevScene& S, const DrcbRenderCfg& cfg, const R* O, const R* D,
                          const uint64_t* pix, const uint64_t* smp, int64_t n, int max_depth,
                          int skip_first, int rr_start, R* L, int64_t* nonfinite,
                          cudaStream_t st);
template <typename R>
int launch_gbuffer_direct(const DevScene& S, const DevCamera& C, const DrcbRenderCfg& cfg,
                          int tile, const DrcbGBuffer& gb, R* direct, int64_t* nonfinite,
                          cudaStream_t st);
// map rays + normalisation; live (n,) optional mask (nullptr = all live)
template <typename R>
int launch_render_stacks(const DevScene& S, const DrcbRenderCfg& cfg, const R* pos, const R* nrm,
                         const uint64_t* keys, const uint8_t* live, int64_t n, float* stacks,
                         R* s_r, R* s_d, R* frames, int64_t* nonfinite, cudaStream_t st,
                         void* nhwc = nullptr, int nhwc_kind = 0, int cpad = 0);
template <typename R>
int launch_shade(const DevScene& S, const DrcbRenderCfg& cfg, const float* pred, const R* s_r,
                 const R* frames, const R* wo, const int32_t* mat, const uint64_t* keys,
                 const uint8_t* live, int64_t n, R* L, cudaStream_t st);
template <typename R>
int launch_interp_composite(const DevScene& S, int W, int H, const DrcbGBuffer& gb,
                            const int32_t* e_px, const int32_t* e_py, const R* e_n,
                            const R* e_rad, int64_t m, const int* m_dev, int r,
                            const R* direct, R* image, cudaStream_t st);
template <typename R>
int launch_pt_frame(const DevScene& S, const DevCamera& C, const DrcbRenderCfg& cfg, int spp,
                    int tile, R* image, int64_t* nonfinite, cudaStream_t st);
template <typename R>
int launch_reference_map(const DevScene& S, const DrcbRenderCfg& cfg, const R* pos, const R* nrm,
                         uint64_t key, int ref_spp, R* out, int64_t* nonfinite, cudaStream_t st);
}  // namespace drcb
