// drcb_capi.cu — extern "C" entry points of libdrcb.so (include/drcb.h) and
// the whole-frame driver drcb_render_drc (drc/cache.py:377-470).
#include <cub/cub.cuh>
#include <atomic>
#include <cstring>
#include <string>

#include "drcb_net.h"

namespace drcb {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return DRCB_ECUDA;
}

int forward_f32(const NetImpl& net, const float* x, float* y, int64_t n, cudaStream_t st);
int forward_tc(NetImpl& net, const float* x, float* y, int64_t n, int mode, cudaStream_t st);
int forward_tc_nhwc(NetImpl& net, const void* x_nhwc, float* y, int64_t n, int mode,
                    cudaStream_t st);
int tc_input_channels(int mode);

int forward_f32_chunked(const NetImpl& net, const float* x, float* y, int64_t n, cudaStream_t st) {
  for (int64_t done = 0; done < n;) {
    int64_t c = n - done < 2048 ? n - done : 2048;
    int rc = forward_f32(net, x + done * 7 * 1024, y + done * 3 * 1024, c, st);
    if (rc) return rc;
    done += c;
  }
  return 0;
}

namespace {

cudaStream_t S_(void* s) { return static_cast<cudaStream_t>(s); }

int check_precision(int p) {
  if (p != 32 && p != 64) return fail(DRCB_ECONFIG, "precision must be 32 or 64");
  return 0;
}

int check_cfg(const DrcbRenderCfg* c) {
  if (!c) return fail(DRCB_ECONTRACT, "null render config");
  if (check_precision(c->precision)) return DRCB_ECONFIG;
  if (c->direct_spp < 1 || c->max_path_depth < 1 || c->rr_start < 1 || c->tile < 1)
    return fail(DRCB_ECONFIG, "direct_spp, max_path_depth, rr_start, tile must be >= 1");
  if (c->mis_samples < 2) return fail(DRCB_ECONFIG, "mis_samples must be >= 2");
  if (c->sampler_kind != 0 && c->sampler_kind != 1)
    return fail(DRCB_ECONFIG, "unknown sampler kind");
  return 0;
}

// gather cache-point hit data from the G-buffer (cache.py:211-220, 239-244)
template <typename R>
__global__ void k_gather_points(DrcbGBuffer gb, int W, const int32_t* px, const int32_t* py,
                                int64_t n, R* pos, R* nrm, R* wo, int32_t* mat, uint8_t* live) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t q = int64_t(py[i]) * W + px[i];
  bool f = gb.found[q];
  live[i] = f;
  const R* P = static_cast<const R*>(gb.position) + 3 * q;
  const R* N = static_cast<const R*>(gb.normal) + 3 * q;
  const R* D = static_cast<const R*>(gb.direction) + 3 * q;
  for (int k = 0; k < 3; ++k) {
    pos[3 * i + k] = P[k];
    nrm[3 * i + k] = N[k];
    wo[3 * i + k] = -D[k];
  }
  mat[i] = f ? gb.mat[q] : 0;
}

// stable compaction of live points into the entry pool after the *base
// entries already there (append order = task order, cache.py:183-190, 450-452)
template <typename R>
__global__ void k_scatter_entries(const uint8_t* live, const int* rank, int64_t n, const int* base,
                                  const int32_t* px, const int32_t* py, const R* nrm, const R* L,
                                  int32_t* epx, int32_t* epy, R* en, R* erad, const R* pos,
                                  const R* gthr, int W, R* epos, R* ethr) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !live[i]) return;
  const int j = *base + rank[i];
  const int64_t pix = int64_t(py[i]) * W + px[i];
  epx[j] = px[i];
  epy[j] = py[i];
  for (int k = 0; k < 3; ++k) {
    en[3 * j + k] = nrm[3 * i + k];
    erad[3 * j + k] = L[3 * i + k];
    epos[3 * j + k] = pos[3 * i + k];  // DrcState.entries (cache.py:196-201)
    ethr[3 * j + k] = gthr[3 * pix + k];
  }
}

__global__ void k_u8_to_int(const uint8_t* a, int* b, int64_t n) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_entry_count(const int* rank, const uint8_t* live, int64_t n, int* m) {
  *m += n > 0 ? rank[n - 1] + int(live[n - 1]) : 0;
}

// Per-frame stage timing (CUDA events on the frame's stream; read only when
// the caller asks for telemetry, so the frame itself never blocks the host).
struct StageEvents {
  cudaEvent_t ev[6] = {};
  bool on = false;
  void create() {
    for (auto& e : ev) cudaEventCreate(&e);
    on = true;
  }
  void rec(int i, cudaStream_t st) {
    if (on) cudaEventRecord(ev[i], st);
  }
  float ms(int a, int b) {
    float t = 0.f;
    if (on) cudaEventElapsedTime(&t, ev[a], ev[b]);
    return t;
  }
  ~StageEvents() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
};

// A frame in progress (drc/cache.py:377-470 as a resumable object): the
// G-buffer and direct pass are computed once (begin); cache points are then
// evaluated in any number of submissions (add_points: maps -> network ->
// shade -> append to the entry pool in submission order, cache.py:183-190,
// 436-452); composite interpolates the entries so far with a pass spacing r
// and adds the direct layer (cache.py:283-345, 463). Everything is
// stream-ordered; nothing synchronises the host except `info`.
template <typename R>
struct FrameCtx {
  const DevScene* S = nullptr;
  DrcbNet* net = nullptr;
  DevCamera C{};
  DrcbRenderCfg cfg{};
  int net_mode = 0;
  int W = 0, H = 0;
  int64_t npx = 0, cap = 0, points = 0;
  uint8_t* fb = nullptr;    // frame buffers (G-buffer, direct, counters)
  uint8_t* pool = nullptr;  // entry pool (cap entries)
  DrcbGBuffer gb{};
  R* direct = nullptr;
  int64_t* d_nf = nullptr;  // non-finite samples
  int* d_m = nullptr;       // entries so far
  int32_t *epx = nullptr, *epy = nullptr;
  R *en = nullptr, *erad = nullptr, *epos = nullptr, *ethr = nullptr;
  StageEvents* E = nullptr;  // stage timing (single-submission frames)

  int begin(cudaStream_t st) {
    keep_pool_memory();
    npx = int64_t(W) * H;
    size_t bytes = npx * (2 + 4 + sizeof(R) * 16) + 256;
    DRCB_CUDA(cudaMallocAsync((void**)&fb, bytes, st));
    uint8_t* cur = fb;
    auto take = [&](size_t b) {
      uint8_t* p = cur;
      cur += (b + 15) & ~size_t(15);
      return p;
    };
    direct = (R*)take(npx * 3 * sizeof(R));
    gb.position = take(npx * 3 * sizeof(R));
    gb.normal = take(npx * 3 * sizeof(R));
    gb.throughput = take(npx * 3 * sizeof(R));
    gb.direction = take(npx * 3 * sizeof(R));
    gb.t_total = take(npx * sizeof(R));
    gb.mat = (int32_t*)take(npx * 4);
    gb.found = take(npx);
    gb.escaped = take(npx);
    d_nf = (int64_t*)take(8);
    d_m = (int*)take(4);
    DRCB_CUDA(cudaMemsetAsync(d_nf, 0, 8, st));
    DRCB_CUDA(cudaMemsetAsync(d_m, 0, 4, st));
    if (cap > 0) {
      DRCB_CUDA(cudaMallocAsync((void**)&pool, size_t(cap) * (8 + 12 * sizeof(R)) + 64, st));
      cur = pool;
      epx = (int32_t*)take(cap * 4);
      epy = (int32_t*)take(cap * 4);
      en = (R*)take(cap * 3 * sizeof(R));
      erad = (R*)take(cap * 3 * sizeof(R));
      epos = (R*)take(cap * 3 * sizeof(R));
      ethr = (R*)take(cap * 3 * sizeof(R));
    }
    DrcbRenderCfg dcfg = cfg;
    dcfg.include_background = 0;  // escaped chains carry the env in the indirect layer
    if (E) E->rec(0, st);
    int rc = launch_gbuffer_direct<R>(*S, C, dcfg, cfg.tile, gb, direct, d_nf, st);
    if (E) E->rec(1, st);
    return rc;
  }

  // evaluate np_ cache points (host arrays, budget order) and append the
  // live ones to the entry pool
  int add_points(const int32_t* px_h, const int32_t* py_h, const uint64_t* keys_h, int64_t np_,
                 cudaStream_t st) {
    if (np_ <= 0) return 0;
    if (points + np_ > cap) return fail(DRCB_ECONTRACT, "frame: more cache points than reserved");
    points += np_;
    size_t pbytes = np_ * (4 * 8 + 8 + 1 + sizeof(R) * (3 * 4 + 2 + 9)) + 32 * 24 +
                    np_ * size_t(7 + 3) * 1024 * 4;
    uint8_t* pb = nullptr;
    DRCB_CUDA(cudaMallocAsync((void**)&pb, pbytes, st));
    uint8_t* cur = pb;
    auto take = [&](size_t b) {
      uint8_t* p = cur;
      cur += (b + 15) & ~size_t(15);
      return p;
    };
    int32_t* px = (int32_t*)take(np_ * 4);
    int32_t* py = (int32_t*)take(np_ * 4);
    uint64_t* keys = (uint64_t*)take(np_ * 8);
    int32_t* mat = (int32_t*)take(np_ * 4);
    uint8_t* live = take(np_);
    int* rank = (int*)take(np_ * 4);
    int* flags = (int*)take(np_ * 4);
    R* pos = (R*)take(np_ * 3 * sizeof(R));
    R* nrm = (R*)take(np_ * 3 * sizeof(R));
    R* wo = (R*)take(np_ * 3 * sizeof(R));
    R* Le = (R*)take(np_ * 3 * sizeof(R));
    R* s_r = (R*)take(np_ * sizeof(R));
    R* s_d = (R*)take(np_ * sizeof(R));
    R* frames = (R*)take(np_ * 9 * sizeof(R));
    float* stacks = (float*)take(np_ * 7 * 1024 * 4);
    float* pred = (float*)take(np_ * 3 * 1024 * 4);
    DRCB_CUDA(cudaMemcpyAsync(px, px_h, np_ * 4, cudaMemcpyHostToDevice, st));
    DRCB_CUDA(cudaMemcpyAsync(py, py_h, np_ * 4, cudaMemcpyHostToDevice, st));
    DRCB_CUDA(cudaMemcpyAsync(keys, keys_h, np_ * 8, cudaMemcpyHostToDevice, st));
    int nb = int((np_ + 127) / 128);
    k_gather_points<R><<<nb, 128, 0, st>>>(gb, W, px, py, np_, pos, nrm, wo, mat, live);
    count_launch();
    const bool tc = net_mode != DRCB_NET_FP32;
    const int64_t np8 = ((np_ + 7) / 8) * 8;
    void* xin = nullptr;
    int cpad = tc ? tc_input_channels(net_mode) : 0;
    if (tc && np_ <= 8192) {
      size_t xb = size_t(np8) * 1024 * cpad * (net_mode == DRCB_NET_TF32 ? 4 : 2);
      DRCB_CUDA(cudaMallocAsync(&xin, xb, st));
      if (np8 > np_)
        DRCB_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(xin) + xb / np8 * np_, 0,
                                  xb / np8 * (np8 - np_), st));
    }
    int rc = launch_render_stacks<R>(*S, cfg, pos, nrm, keys, live, np_, xin ? nullptr : stacks, s_r,
                                     s_d, frames, d_nf, st, xin,
                                     xin ? (net_mode == DRCB_NET_BF16 ? 1 : (net_mode == DRCB_NET_FP16 ? 3 : 2)) : 0,
                                     cpad);
    if (rc) return rc;
    if (E) E->rec(2, st);
    if (!tc)
      rc = forward_f32_chunked(net->impl, stacks, pred, np_, st);
    else if (xin)
      rc = forward_tc_nhwc(net->impl, xin, pred, np_, net_mode, st);
    else
      rc = forward_tc(net->impl, stacks, pred, np_, net_mode, st);
    if (xin) DRCB_CUDA(cudaFreeAsync(xin, st));
    if (rc) return rc;
    if (E) E->rec(3, st);
    rc = launch_shade<R>(*S, cfg, pred, s_r, frames, wo, mat, keys, live, np_, Le, st);
    if (rc) return rc;
    // stable compaction of live points, appended after the entries so far
    k_u8_to_int<<<nb, 128, 0, st>>>(live, flags, np_);
    size_t tmpb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmpb, flags, rank, int(np_), st);
    void* tmp = nullptr;
    DRCB_CUDA(cudaMallocAsync(&tmp, tmpb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tmpb, flags, rank, int(np_), st);
    DRCB_CUDA(cudaFreeAsync(tmp, st));
    k_scatter_entries<R><<<nb, 128, 0, st>>>(live, rank, np_, d_m, px, py, nrm, Le, epx, epy, en,
                                             erad, pos, static_cast<const R*>(gb.throughput), W,
                                             epos, ethr);
    k_entry_count<<<1, 1, 0, st>>>(rank, live, np_, d_m);
    count_launch(5);  // u8_to_int, scan (2), scatter, entry_count
    if (E) E->rec(4, st);
    DRCB_CUDA(cudaFreeAsync(pb, st));
    return 0;
  }

  // image = direct + interpolation of the entries so far at spacing r
  int composite(int r, R* image, cudaStream_t st) {
    return launch_interp_composite<R>(*S, W, H, gb, epx, epy, en, erad, cap > 0 ? cap : 0,
                                      cap > 0 ? d_m : nullptr, r, direct, image, st);
  }

  int entries_out(const DrcbEntries& out, cudaStream_t st) {
    if (cap <= 0) return 0;
    const size_t v = size_t(cap) * 3 * sizeof(R);
    if (out.px) DRCB_CUDA(cudaMemcpyAsync(out.px, epx, cap * 4, cudaMemcpyDeviceToDevice, st));
    if (out.py) DRCB_CUDA(cudaMemcpyAsync(out.py, epy, cap * 4, cudaMemcpyDeviceToDevice, st));
    if (out.position) DRCB_CUDA(cudaMemcpyAsync(out.position, epos, v, cudaMemcpyDeviceToDevice, st));
    if (out.normal) DRCB_CUDA(cudaMemcpyAsync(out.normal, en, v, cudaMemcpyDeviceToDevice, st));
    if (out.radiance) DRCB_CUDA(cudaMemcpyAsync(out.radiance, erad, v, cudaMemcpyDeviceToDevice, st));
    if (out.throughput) DRCB_CUDA(cudaMemcpyAsync(out.throughput, ethr, v, cudaMemcpyDeviceToDevice, st));
    return 0;
  }

  int counters(int64_t& m, int64_t& nf, cudaStream_t st) {
    int mm = 0;
    int64_t n = 0;
    DRCB_CUDA(cudaMemcpyAsync(&mm, d_m, 4, cudaMemcpyDeviceToHost, st));
    DRCB_CUDA(cudaMemcpyAsync(&n, d_nf, 8, cudaMemcpyDeviceToHost, st));
    DRCB_CUDA(cudaStreamSynchronize(st));
    m = mm;
    nf = n;
    return 0;
  }

  int end(cudaStream_t st) {
    if (pool) DRCB_CUDA(cudaFreeAsync(pool, st));
    if (fb) DRCB_CUDA(cudaFreeAsync(fb, st));
    pool = fb = nullptr;
    return 0;
  }
};

template <typename R>
int render_frame(const DrcbScene* scene, DrcbNet* net, const DrcbCamera* cam,
                 const DrcbRenderCfg* cfg, const int32_t* px_h, const int32_t* py_h,
                 const uint64_t* keys_h, int64_t np_, int r_final, int net_mode, R* image,
                 int64_t* tel, cudaStream_t st, const DrcbEntries* dump = nullptr) {
  FrameCtx<R> F;
  F.S = &scene->dev;
  F.net = net;
  F.C = make_camera(*cam);
  F.W = F.C.W;
  F.H = F.C.H;
  F.cfg = *cfg;
  F.net_mode = net_mode;
  F.cap = np_;
  StageEvents E;
  if (tel) {
    E.create();
    F.E = &E;
  }
  int rc = F.begin(st);
  if (!rc) rc = F.add_points(px_h, py_h, keys_h, np_, st);
  if (np_ <= 0) {
    E.rec(2, st);
    E.rec(3, st);
    E.rec(4, st);
  }
  if (!rc) rc = F.composite(r_final, image, st);
  E.rec(5, st);
  if (!rc && dump) rc = F.entries_out(*dump, st);
  int64_t m = 0, nf = 0;
  if (!rc && tel) rc = F.counters(m, nf, st);
  int rc2 = F.end(st);
  if (rc) return rc;
  if (rc2) return rc2;
  if (tel) {
    tel[0] = m;
    tel[1] = 0;  // fallback pixels: unreachable by construction (cache.py:306-307)
    tel[2] = nf;
    tel[3] = np_;
    // stage times in microseconds: gbuffer+direct, maps, network, shade+interp
    tel[4] = int64_t(1000.0 * E.ms(0, 1));
    tel[5] = int64_t(1000.0 * E.ms(1, 2));
    tel[6] = int64_t(1000.0 * E.ms(2, 3));
    tel[7] = int64_t(1000.0 * E.ms(3, 5));
    tel[8] = int64_t(1000.0 * E.ms(3, 4));  // shade + entry compaction
    tel[9] = int64_t(1000.0 * E.ms(4, 5));  // interpolation + composite
  }
  return 0;
}

}  // namespace
}  // namespace drcb

using namespace drcb;

#define NEED(x) \
  if (!(x)) return fail(DRCB_ECONTRACT, std::string(__func__) + ": null " #x)

extern "C" const char* drcb_last_error(void) { return g_err.c_str(); }
extern "C" int drcb_version(void) { return 1; }
extern "C" int64_t drcb_kernel_launches(void) { return g_launches.load(); }

namespace drcb {
namespace probe {
// L2 read bandwidth probe: every thread streams 16-B loads over an
// L2-resident buffer `iters` times (ld.global.cg: L2, not L1) and folds them
// into one word, so the loads cannot be elided
__global__ void __launch_bounds__(512) k_l2_read(const uint4* __restrict__ buf, int64_t n16,
                                                 int iters, unsigned long long* sink) {
  uint32_t acc = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(buf + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1ull);  // practically never; keeps the loads live
}
}  // namespace probe
}  // namespace drcb

// Profiling hook: stream `bytes` (a buffer that fits in L2) `iters` times
// through L2 -> SM loads on `stream` (the caller times it with events):
// the measured L2 read peak the traversal stages are compared against.
extern "C" int drcb_l2_read_probe(const void* buf, int64_t bytes, int32_t iters,
                                  unsigned long long* sink, void* stream) {
  NEED(buf);
  NEED(sink);
  if (bytes < 16 || iters < 1) return fail(DRCB_ECONTRACT, "drcb_l2_read_probe: bad size");
  drcb::probe::k_l2_read<<<unsigned(drcb::sm_count() * 4), 512, 0, S_(stream)>>>(
      static_cast<const uint4*>(buf), bytes / 16, iters, sink);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_l2_read");
}

extern "C" int drcb_intersect(const DrcbScene* scene, int32_t precision, const void* O,
                              const void* D, int64_t n, const void* tmin, const void* tmax,
                              int32_t record, uint8_t* hit, void* t, int64_t* prim, int32_t* mat,
                              void* pos, void* nrm, void* stream) {
  NEED(scene);
  if (n < 0) return fail(DRCB_ECONTRACT, "drcb_intersect: negative ray count");
  if (n == 0) return 0;  // an empty batch (the reference returns empty arrays)
  NEED(hit);
  if (precision == DRCB_PREC_MIXED)
    return launch_intersect_mixed(scene->dev, (const double*)O, (const double*)D, n,
                                  (const double*)tmin, (const double*)tmax, record, hit,
                                  (double*)t, prim, mat, (double*)pos, (double*)nrm, S_(stream));
  if (check_precision(precision)) return DRCB_ECONFIG;
  if (precision == 64)
    return launch_intersect<double>(scene->dev, (const double*)O, (const double*)D, n,
                                    (const double*)tmin, (const double*)tmax, record, hit,
                                    (double*)t, prim, mat, (double*)pos, (double*)nrm, S_(stream));
  return launch_intersect<float>(scene->dev, (const float*)O, (const float*)D, n,
                                 (const float*)tmin, (const float*)tmax, record, hit, (float*)t,
                                 prim, mat, (float*)pos, (float*)nrm, S_(stream));
}

extern "C" int drcb_primary_chain(const DrcbScene* scene, int32_t precision, const void* O,
                                  const void* D, int64_t n, const DrcbGBuffer* out, void* stream) {
  NEED(scene);
  NEED(out);
  if (check_precision(precision)) return DRCB_ECONFIG;
  if (precision == 64)
    return launch_primary_chain<double>(scene->dev, (const double*)O, (const double*)D, n, *out,
                                        S_(stream));
  return launch_primary_chain<float>(scene->dev, (const float*)O, (const float*)D, n, *out,
                                     S_(stream));
}

extern "C" int drcb_li_direct(const DrcbScene* scene, const DrcbRenderCfg* cfg, const void* O,
                              const void* D, const uint64_t* pix, const uint64_t* smp, int64_t n,
                              int32_t include_background, void* L, int64_t* nonfinite,
                              void* stream) {
  NEED(scene);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (cfg->precision == 64)
    return launch_li_direct<double>(scene->dev, *cfg, (const double*)O, (const double*)D, pix, smp,
                                    n, include_background, (double*)L, nonfinite, S_(stream));
  return launch_li_direct<float>(scene->dev, *cfg, (const float*)O, (const float*)D, pix, smp, n,
                                 include_background, (float*)L, nonfinite, S_(stream));
}

extern "C" int drcb_trace_radiance(const DrcbScene* scene, const DrcbRenderCfg* cfg,
                                   const void* O, const void* D, const uint64_t* pix,
                                   const uint64_t* smp, int64_t n, int32_t max_depth,
                                   int32_t skip_first_emission, int32_t rr_start, void* L,
                                   int64_t* nonfinite, void* stream) {
  NEED(scene);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (max_depth < 1) return fail(DRCB_ECONTRACT, "max_depth must be >= 1");
  if (cfg->precision == 64)
    return launch_trace_radiance<double>(scene->dev, *cfg, (const double*)O, (const double*)D, pix,
                                         smp, n, max_depth, skip_first_emission, rr_start,
                                         (double*)L, nonfinite, S_(stream));
  return launch_trace_radiance<float>(scene->dev, *cfg, (const float*)O, (const float*)D, pix, smp,
                                      n, max_depth, skip_first_emission, rr_start, (float*)L,
                                      nonfinite, S_(stream));
}

extern "C" int drcb_gbuffer_direct(const DrcbScene* scene, const DrcbCamera* cam,
                                   const DrcbRenderCfg* cfg, const DrcbGBuffer* gb, void* direct,
                                   int64_t* nonfinite, void* stream) {
  NEED(scene);
  NEED(cam);
  NEED(gb);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  DevCamera C = make_camera(*cam);
  if (cfg->precision == 64)
    return launch_gbuffer_direct<double>(scene->dev, C, *cfg, cfg->tile, *gb, (double*)direct,
                                         nonfinite, S_(stream));
  return launch_gbuffer_direct<float>(scene->dev, C, *cfg, cfg->tile, *gb, (float*)direct,
                                      nonfinite, S_(stream));
}

extern "C" int drcb_render_stacks(const DrcbScene* scene, const DrcbRenderCfg* cfg,
                                  const void* pos, const void* nrm, const uint64_t* keys,
                                  int64_t n, float* stacks, void* s_r, void* s_d, void* frames,
                                  int64_t* nonfinite, void* stream) {
  NEED(scene);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (cfg->precision == 64)
    return launch_render_stacks<double>(scene->dev, *cfg, (const double*)pos, (const double*)nrm,
                                        keys, nullptr, n, stacks, (double*)s_r, (double*)s_d,
                                        (double*)frames, nonfinite, S_(stream));
  return launch_render_stacks<float>(scene->dev, *cfg, (const float*)pos, (const float*)nrm, keys,
                                     nullptr, n, stacks, (float*)s_r, (float*)s_d, (float*)frames,
                                     nonfinite, S_(stream));
}

extern "C" int drcb_shade(const DrcbScene* scene, const DrcbRenderCfg* cfg, const float* pred,
                          const void* s_r, const void* frames, const void* wo, const int32_t* mat,
                          const uint64_t* keys, int64_t n, void* L, void* stream) {
  NEED(scene);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (cfg->precision == 64)
    return launch_shade<double>(scene->dev, *cfg, pred, (const double*)s_r, (const double*)frames,
                                (const double*)wo, mat, keys, nullptr, n, (double*)L, S_(stream));
  return launch_shade<float>(scene->dev, *cfg, pred, (const float*)s_r, (const float*)frames,
                             (const float*)wo, mat, keys, nullptr, n, (float*)L, S_(stream));
}

extern "C" int drcb_interp_composite(const DrcbScene* scene, int32_t precision, int32_t width,
                                     int32_t height, const DrcbGBuffer* gb, const int32_t* e_px,
                                     const int32_t* e_py, const void* e_normal, const void* e_rad,
                                     int64_t m, int32_t r, const void* direct, void* image,
                                     void* stream) {
  NEED(scene);
  NEED(gb);
  if (check_precision(precision)) return DRCB_ECONFIG;
  if (precision == 64)
    return launch_interp_composite<double>(scene->dev, width, height, *gb, e_px, e_py,
                                           (const double*)e_normal, (const double*)e_rad, m,
                                           nullptr, r,
                                           (const double*)direct, (double*)image, S_(stream));
  return launch_interp_composite<float>(scene->dev, width, height, *gb, e_px, e_py,
                                        (const float*)e_normal, (const float*)e_rad, m, nullptr, r,
                                        (const float*)direct, (float*)image, S_(stream));
}

extern "C" int drcb_render_drc(const DrcbScene* scene, const DrcbNet* net, const DrcbCamera* cam,
                               const DrcbRenderCfg* cfg, const int32_t* px_host,
                               const int32_t* py_host, const uint64_t* keys_host,
                               int64_t n_points, int32_t r_final, int32_t net_mode, void* image,
                               int64_t* telemetry_host, void* stream) {
  NEED(scene);
  NEED(cam);
  NEED(image);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (n_points > 0 && (!net || !px_host || !py_host || !keys_host))
    return fail(DRCB_ECONTRACT, "drcb_render_drc: points given without network/arrays");
  if (n_points > 0 && net->impl.k < 4) return fail(DRCB_ECONFIG, "bad network");
  for (int64_t i = 0; i < n_points; ++i)
    if (px_host[i] < 0 || px_host[i] >= cam->width || py_host[i] < 0 || py_host[i] >= cam->height)
      return fail(DRCB_ECONTRACT, "cache point outside the image");
  DrcbNet* mnet = const_cast<DrcbNet*>(net);
  if (cfg->precision == 64)
    return render_frame<double>(scene, mnet, cam, cfg, px_host, py_host, keys_host, n_points,
                                r_final, net_mode, (double*)image, telemetry_host, S_(stream));
  return render_frame<float>(scene, mnet, cam, cfg, px_host, py_host, keys_host, n_points, r_final,
                             net_mode, (float*)image, telemetry_host, S_(stream));
}

extern "C" int drcb_render_drc_entries(const DrcbScene* scene, const DrcbNet* net,
                                       const DrcbCamera* cam, const DrcbRenderCfg* cfg,
                                       const int32_t* px_host, const int32_t* py_host,
                                       const uint64_t* keys_host, int64_t n_points,
                                       int32_t r_final, int32_t net_mode, void* image,
                                       int64_t* telemetry_host, const DrcbEntries* entries,
                                       void* stream) {
  NEED(entries);
  if (n_points > 0 && (!entries->px || !entries->py || !entries->position || !entries->normal ||
                       !entries->radiance || !entries->throughput))
    return fail(DRCB_ECONTRACT, "drcb_render_drc_entries: null entry buffer");
  NEED(scene);
  NEED(cam);
  NEED(image);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (n_points > 0 && (!net || !px_host || !py_host || !keys_host))
    return fail(DRCB_ECONTRACT, "drcb_render_drc_entries: points given without network/arrays");
  for (int64_t i = 0; i < n_points; ++i)
    if (px_host[i] < 0 || px_host[i] >= cam->width || py_host[i] < 0 || py_host[i] >= cam->height)
      return fail(DRCB_ECONTRACT, "cache point outside the image");
  DrcbNet* mnet = const_cast<DrcbNet*>(net);
  if (cfg->precision == 64)
    return render_frame<double>(scene, mnet, cam, cfg, px_host, py_host, keys_host, n_points,
                                r_final, net_mode, (double*)image, telemetry_host, S_(stream),
                                entries);
  return render_frame<float>(scene, mnet, cam, cfg, px_host, py_host, keys_host, n_points, r_final,
                             net_mode, (float*)image, telemetry_host, S_(stream), entries);
}

// ---- progressive frames (drc/cache.py:426-469 control plane): the host
// runs the pass loop, polls interrupts between passes and takes snapshots
struct DrcbFrame {
  int prec = 64;
  FrameCtx<double> d;
  FrameCtx<float> f;
};

namespace {
template <typename F>
int with_frame(DrcbFrame* fr, F&& fn) {
  return fr->prec == 64 ? fn(fr->d) : fn(fr->f);
}
}  // namespace

extern "C" int drcb_frame_begin(const DrcbScene* scene, const DrcbNet* net, const DrcbCamera* cam,
                                const DrcbRenderCfg* cfg, int32_t net_mode, int64_t max_points,
                                DrcbFrame** out, void* stream) {
  NEED(scene);
  NEED(cam);
  NEED(out);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (max_points < 0) return fail(DRCB_ECONTRACT, "drcb_frame_begin: negative max_points");
  if (max_points > 0 && !net) return fail(DRCB_ECONTRACT, "drcb_frame_begin: points need a network");
  DrcbFrame* fr = new DrcbFrame();
  fr->prec = cfg->precision;
  int rc = with_frame(fr, [&](auto& F) {
    F.S = &scene->dev;
    F.net = const_cast<DrcbNet*>(net);
    F.C = make_camera(*cam);
    F.W = F.C.W;
    F.H = F.C.H;
    F.cfg = *cfg;
    F.net_mode = net_mode;
    F.cap = max_points;
    return F.begin(S_(stream));
  });
  if (rc) {
    with_frame(fr, [&](auto& F) { return F.end(S_(stream)); });
    delete fr;
    return rc;
  }
  *out = fr;
  return 0;
}

extern "C" int drcb_frame_add_points(DrcbFrame* fr, const int32_t* px_host, const int32_t* py_host,
                                     const uint64_t* keys_host, int64_t n, void* stream) {
  NEED(fr);
  if (n <= 0) return 0;
  if (!px_host || !py_host || !keys_host) return fail(DRCB_ECONTRACT, "drcb_frame_add_points: null arrays");
  return with_frame(fr, [&](auto& F) {
    for (int64_t i = 0; i < n; ++i)
      if (px_host[i] < 0 || px_host[i] >= F.W || py_host[i] < 0 || py_host[i] >= F.H)
        return fail(DRCB_ECONTRACT, "cache point outside the image");
    return F.add_points(px_host, py_host, keys_host, n, S_(stream));
  });
}

extern "C" int drcb_frame_composite(DrcbFrame* fr, int32_t r, void* image, void* stream) {
  NEED(fr);
  NEED(image);
  if (r < 1) return fail(DRCB_ECONFIG, "drcb_frame_composite: spacing r must be >= 1");
  if (fr->prec == 64) return fr->d.composite(r, static_cast<double*>(image), S_(stream));
  return fr->f.composite(r, static_cast<float*>(image), S_(stream));
}

extern "C" int drcb_frame_info(DrcbFrame* fr, int64_t* out4, void* stream) {
  NEED(fr);
  NEED(out4);
  return with_frame(fr, [&](auto& F) {
    int64_t m = 0, nf = 0;
    int rc = F.counters(m, nf, S_(stream));
    out4[0] = m;
    out4[1] = nf;
    out4[2] = F.points;
    out4[3] = F.cap;
    return rc;
  });
}

extern "C" int drcb_frame_entries(DrcbFrame* fr, const DrcbEntries* out, void* stream) {
  NEED(fr);
  NEED(out);
  return with_frame(fr, [&](auto& F) { return F.entries_out(*out, S_(stream)); });
}

extern "C" int drcb_frame_end(DrcbFrame* fr, void* stream) {
  if (!fr) return 0;
  int rc = with_frame(fr, [&](auto& F) { return F.end(S_(stream)); });
  delete fr;
  return rc;
}

extern "C" int drcb_render_pt(const DrcbScene* scene, const DrcbCamera* cam,
                              const DrcbRenderCfg* cfg, void* image, int64_t* nonfinite,
                              void* stream) {
  NEED(scene);
  NEED(cam);
  NEED(image);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  DevCamera C = make_camera(*cam);
  if (cfg->precision == 64)
    return launch_pt_frame<double>(scene->dev, C, *cfg, cfg->direct_spp, cfg->tile,
                                   (double*)image, nonfinite, S_(stream));
  return launch_pt_frame<float>(scene->dev, C, *cfg, cfg->direct_spp, cfg->tile, (float*)image,
                                nonfinite, S_(stream));
}

extern "C" int drcb_reference_map(const DrcbScene* scene, const DrcbRenderCfg* cfg,
                                  const void* pos, const void* nrm, uint64_t key, int32_t ref_spp,
                                  void* out, int64_t* nonfinite, void* stream) {
  NEED(scene);
  NEED(pos);
  NEED(nrm);
  NEED(out);
  if (check_cfg(cfg)) return DRCB_ECONFIG;
  if (ref_spp < 1) return fail(DRCB_ECONFIG, "ref_spp must be >= 1");
  if (cfg->precision == 64)
    return launch_reference_map<double>(scene->dev, *cfg, (const double*)pos, (const double*)nrm,
                                        key, ref_spp, (double*)out, nonfinite, S_(stream));
  return launch_reference_map<float>(scene->dev, *cfg, (const float*)pos, (const float*)nrm, key,
                                     ref_spp, (float*)out, nonfinite, S_(stream));
}

extern "C" int drcb_net_forward(const DrcbNet* net, const float* x, float* y, int64_t n,
                                int32_t mode, void* stream) {
  NEED(net);
  if (n <= 0) return 0;
  NEED(x);
  NEED(y);
  if (mode == DRCB_NET_FP32) return forward_f32_chunked(net->impl, x, y, n, S_(stream));
  if (mode == DRCB_NET_TF32 || mode == DRCB_NET_BF16 || mode == DRCB_NET_FP16)
    return forward_tc(const_cast<DrcbNet*>(net)->impl, x, y, n, mode, S_(stream));
  return fail(DRCB_ECONFIG, "unknown network mode");
}
