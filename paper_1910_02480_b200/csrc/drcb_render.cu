// drcb_render.cu — ray/path kernels of one DRC frame, instantiated for fp64
// (parity) and fp32 (fast). Compiled with -fmad=false (see Makefile).
//
//   k_intersect        intersect_batch / occluded_batch  (geometry.py:217-329)
//   k_primary_chain    primary_chain_batch               (integrators.py:427-518)
//   k_li_direct        li_direct_batch                   (integrators.py:305-424)
//   k_trace            trace_radiance_batch              (integrators.py:175-302)
//   k_gbuffer_direct   DrcState geo + direct pass, fused (cache.py:157-176, 393-423)
//   k_map_rays         render_input_stacks_batch rays    (hemimap.py:229-262)
//   k_stack_normalize  per-map s_r / s_d + fp32 stack    (hemimap.py:264-281)
//   k_shade            build_map_distribution+shade_indirect (hemimap.py:156-197,
//                      integrators.py:564-614)
//   k_interp           _interpolate_layer + composite    (cache.py:283-345, 463)
#include <cub/cub.cuh>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "drcb_internal.h"
#include "drcb_trace.cuh"

#ifndef DRCB_RENDER_PREC
#define DRCB_RENDER_PREC 64
#endif
// kernels live in a per-build namespace: both objects define them
#if DRCB_RENDER_PREC == 32
#define DRCB_RENDER_NS render_f32
#else
#define DRCB_RENDER_NS render_f64
#endif

namespace drcb {

namespace DRCB_RENDER_NS {

constexpr int TPB = 128;
#ifndef DIRECT_CTAS
#define DIRECT_CTAS 8  // CTAs/SM the direct-pass kernel's registers are sized for
#endif

inline int nblocks(int64_t n, int tpb = TPB) { return int((n + tpb - 1) / tpb); }

template <typename R>
__global__ void k_intersect(DevScene S, const R* __restrict__ O, const R* __restrict__ D,
                            int64_t n, const R* tmin, const R* tmax, int record, uint8_t* hit,
                            R* t, int64_t* prim, int32_t* mat, R* pos, R* nrm) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3<R> o = ldr3(O + 3 * i), d = ldr3(D + 3 * i);
  R lo = tmin ? tmin[i] : R(T_EPS);
  R hi = tmax ? tmax[i] : R(INFINITY);
  if (!record) {
    HitRec<R> h = traverse<R, false>(S, o, d, lo, hi);
    hit[i] = h.prim >= 0;
    if (t) t[i] = h.prim >= 0 ? h.t : R(INFINITY);
    if (prim) prim[i] = h.prim;
    return;
  }
  SurfHit<R> h = intersect(S, o, d, lo, hi);
  hit[i] = h.hit;
  if (t) t[i] = h.t;
  if (prim) prim[i] = h.prim;
  if (mat) mat[i] = h.mat;
  if (pos) st3(pos + 3 * i, h.pos);
  if (nrm) st3(nrm + 3 * i, h.normal);
}

// fp32 build, mixed mode: fp64 rays (drcb_intersect, DRCB_PREC_MIXED) cast
// by the fp32 traversal, undecided / near-tie candidates re-tested against
// the fp64 ray itself
__global__ void k_intersect_mixed(DevScene S, const double* __restrict__ O, const double* __restrict__ D,
                                  int64_t n, const double* tmin, const double* tmax, int record,
                                  uint8_t* hit, double* t, int64_t* prim, int32_t* mat, double* pos,
                                  double* nrm) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V3<float> o = cvt<float>(ldr3(O + 3 * i)), d = cvt<float>(ldr3(D + 3 * i));
  const double lo64 = tmin ? tmin[i] : T_EPS, hi64 = tmax ? tmax[i] : double(INFINITY);
  const float lo = lo64 == T_EPS ? float(T_EPS) : float(lo64);
  const float hi = float(hi64);
  const Ray64Ptr ref{O + 3 * i, D + 3 * i};
  SurfHit<float> h = intersect<float, Ray64Ptr>(S, o, d, lo, hi, ref);
  hit[i] = h.hit;
  if (t) t[i] = double(h.t);
  if (prim) prim[i] = h.prim;
  if (record) {
    if (mat) mat[i] = h.mat;
    if (pos) st3(pos + 3 * i, cvt<double>(h.pos));
    if (nrm) st3(nrm + 3 * i, cvt<double>(h.normal));
  }
}

// the pixel's fp64 camera ray (scene.py:76-93), recomputed only when a
// primary-cast candidate needs the fp64 re-test
struct CameraRay64 {
  const DevCamera* C;
  float px, py;
  template <typename R>
  __device__ __forceinline__ void get(V3<R>, V3<R>, V3<Dn>& o, V3<Dn>& d) const {
    o = ld3<Dn>(C->pos);
    d = camera_dir<Dn>(*C, Dn(double(px)), Dn(double(py)));
  }
};

template <typename R>
__device__ __forceinline__ void store_chain(const DrcbGBuffer& gb, int64_t i, const ChainOut<R>& c) {
  gb.found[i] = c.found;
  gb.escaped[i] = c.escaped;
  st3(static_cast<R*>(gb.position) + 3 * i, c.pos);
  st3(static_cast<R*>(gb.normal) + 3 * i, c.normal);
  st3(static_cast<R*>(gb.throughput) + 3 * i, c.thr);
  st3(static_cast<R*>(gb.direction) + 3 * i, c.dir);
  static_cast<R*>(gb.t_total)[i] = c.t_total;
  gb.mat[i] = c.mat;
}

template <typename R>
__global__ void k_primary_chain(DevScene S, const R* __restrict__ O, const R* __restrict__ D,
                                int64_t n, DrcbGBuffer gb) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  store_chain(gb, i, primary_chain(S, ldr3(O + 3 * i), ldr3(D + 3 * i)));
}

__device__ __forceinline__ void add_nonfinite(int64_t* ctr, int c) {
  if (ctr && c) atomicAdd((unsigned long long*)ctr, (unsigned long long)c);
}

template <typename R>
__global__ void k_li_direct(DevScene S, DrcbRenderCfg cfg, const R* __restrict__ O,
                            const R* __restrict__ D, const uint64_t* pix, const uint64_t* smp,
                            int64_t n, int include_bg, R* L, int64_t* nonfinite) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (i < n) {
    PathRng rng;
    rng.init(cfg.seed, pix[i], smp[i], cfg.sampler_kind, uint32_t(cfg.direct_spp > 1 ? cfg.direct_spp : 1));
    V3<R> l = direct_path(S, ldr3(O + 3 * i), ldr3(D + 3 * i), rng, include_bg != 0, nf);
    st3(L + 3 * i, l);
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

template <typename R>
__global__ void k_trace(DevScene S, DrcbRenderCfg cfg, const R* __restrict__ O,
                        const R* __restrict__ D, const uint64_t* pix, const uint64_t* smp,
                        int64_t n, int max_depth, int skip_first, int rr_start, R* L,
                        int64_t* nonfinite) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (i < n) {
    PathRng rng;
    // trace_radiance_batch is always called with a spp=1 sampler in the
    // reference pipeline; honour the configured kind/spp for direct calls.
    rng.init(cfg.seed, pix[i], smp[i], cfg.sampler_kind, uint32_t(cfg.direct_spp > 1 ? cfg.direct_spp : 1));
    V3<R> l = trace_path<R>(S, ldr3(O + 3 * i), ldr3(D + 3 * i), rng, max_depth, skip_first != 0,
                            rr_start, nullptr, nf);
    st3(L + 3 * i, l);
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// One thread per pixel: the unjittered centre chain (G-buffer) and the
// direct_spp jittered li_direct samples, averaged (cache.py:157-176, 393-423).
template <typename R>
__global__ void __launch_bounds__(TPB) k_gbuffer_direct(DevScene S, const __grid_constant__ DevCamera C, DrcbRenderCfg cfg,
                                                         int tile, DrcbGBuffer gb, R* direct,
                                                         int64_t* nonfinite) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t npx = int64_t(C.W) * C.H;
  int nf = 0;
  if (i < npx) {
    int x = int(i % C.W), y = int(i / C.W);
    V3<R> cam = ld3<R>(C.pos);
    V3<R> dc = camera_dir<R>(C, R(x) + R(0.5), R(y) + R(0.5));
    store_chain(gb, i, primary_chain(S, cam, dc, CameraRay64{&C, x + 0.5f, y + 0.5f}));
    // direct pass; samples are summed in the reference's per-tile chunks
    int spp = cfg.direct_spp;
    int tx0 = (x / tile) * tile, ty0 = (y / tile) * tile;
    int tw = min(tile, C.W - tx0), th = min(tile, C.H - ty0);
    int chunk = max(1, 16384 / (tw * th));
    PathRng rng;
    V3<R> acc = {R(0), R(0), R(0)};
    for (int s0 = 0; s0 < spp; s0 += chunk) {
      int ns = min(chunk, spp - s0);
      V3<R> part;
      for (int s = s0; s < s0 + ns; ++s) {
        rng.init(cfg.seed, uint64_t(i), uint64_t(s), cfg.sampler_kind, uint32_t(spp > 1 ? spp : 1));
        R jx = to_unit<R>(rng.sample(0)), jy = to_unit<R>(rng.sample(1));
        V3<R> d = camera_dir<R>(C, R(x) + jx, R(y) + jy);
        V3<R> l = direct_path(S, cam, d, rng, cfg.include_background != 0, nf);
        part = (s == s0) ? l : part + l;
      }
      acc = acc + part;
    }
    R inv = R(spp);
    st3(direct + 3 * i, mk<R>(acc.x / inv, acc.y / inv, acc.z / inv));
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// Split form of the direct pass: one thread per pixel for the centre chain,
// one thread per (pixel, sample) for the jittered li_direct paths, and an
// ordered per-pixel reduction that sums samples in the reference's per-tile
// chunks ((s0 + s1 + ...) per chunk, chunks accumulated from 0) and divides
// by direct_spp (cache.py:399-413).
// thread k of a frame -> pixel: 32 consecutive threads cover an 8x4 pixel
// block (coherent primary and shadow rays per warp) when the frame tiles
// evenly, row-major otherwise
__device__ __forceinline__ int64_t pixel_of(const DevCamera& C, int64_t k) {
  if ((C.W & 7) || (C.H & 3)) return k;
  const int64_t b = k >> 5;
  const int w = int(k & 31), bpr = C.W >> 3;
  return (int64_t(b / bpr) * 4 + (w >> 3)) * C.W + int64_t(b % bpr) * 8 + (w & 7);
}

template <typename R>
__global__ void __launch_bounds__(TPB, 8) k_gbuffer(DevScene S, const __grid_constant__ DevCamera C,
                                                    DrcbGBuffer gb) {
  int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= int64_t(C.W) * C.H) return;
  const int64_t i = pixel_of(C, k);
  int x = int(i % C.W), y = int(i / C.W);
  V3<R> dc = camera_dir<R>(C, R(x) + R(0.5), R(y) + R(0.5));
  store_chain(gb, i, primary_chain(S, ld3<R>(C.pos), dc, CameraRay64{&C, x + 0.5f, y + 0.5f}));
}

template <typename R>
__global__ void __launch_bounds__(TPB, DIRECT_CTAS) k_direct_samples(DevScene S, DevCamera C, DrcbRenderCfg cfg,
                                                         R* samples, int64_t* nonfinite) {
  const int spp = cfg.direct_spp;
  const int64_t npx = int64_t(C.W) * C.H;
  int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (g < npx * spp) {
    // sample-major: neighbouring threads trace neighbouring pixels (8x4 blocks)
    const int64_t i = pixel_of(C, g % npx);
    int s = int(g / npx);
    int x = int(i % C.W), y = int(i / C.W);
    PathRng rng;
    rng.init(cfg.seed, uint64_t(i), uint64_t(s), cfg.sampler_kind, uint32_t(spp > 1 ? spp : 1));
    R jx = to_unit<R>(rng.sample(0)), jy = to_unit<R>(rng.sample(1));
    V3<R> d = camera_dir<R>(C, R(x) + jx, R(y) + jy);
    st3(samples + 3 * (int64_t(s) * npx + i),
        direct_path(S, ld3<R>(C.pos), d, rng, cfg.include_background != 0, nf));
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// direct_spp == 1: the G-buffer centre chain and the pixel's one li_direct
// path in one thread (one launch, no per-sample buffer; the jittered camera
// ray re-walks the BVH nodes the centre ray just brought into L1). The
// result is exactly k_direct_reduce's for one sample: (0 + L) / 1.
template <typename R>
__global__ void __launch_bounds__(TPB, DIRECT_CTAS) k_gbuffer_direct1(DevScene S, const __grid_constant__ DevCamera C,
                                                                     DrcbRenderCfg cfg,
                                                                     DrcbGBuffer gb, R* direct,
                                                                     int64_t* nonfinite) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (k < int64_t(C.W) * C.H) {
    const int64_t i = pixel_of(C, k);
    const int x = int(i % C.W), y = int(i / C.W);
    const V3<R> cam = ld3<R>(C.pos);
    store_chain(gb, i, primary_chain(S, cam, camera_dir<R>(C, R(x) + R(0.5), R(y) + R(0.5)),
                                     CameraRay64{&C, x + 0.5f, y + 0.5f}));
    PathRng rng;
    rng.init(cfg.seed, uint64_t(i), 0ull, cfg.sampler_kind, 1u);
    const R jx = to_unit<R>(rng.sample(0)), jy = to_unit<R>(rng.sample(1));
    const V3<R> d = camera_dir<R>(C, R(x) + jx, R(y) + jy);
    const V3<R> l = direct_path(S, cam, d, rng, cfg.include_background != 0, nf);
    const V3<R> acc = mk<R>(R(0), R(0), R(0)) + l;
    st3(direct + 3 * i, divs(acc, R(1)));
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

template <typename R>
__global__ void k_direct_reduce(DevCamera C, int spp, int tile, const R* __restrict__ samples,
                                R* direct) {
  const int64_t npx = int64_t(C.W) * C.H;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= npx) return;
  int x = int(i % C.W), y = int(i / C.W);
  int tx0 = (x / tile) * tile, ty0 = (y / tile) * tile;
  int tw = min(tile, C.W - tx0), th = min(tile, C.H - ty0);
  int chunk = max(1, 16384 / (tw * th));
  V3<R> acc = {R(0), R(0), R(0)};
  for (int s0 = 0; s0 < spp; s0 += chunk) {
    int ns = min(chunk, spp - s0);
    V3<R> part = ldr3(samples + 3 * (int64_t(s0) * npx + i));
    for (int s = s0 + 1; s < s0 + ns; ++s) part = part + ldr3(samples + 3 * (int64_t(s) * npx + i));
    acc = acc + part;
  }
  st3(direct + 3 * i, divs(acc, R(spp)));
}

// local texel directions (texel_local) tabulated once per precision by the
// same device function: the path kernel's fresh lanes read 3 values instead
// of evaluating three precise sin/cos
template <typename R>
__device__ R g_texel_dirs[3 * MAP_TEXELS];

template <typename R>
__global__ void k_texel_dirs() {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= MAP_TEXELS) return;
  const V3<R> d = texel_local<R>(t % MAP_RES, t / MAP_RES);
  g_texel_dirs<R>[3 * t] = d.x;
  g_texel_dirs<R>[3 * t + 1] = d.y;
  g_texel_dirs<R>[3 * t + 2] = d.z;
}

// Map paths of all cache points (hemimap.py:236-262 + integrators.py:175-302)
// as a persistent kernel with per-lane path regeneration: a lane whose path
// terminates (escape, RR, max depth) immediately takes the next texel from a
// global counter, so warps stay full instead of idling behind the longest
// path of the warp. The segment-0 cast doubles as the first-hit feature cast
// (the reference casts it twice, hemimap.py:250 and segment 0).
constexpr int MAP_TPB = 256;
// CTAs per SM the path kernel's registers are sized for (fp32 build: 5,
// measured 3.42 / 3.18 / 3.08 / 3.22 / 3.58 ms for 3 / 4 / 5 / 6 / 8)
#ifndef MAP_CTAS
#define MAP_CTAS 4
#endif

template <typename R>
__global__ void __launch_bounds__(MAP_TPB, MAP_CTAS) k_map_paths(DevScene S, DrcbRenderCfg cfg,
                                                          const R* __restrict__ pos,
                                                          const R* __restrict__ nrm,
                                                          const uint64_t* __restrict__ keys,
                                                          const uint8_t* __restrict__ live,
                                                          int64_t total, unsigned long long* counter,
                                                          R* rad, R* dist, R* nloc,
                                                          int64_t* nonfinite, int tab,
                                                          const R* __restrict__ frames,
                                                          const uint64_t* __restrict__ pre2) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  bool have = false, done_all = false;
  int64_t job = 0, slot = 0;
  int seg = 0;
  bool prev_delta = true;
  R prev_pdf = R(0);
  V3<R> O, D, beta, L;
  PathRng rng;
  int nf = 0;
  const V3<R> env = ld3<R>(S.env);
  while (true) {
    bool need = !have && !done_all;
    unsigned m = __ballot_sync(FULL, need);
    bool fresh = false;
    if (m) {
      int leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
      base = __shfl_sync(FULL, base, leader);
      if (need) {
        job = int64_t(base) + __popc(m & ((1u << lane) - 1u));
        if (job >= total) {
          done_all = true;
        } else if (!live || live[job / MAP_TEXELS]) {
          have = true;
          fresh = true;
        }
      }
    }
    if (__all_sync(FULL, !have && done_all)) break;
    if (!have) continue;
    bool skip = false;
    int64_t p = 0;
    int tex = 0;
    if (fresh) {
      p = job / MAP_TEXELS;
      // 32 consecutive jobs = an 8x4 texel block (a compact solid angle)
      // rather than a 32-texel row: coherent first-bounce rays per warp
      const int k = int(job % MAP_TEXELS), blk = k >> 5, w = k & 31;
      tex = ((blk >> 2) * 4 + (w >> 3)) * MAP_RES + (blk & 3) * 8 + (w & 7);
      slot = p * MAP_TEXELS + tex;
      const V3<R> hp = ldr3(pos + 3 * p);
      const R* F = frames + 9 * p;  // k_point_frames: frame_scalar of the point normal
      Frame<R> fr{ldr3(F), ldr3(F + 3), ldr3(F + 6)};  // fr.n is the point normal itself
      D = fr.to_world(tab ? ldr3(g_texel_dirs<R> + 3 * tex) : texel_local<R>(tex % MAP_RES, tex / MAP_RES));
      O = hp + R(T_EPS) * fr.n;
    }
    // single traversal call site for fresh and continuing lanes
    SurfHit<R> h = intersect(S, O, D);
    if (fresh) {
      // first-hit features: distance and front-facing normal in the map frame
      const R* F = frames + 9 * p;
      Frame<R> fr{ldr3(F), ldr3(F + 3), ldr3(F + 6)};
      bool facing = dot(h.normal, D) > R(0);
      V3<R> nf3 = facing ? -h.normal : h.normal;
      dist[slot] = h.hit ? h.t : R(0);
      st3(nloc + 3 * slot, h.hit ? fr.to_local(nf3) : mk<R>(R(0), R(0), R(0)));
      rng.init_pre(pre2[p], cfg.seed, keys[p], uint64_t(tex), cfg.sampler_kind,
               uint32_t(cfg.map_spp > 1 ? cfg.map_spp : 1));
      L = mk<R>(R(0), R(0), R(0));
      beta = mk<R>(R(1), R(1), R(1));
      seg = 0;
      prev_pdf = R(0);
      prev_delta = true;
      skip = true;  // skip_first_emission at segment 0
    }
    // ---- one segment of trace_radiance_batch
    bool end = false;
    if (!h.hit) {
      if (S.has_env && !skip) L = L + beta * env;
      end = true;
    } else {
      const int mat = h.mat;
      const bool facing = dot(h.normal, D) < R(0);
      if (S.mat_emitter[mat] && facing && !skip) {
        R w = R(1);
        if (seg > 0 && !prev_delta) {
          R pdf_nee = nee_pdf_for_hit(S, h.prim, h.t, -dot(h.normal, D));
          w = power_heuristic(prev_pdf, pdf_nee);
        }
        L = L + (beta * ld3<R>(S.mat_emis + 3 * mat)) * mk<R>(w, w, w);
      }
      if (seg == cfg.max_path_depth) {
        end = true;
      } else {
        V3<R> n_front = facing ? h.normal : -h.normal;
        Frame<R> fr = frame_batch(S, n_front);
        V3<R> wo_local = fr.to_local(-D);
        uint64_t base = 2 + 8 * (uint64_t)seg;
        if (S.n_lights > 0 && !S.mat_spec[mat])
          L = L + beta * nee(S, rng, base, h.pos, n_front, fr, mat, wo_local);
        R u1 = sample_dim<R>(rng, base + 3), u2 = sample_dim<R>(rng, base + 4);
        BsdfSample<R> bs = bsdf_sample(S, mat, wo_local, u1, u2, facing);
        R cos_i = fabs(bs.li.z);
        R k = cos_i / bs.pdf;
        beta = beta * (bs.spec ? bs.value : bs.value * mk<R>(k, k, k));
        R side = bs.li.z >= R(0) ? R(1) : R(-1);
        O = h.pos + (R(T_EPS) * side) * n_front;
        D = fr.to_world(bs.li);
        prev_pdf = bs.pdf;
        prev_delta = bs.spec;
        bool alive = any_pos(beta) && all_finite(beta);
        if (seg + 1 >= cfg.rr_start) {
          R q = fmin(fmax(maxc(beta), R(RR_FLOOR)), R(1));
          bool survive = sample_dim<R>(rng, base + 5) < q;
          beta = divs(beta, q);
          alive = alive && survive;
        }
        ++seg;
        end = !alive;
      }
    }
    if (end) {
      if (!all_finite(L)) {
        L = mk<R>(R(0), R(0), R(0));
        ++nf;
      }
      st3(rad + 3 * slot, L);
      have = false;
    }
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// cache-point frames (build_frame of the front normal, hemimap.py:238)
template <typename R>
__global__ void k_point_frames(DevScene S, const R* __restrict__ nrm, int64_t n, R* frames,
                               const uint64_t* __restrict__ keys = nullptr, uint64_t seed = 0,
                               uint64_t* pre2 = nullptr) {
  int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  // the per-point part of the path samplers' hash prefix (PathRng::init_pre)
  if (pre2) pre2[p] = hash_step(hash_step(SEED0, seed), keys[p]);
  Frame<R> fr = frame_scalar(S, ldr3(nrm + 3 * p));
  st3(frames + 9 * p, fr.t);
  st3(frames + 9 * p + 3, fr.b);
  st3(frames + 9 * p + 6, fr.n);
}

// render(mode="pt") (integrators.py:678-722): spp jittered camera paths per
// pixel through trace_radiance_batch, summed in the reference's per-tile
// sample chunks, averaged. One thread per pixel.
template <typename R>
__global__ void __launch_bounds__(TPB) k_pt_frame(DevScene S, DevCamera C, DrcbRenderCfg cfg,
                                                   int spp, int tile, R* image,
                                                   int64_t* nonfinite) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (i < int64_t(C.W) * C.H) {
    int x = int(i % C.W), y = int(i / C.W);
    V3<R> cam = ld3<R>(C.pos);
    int tx0 = (x / tile) * tile, ty0 = (y / tile) * tile;
    int tw = min(tile, C.W - tx0), th = min(tile, C.H - ty0);
    int chunk = max(1, 16384 / (tw * th));
    PathRng rng;
    V3<R> acc = {R(0), R(0), R(0)};
    for (int s0 = 0; s0 < spp; s0 += chunk) {
      int ns = min(chunk, spp - s0);
      V3<R> part;
      for (int s = s0; s < s0 + ns; ++s) {
        rng.init(cfg.seed, uint64_t(i), uint64_t(s), cfg.sampler_kind, uint32_t(spp > 1 ? spp : 1));
        R jx = to_unit<R>(rng.sample(0)), jy = to_unit<R>(rng.sample(1));
        V3<R> d = camera_dir<R>(C, R(x) + jx, R(y) + jy);
        V3<R> l = trace_path<R>(S, cam, d, rng, cfg.max_path_depth, false, cfg.rr_start, nullptr, nf);
        part = (s == s0) ? l : part + l;
      }
      acc = acc + part;
    }
    st3(image + 3 * i, divs(acc, R(spp)));
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// _reference_map (dataset.py:107-127): ref_spp paths per texel of one cache
// point (pixel key = texel + key * 4096, sample key = s), skip first emission.
// One thread per path (sample s, texel) of a group of samples writes its
// radiance; the reduction then adds them in the reference's order.
template <typename R>
__global__ void __launch_bounds__(TPB) k_reference_paths(DevScene S, DrcbRenderCfg cfg,
                                                          const R* __restrict__ pos,
                                                          const R* __restrict__ nrm,
                                                          uint64_t key, int ref_spp, int s_begin,
                                                          int s_count, R* paths,
                                                          int64_t* nonfinite) {
  int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int nf = 0;
  if (g < int64_t(s_count) * MAP_TEXELS) {
    const int tex = int(g % MAP_TEXELS), s = s_begin + int(g / MAP_TEXELS);
    V3<R> hp = ldr3(pos), hn = ldr3(nrm);
    Frame<R> fr = frame_scalar(S, hn);
    V3<R> D = fr.to_world(texel_local<R>(tex % MAP_RES, tex / MAP_RES));
    V3<R> O = hp + R(T_EPS) * hn;
    uint64_t pix = uint64_t(tex) + key * uint64_t(1 << 12);
    PathRng rng;
    rng.init(cfg.seed, pix, uint64_t(s), cfg.sampler_kind, uint32_t(ref_spp > 1 ? ref_spp : 1));
    st3(paths + 3 * g, trace_path<R>(S, O, D, rng, cfg.max_path_depth, true, cfg.rr_start, nullptr, nf));
  }
  if (nonfinite) add_nonfinite(nonfinite, nf);
}

// the reference's sums: per chunk of `chunk` samples the sequential sum
// (numpy's axis-0 sum), total = ((0 + chunk_0) + chunk_1) + ...; the group's
// chunks [c_begin, c_end) continue `tot`; the last group writes total / ref_spp
template <typename R>
__global__ void k_reference_reduce(const R* __restrict__ paths, int s_begin, int chunk,
                                   int c_begin, int c_end, int ref_spp, R* tot_buf, R* out,
                                   int last) {
  int tex = blockIdx.x * blockDim.x + threadIdx.x;
  if (tex >= MAP_TEXELS) return;
  V3<R> tot = c_begin == 0 ? mk<R>(R(0), R(0), R(0)) : ldr3(tot_buf + 3 * tex);
  for (int c = c_begin; c < c_end; ++c) {
    const int s0 = c * chunk, ns = min(chunk, ref_spp - s0);
    V3<R> part = ldr3(paths + 3 * (int64_t(s0 - s_begin) * MAP_TEXELS + tex));
    for (int s = s0 + 1; s < s0 + ns; ++s)
      part = part + ldr3(paths + 3 * (int64_t(s - s_begin) * MAP_TEXELS + tex));
    tot = tot + part;
  }
  if (last)
    st3(out + 3 * tex, divs(tot, R(ref_spp)));
  else
    st3(tot_buf + 3 * tex, tot);
}

// numpy pairwise summation of 1024 contiguous values (8-accumulator blocks of
// 128, binary tree above), replicated bit for bit. `a` is in shared memory;
// must be called by all threads of the block; result valid in all threads.
template <typename R>
__device__ R pairwise1024(const R* a, R* scratch /* >= 64 */) {
  int t = threadIdx.x;
  if (t < 64) {
    int blk = t >> 3, j = t & 7;
    const R* b = a + 128 * blk;
    R r = b[j];
    for (int i = 8; i < 128; i += 8) r = r + b[i + j];
    scratch[t] = r;
  }
  __syncthreads();
  R res;
  {
    R B[8];
    for (int blk = 0; blk < 8; ++blk) {
      const R* r = scratch + 8 * blk;
      B[blk] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    }
    res = ((B[0] + B[1]) + (B[2] + B[3])) + ((B[4] + B[5]) + (B[6] + B[7]));
  }
  __syncthreads();
  return res;
}

// numpy pairwise sum of 32 contiguous values (n <= 128 branch)
template <typename R>
__device__ __forceinline__ R pairwise32(const R* a) {
  R r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  for (int i = 8; i < 32; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

constexpr double LUMA_R = 0.2126, LUMA_G = 0.7152, LUMA_B = 0.0722;  // hemimap.py:26

// One block (256 threads) per cache point: s_r = mean luminance + 1e-3,
// s_d = max distance (or 1), fp32 NCHW stack [rad/s_r, n_local, d/s_d].
// nhwc_kind: 0 = none, 1 = bf16, 2 = tf32-rounded fp32, 3 = fp16 compact NHWC input of
// the tensor-core network (cpad = 8: 7 channels + 1 zero), written here directly
template <typename R>
__global__ void __launch_bounds__(256) k_stack_normalize(const R* __restrict__ rad,
                                                         const R* __restrict__ dist,
                                                         const R* __restrict__ nloc,
                                                         const uint8_t* __restrict__ live,
                                                         int64_t n, float* stacks, R* s_r,
                                                         R* s_d, void* nhwc, int nhwc_kind,
                                                         int cpad) {
  __shared__ R lum[MAP_TEXELS];
  __shared__ R scratch[64];
  __shared__ R dmax[8];
  int64_t p = blockIdx.x;
  if (p >= n) return;
  float* out = stacks ? stacks + p * 7 * MAP_TEXELS : nullptr;
  if (live && !live[p]) {
    if (stacks)
      for (int t = threadIdx.x; t < 7 * MAP_TEXELS; t += blockDim.x) out[t] = 0.f;
    if (nhwc_kind) {
      int es = nhwc_kind == 2 ? 4 : 2;
      uint4* o = reinterpret_cast<uint4*>(static_cast<uint8_t*>(nhwc) + size_t(p) * MAP_TEXELS * cpad * es);
      for (int t = threadIdx.x; t < MAP_TEXELS * cpad * es / 16; t += blockDim.x) o[t] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) { s_r[p] = R(1); s_d[p] = R(1); }
    return;
  }
  const R* rp = rad + p * MAP_TEXELS * 3;
  const R* dp = dist + p * MAP_TEXELS;
  R dm = R(0);
  for (int t = threadIdx.x; t < MAP_TEXELS; t += blockDim.x) {
    lum[t] = (rp[3 * t] * R(LUMA_R) + rp[3 * t + 1] * R(LUMA_G)) + rp[3 * t + 2] * R(LUMA_B);
    dm = fmax(dm, dp[t]);
  }
  for (int off = 16; off > 0; off >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, off));
  if ((threadIdx.x & 31) == 0) dmax[threadIdx.x >> 5] = dm;
  __syncthreads();
  R sum = pairwise1024(lum, scratch);
  R sr = sum / R(MAP_TEXELS) + R(1e-3);
  R mx = dmax[0];
  for (int w = 1; w < 8; ++w) mx = fmax(mx, dmax[w]);
  R sd = mx > R(0) ? mx : R(1);
  const R* np_ = nloc + p * MAP_TEXELS * 3;
  for (int t = threadIdx.x; t < MAP_TEXELS; t += blockDim.x) {
    float v[8];
    for (int c = 0; c < 3; ++c) v[c] = float(rp[3 * t + c] / sr);
    for (int c = 0; c < 3; ++c) v[3 + c] = float(np_[3 * t + c]);
    v[6] = float(dp[t] / sd);
    v[7] = 0.f;
    if (stacks)
      for (int c = 0; c < 7; ++c) out[c * MAP_TEXELS + t] = v[c];
    if (nhwc_kind == 1 || nhwc_kind == 3) {
      uint32_t w[4];
      for (int j = 0; j < 4; ++j) {
        if (nhwc_kind == 1) {
          __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          w[j] = *reinterpret_cast<uint32_t*>(&b);
        } else {
          __half2 b = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
          w[j] = *reinterpret_cast<uint32_t*>(&b);
        }
      }
      reinterpret_cast<uint4*>(nhwc)[p * MAP_TEXELS + t] = make_uint4(w[0], w[1], w[2], w[3]);
    } else if (nhwc_kind == 2) {
      uint32_t w[8];
      for (int j = 0; j < 8; ++j) asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(w[j]) : "f"(v[j]));
      uint4* o = reinterpret_cast<uint4*>(nhwc) + 2 * (p * MAP_TEXELS + t);
      o[0] = make_uint4(w[0], w[1], w[2], w[3]);
      o[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
  if (threadIdx.x == 0) {
    s_r[p] = sr;
    s_d[p] = sd;
  }
}

// numpy remainder (floored modulo) for y > 0
template <typename R>
__device__ __forceinline__ R py_mod(R x, R y) {
  R m = fmod(x, y);
  if (m != R(0)) {
    if ((m < R(0)) != (y < R(0))) m += y;
  } else {
    m = copysign(R(0), y);
  }
  return m;
}

// _texels_from_local (hemimap.py:106-114)
template <typename R>
__device__ __forceinline__ bool texel_of(V3<R> l, int& u, int& v) {
  R z = fmin(fmax(l.z, R(-1)), R(1));
  bool valid = z >= R(0);
  R theta = acos(z);
  R phi = py_mod(atan2(l.y, l.x), R(2.0 * PI));
  long long uu = (long long)(phi / R(2.0 * PI) * R(MAP_RES));
  long long vv = (long long)(theta / R(PI / 2.0) * R(MAP_RES));
  u = int(uu < MAP_RES - 1 ? uu : MAP_RES - 1);
  v = int(vv < MAP_RES - 1 ? vv : MAP_RES - 1);
  if (!valid) { u = 0; v = 0; }
  return valid;
}

template <typename R>
__device__ __forceinline__ R texel_sin_theta(int v) {
  return sin(R(PI / 2.0) * (R(v) + R(0.5)) / R(MAP_RES));
}

// One WARP per cache point (SHADE_WARPS maps per block): the map's 2D
// distribution and the MIS shading estimate (integrators.py:564-614,
// hemimap.py:156-197). Arithmetic and summation orders are those of the
// reference's numpy calls: numpy's pairwise sum for the normaliser and the
// row masses, sequential cumsums for the row and column CDFs. The column CDF
// of a row is only needed for the rows that are sampled, so each map-sampling
// lane rebuilds its own row's CDF on the fly (the same divisions and adds the
// full table would hold) instead of storing 1,024 CDF values per map.
constexpr int SHADE_PITCH = MAP_RES + 1;  // padded rows: lane v reads row v conflict-free

template <typename R>
struct ShadeSmem {
  R prob[MAP_RES * SHADE_PITCH];
  R rows[MAP_RES];
  R sin_v[MAP_RES];
  R part[64];
};

template <typename R>
constexpr int shade_warps() { return sizeof(R) == 4 ? 8 : 4; }

template <typename R>
__global__ void __launch_bounds__(32 * shade_warps<R>()) k_shade(
    DevScene S, DrcbRenderCfg cfg, const float* __restrict__ pred, const R* __restrict__ s_r,
    const R* __restrict__ frames, const R* __restrict__ wo, const int32_t* __restrict__ mats,
    const uint64_t* __restrict__ keys, const uint8_t* __restrict__ live, int64_t n, R* Lout) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ ShadeSmem<R> sm_all[shade_warps<R>()];
  const int lane = threadIdx.x & 31;
  ShadeSmem<R>& sm = sm_all[threadIdx.x >> 5];
  const int64_t p = int64_t(blockIdx.x) * shade_warps<R>() + (threadIdx.x >> 5);
  if (p >= n) return;
  if (live && !live[p]) {
    if (lane < 3) Lout[3 * p + lane] = R(0);
    return;
  }
  const float* pd = pred + p * 3 * MAP_TEXELS;  // (3,32,32)
  const R scale = s_r[p];
  sm.sin_v[lane] = texel_sin_theta<R>(lane);
  __syncwarp();
  // weights w = lum * sin(theta_v) + 1e-8 (build_map_distribution); lane =
  // column u, so the loads of a row are coalesced
  for (int v = 0; v < MAP_RES; ++v) {
    const int t = v * MAP_RES + lane;
    R r = R(pd[t]) * scale, g = R(pd[MAP_TEXELS + t]) * scale, b = R(pd[2 * MAP_TEXELS + t]) * scale;
    R lum = (r * R(LUMA_R) + g * R(LUMA_G)) + b * R(LUMA_B);
    sm.prob[v * SHADE_PITCH + lane] = lum * sm.sin_v[v] + R(1e-8);
  }
  __syncwarp();
  // numpy pairwise sum of the 1,024 weights: 8 blocks of 128, each 8
  // strided accumulators of 16 terms, then the fixed trees
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h, blk = t >> 3, j = t & 7;
    R acc = R(0);
    for (int k = 0; k < 16; ++k) {
      const int f = 128 * blk + 8 * k + j;  // flat texel index
      const R w = sm.prob[(f >> 5) * SHADE_PITCH + (f & 31)];
      acc = (k == 0) ? w : acc + w;
    }
    sm.part[t] = acc;
  }
  __syncwarp();
  R B[8];
  for (int blk = 0; blk < 8; ++blk) {
    const R* q = sm.part + 8 * blk;
    B[blk] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
  }
  const R wsum = ((B[0] + B[1]) + (B[2] + B[3])) + ((B[4] + B[5]) + (B[6] + B[7]));
  __syncwarp();
  for (int v = 0; v < MAP_RES; ++v) sm.prob[v * SHADE_PITCH + lane] = sm.prob[v * SHADE_PITCH + lane] / wsum;
  __syncwarp();
  {  // row masses: numpy pairwise sum of 32 (8 accumulators, fixed tree)
    const R* a = sm.prob + lane * SHADE_PITCH;
    R q[8];
    for (int j = 0; j < 8; ++j) q[j] = a[j];
    for (int k = 8; k < 32; k += 8)
      for (int j = 0; j < 8; ++j) q[j] = q[j] + a[k + j];
    sm.rows[lane] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
  }
  __syncwarp();
  const R* F = frames + 9 * p;
  Frame<R> fr{ldr3(F), ldr3(F + 3), ldr3(F + 6)};
  V3<R> wo_local = fr.to_local(ldr3(wo + 3 * p));
  const int mat = mats[p];
  const int n_map = cfg.mis_samples / 2;
  const int n_bsdf = cfg.mis_samples - n_map;
  const R omega0 = (R(2.0 * PI) / R(MAP_RES)) * (R(PI) / (R(2) * R(MAP_RES)));
  PathRng rng;
  // map samples (lanes < n_map <= 32)
  V3<R> c = {R(0), R(0), R(0)};
  if (lane < n_map) {
    rng.init(cfg.seed, keys[p], uint64_t(lane), cfg.sampler_kind, 1u);
    R u1 = to_unit<R>(rng.sample(SHADE_DIM_BASE + 0));
    R u2 = to_unit<R>(rng.sample(SHADE_DIM_BASE + 1));
    // row: searchsorted(cumsum(rows), u1, side="right") with cdf[-1] = 1
    int v = 0;
    R acc = sm.rows[0];
    while (v < MAP_RES && (v == MAP_RES - 1 ? R(1) : acc) <= u1) {
      ++v;
      if (v < MAP_RES) acc = acc + sm.rows[v];
    }
    v = min(v, MAP_RES - 1);
    // column: count(cumsum(prob[v] / rows[v]) <= u2) with cdf[-1] = 1
    const R* row = sm.prob + v * SHADE_PITCH;
    const R rv = sm.rows[v];
    int u = 0;
    R cacc = R(0);
    for (int k = 0; k < MAP_RES; ++k) {
      R cc = row[k] / rv;
      cacc = (k == 0) ? cc : cacc + cc;
      u += ((k == MAP_RES - 1 ? R(1) : cacc) <= u2);
    }
    u = min(u, MAP_RES - 1);
    R pr = row[u];
    V3<R> dir = fr.to_world(texel_local<R>(u, v));
    R pdf = pr / (omega0 * sm.sin_v[v]);
    V3<R> radv = {R(pd[v * MAP_RES + u]) * scale, R(pd[MAP_TEXELS + v * MAP_RES + u]) * scale,
                  R(pd[2 * MAP_TEXELS + v * MAP_RES + u]) * scale};
    V3<R> li = fr.to_local(dir);
    V3<R> f;
    R pdf_b;
    bsdf_eval(S, mat, wo_local, li, f, pdf_b);
    R cos_i = fmax(li.z, R(0));
    R w = power_heuristic(pdf, pdf_b);
    R k = (w * cos_i) / pdf;
    c = (f * radv) * mk<R>(k, k, k);
  }
  // BSDF samples (lanes < n_bsdf <= 32)
  V3<R> cb = {R(0), R(0), R(0)};
  if (lane < n_bsdf) {
    rng.init(cfg.seed, keys[p], uint64_t(lane), cfg.sampler_kind, 1u);
    R u1 = to_unit<R>(rng.sample(SHADE_DIM_BASE + 2));
    R u2 = to_unit<R>(rng.sample(SHADE_DIM_BASE + 3));
    BsdfSample<R> bs = bsdf_sample(S, mat, wo_local, u1, u2, true);
    int u, v;
    bool valid = texel_of(bs.li, u, v);
    V3<R> radv = {R(0), R(0), R(0)};
    R pdf_m = R(0);
    if (valid) {
      int q = v * MAP_RES + u;
      radv = {R(pd[q]) * scale, R(pd[MAP_TEXELS + q]) * scale, R(pd[2 * MAP_TEXELS + q]) * scale};
      pdf_m = sm.prob[v * SHADE_PITCH + u] / (omega0 * sm.sin_v[v]);
    }
    R cos_i = fmax(bs.li.z, R(0));
    R w = power_heuristic(bs.pdf, pdf_m);
    R k = (w * cos_i) / bs.pdf;
    cb = (bs.value * radv) * mk<R>(k, k, k);
  }
  // sequential sums in sample order (lane 0 collects)
  V3<R> sm_ = {R(0), R(0), R(0)}, sb = {R(0), R(0), R(0)};
  for (int k = 0; k < 32; ++k) {
    V3<R> a = {__shfl_sync(FULL, c.x, k), __shfl_sync(FULL, c.y, k), __shfl_sync(FULL, c.z, k)};
    V3<R> b = {__shfl_sync(FULL, cb.x, k), __shfl_sync(FULL, cb.y, k), __shfl_sync(FULL, cb.z, k)};
    if (k < n_map) sm_ = (k == 0) ? a : sm_ + a;
    if (k < n_bsdf) sb = (k == 0) ? b : sb + b;
  }
  if (lane == 0) {
    V3<R> total = divs(sm_, R(n_map));
    total = total + divs(sb, R(n_bsdf));
    if (!all_finite(total)) total = {R(0), R(0), R(0)};
    st3(Lout + 3 * p, total);
  }
}

// ---------------------------------------------------------------------------
// interpolation: entries bucketed on a screen grid (replaces cKDTree,
// cache.py:205-208, 305-307); exact predicates of the reference:
//   d1 = sqrt(min dx^2+dy^2), r_eff = max(r, 1.5 d1),
//   gather dx^2+dy^2 <= (2 r_eff)^2, w = w_p w_n + w_p + 1e-4.
constexpr int BUCKET = 16;

__global__ void k_bucket_count(const int32_t* px, const int32_t* py, int64_t m, const int* m_dev,
                               int nbx, int* counts) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= (m_dev ? int64_t(*m_dev) : m)) return;
  atomicAdd(&counts[(py[i] / BUCKET) * nbx + px[i] / BUCKET], 1);
}

__global__ void k_bucket_fill(const int32_t* px, const int32_t* py, int64_t m, const int* m_dev,
                              int nbx, const int* offsets, int* cursor, int* items) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= (m_dev ? int64_t(*m_dev) : m)) return;
  int b = (py[i] / BUCKET) * nbx + px[i] / BUCKET;
  int slot = atomicAdd(&cursor[b], 1);
  items[offsets[b] + slot] = int(i);
}

// ascending entry order inside each bucket (determinism)
__global__ void k_bucket_sort(const int* offsets, int nb, int* items) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  int s = offsets[b], e = offsets[b + 1];
  for (int i = s + 1; i < e; ++i) {
    int v = items[i];
    int j = i - 1;
    while (j >= s && items[j] > v) {
      items[j + 1] = items[j];
      --j;
    }
    items[j + 1] = v;
  }
}

// the entries' pixel, normal and radiance copied into item order once per
// frame (m <= 65,536 entries): the interpolation's gather loops then read
// consecutive records instead of an index followed by dependent loads of
// three SoA tables (same values, same order: bit-identical)
template <typename R>
struct alignas(4 * sizeof(R)) Rec4 {
  R x, y, z, w;
};
template <typename R>
__global__ void k_bucket_gather(const int* __restrict__ items, int64_t m, const int* m_dev,
                                const int32_t* __restrict__ epx, const int32_t* __restrict__ epy,
                                const R* __restrict__ en, const R* __restrict__ erad, int2* ipx,
                                Rec4<R>* inrm, Rec4<R>* irad) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= (m_dev ? int64_t(*m_dev) : m)) return;
  const int e = items[q];
  ipx[q] = make_int2(epx[e], epy[e]);
  inrm[q] = Rec4<R>{en[3 * e], en[3 * e + 1], en[3 * e + 2], R(0)};
  irad[q] = Rec4<R>{erad[3 * e], erad[3 * e + 1], erad[3 * e + 2], R(0)};
}

// `items` is bucket-major and the buckets of a grid row are consecutive, so
// the entries of buckets [bx0, bx1] of row yy are ONE contiguous range of
// items: the gather loops run per bucket row, in exactly the bucket/entry
// order of a per-bucket loop (same sums), without per-bucket loop overhead.
template <typename R>
__global__ void __launch_bounds__(TPB) k_interp(DevScene S, int W, int H, DrcbGBuffer gb,
                                                 const int2* __restrict__ ipx,
                                                 const Rec4<R>* __restrict__ inrm,
                                                 const Rec4<R>* __restrict__ irad, int64_t m_cap,
                                                 const int* __restrict__ m_dev, int r,
                                                 int nbx, int nby, const int* __restrict__ off,
                                                 const R* __restrict__ direct, R* image) {
  // a block is a 16 x (TPB/16) pixel tile inside one bucket column: a warp's
  // 16x2 pixels share their bucket ranges (uniform loop bounds)
  const int x = int(blockIdx.x) * BUCKET + int(threadIdx.x % BUCKET);
  const int y = int(blockIdx.y) * (TPB / BUCKET) + int(threadIdx.x / BUCKET);
  if (x >= W || y >= H) return;
  const int64_t i = int64_t(y) * W + x;
  const int64_t m = m_dev ? int64_t(*m_dev) : m_cap;
  V3<R> layer = {R(0), R(0), R(0)};
  V3<R> thr = ldr3(static_cast<const R*>(gb.throughput) + 3 * i);
  if (gb.escaped[i] && S.has_env) layer = thr * ld3<R>(S.env);
  if (gb.found[i] && m > 0) {
    const int bx = x / BUCKET, by = y / BUCKET;
    // nearest entry by expanding Chebyshev rings of buckets
    long long best = LLONG_MAX;
    const int maxring = max(nbx, nby);
    auto scan = [&](int q0, int q1) {
#pragma unroll 1
      for (int q = q0; q < q1; ++q) {
        const int2 pe = ipx[q];
        const long long dx = pe.x - x, dy = pe.y - y;
        const long long d2 = dx * dx + dy * dy;
        if (d2 < best) best = d2;
      }
    };
    for (int k = 0; k <= maxring; ++k) {
      const int xa = max(bx - k, 0), xb = min(bx + k, nbx - 1);
      for (int yy = max(by - k, 0); yy <= min(by + k, nby - 1); ++yy) {
        const int row = yy * nbx;
        if (yy == by - k || yy == by + k) {
          scan(off[row + xa], off[row + xb + 1]);  // a whole ring row
        } else {
          if (bx - k >= 0) scan(off[row + bx - k], off[row + bx - k + 1]);
          if (k > 0 && bx + k < nbx) scan(off[row + bx + k], off[row + bx + k + 1]);
        }
      }
      const long long lim = (long long)k * BUCKET + 1;
      if (best != LLONG_MAX && best <= lim * lim) break;
    }
    const R d1 = sqrt(R(best));
    const R r_eff = fmax(R(r), R(1.5) * d1);
    const R rad = R(2) * r_eff;
    const R rad2 = rad * rad;
    const V3<R> npx = ldr3(static_cast<const R*>(gb.normal) + 3 * i);
    const int reach = int(ceil(double(rad))) + 1;
    const int bx0 = max(0, (x - reach) / BUCKET), bx1 = min(nbx - 1, (x + reach) / BUCKET);
    const int by0 = max(0, (y - reach) / BUCKET), by1 = min(nby - 1, (y + reach) / BUCKET);
    V3<R> num = {R(0), R(0), R(0)};
    R den = R(0);
    for (int yy = by0; yy <= by1; ++yy) {
      const int q1 = off[yy * nbx + bx1 + 1];
#pragma unroll 1
      for (int q = off[yy * nbx + bx0]; q < q1; ++q) {
        const int2 pe = ipx[q];
        const R dx = R(pe.x - x), dy = R(pe.y - y);
        const R d2 = dx * dx + dy * dy;
        if (!(d2 <= rad2)) continue;
        const R dist = sqrt(d2);
        const R w_p = fmax(R(0), R(1) - dist / r_eff);
        const Rec4<R> ne = inrm[q];
        const R w_n = fmax(R(0), dot(V3<R>{ne.x, ne.y, ne.z}, npx));
        const R wgt = (w_p * w_n + w_p) + R(1e-4);
        const Rec4<R> le = irad[q];
        num = num + wgt * V3<R>{le.x, le.y, le.z};
        den = den + wgt;
      }
    }
    if (den > R(0)) layer = thr * divs(num, den);
  }
  V3<R> out = layer;
  if (direct) out = ldr3(direct + 3 * i) + layer;
  st3(image + 3 * i, out);
}

}  // namespace DRCB_RENDER_NS
using namespace DRCB_RENDER_NS;

// ---------------------------------------------------------------------------
// launchers

#define LAUNCH_CHECK()                                                    \
  do {                                                                    \
    count_launch();                                                       \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return cuda_fail(_e, __func__);                \
  } while (0)

template <typename R>
int launch_intersect(const DevScene& S, const R* O, const R* D, int64_t n, const R* tmin,
                     const R* tmax, int record, uint8_t* hit, R* t, int64_t* prim, int32_t* mat,
                     R* pos, R* nrm, cudaStream_t st) {
  if (n <= 0) return 0;
  k_intersect<R><<<nblocks(n), TPB, 0, st>>>(S, O, D, n, tmin, tmax, record, hit, t, prim, mat,
                                              pos, nrm);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_primary_chain(const DevScene& S, const R* O, const R* D, int64_t n,
                         const DrcbGBuffer& gb, cudaStream_t st) {
  if (n <= 0) return 0;
  k_primary_chain<R><<<nblocks(n), TPB, 0, st>>>(S, O, D, n, gb);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_li_direct(const DevScene& S, const DrcbRenderCfg& cfg, const R* O, const R* D,
                     const uint64_t* pix, const uint64_t* smp, int64_t n, int include_bg, R* L,
                     int64_t* nonfinite, cudaStream_t st) {
  if (n <= 0) return 0;
  k_li_direct<R><<<nblocks(n), TPB, 0, st>>>(S, cfg, O, D, pix, smp, n, include_bg, L, nonfinite);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_trace_radiance(const DevScene& S, const DrcbRenderCfg& cfg, const R* O, const R* D,
                          const uint64_t* pix, const uint64_t* smp, int64_t n, int max_depth,
                          int skip_first, int rr_start, R* L, int64_t* nonfinite,
                          cudaStream_t st) {
  if (n <= 0) return 0;
  k_trace<R><<<nblocks(n), TPB, 0, st>>>(S, cfg, O, D, pix, smp, n, max_depth, skip_first,
                                          rr_start, L, nonfinite);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_gbuffer_direct(const DevScene& S, const DevCamera& C, const DrcbRenderCfg& cfg,
                          int tile, const DrcbGBuffer& gb, R* direct, int64_t* nonfinite,
                          cudaStream_t st) {
  int64_t n = int64_t(C.W) * C.H;
  if (n <= 0) return 0;
  const int spp = cfg.direct_spp;
  if (spp == 1 && getenv("DRCB_SPLIT_DIRECT") == nullptr) {
    k_gbuffer_direct1<R><<<nblocks(n), TPB, 0, st>>>(S, C, cfg, gb, direct, nonfinite);
    LAUNCH_CHECK();
    return 0;
  }
  k_gbuffer<R><<<nblocks(n), TPB, 0, st>>>(S, C, gb);
  LAUNCH_CHECK();
  R* samples = nullptr;
  DRCB_CUDA(cudaMallocAsync((void**)&samples, sizeof(R) * 3 * size_t(n) * spp, st));
  k_direct_samples<R><<<nblocks(n * spp), TPB, 0, st>>>(S, C, cfg, samples, nonfinite);
  LAUNCH_CHECK();
  k_direct_reduce<R><<<nblocks(n), TPB, 0, st>>>(C, spp, tile, samples, direct);
  LAUNCH_CHECK();
  DRCB_CUDA(cudaFreeAsync(samples, st));
  return 0;
}

template <typename R>
int launch_render_stacks(const DevScene& S, const DrcbRenderCfg& cfg, const R* pos, const R* nrm,
                         const uint64_t* keys, const uint8_t* live, int64_t n, float* stacks,
                         R* s_r, R* s_d, R* frames, int64_t* nonfinite, cudaStream_t st,
                         void* nhwc, int nhwc_kind, int cpad) {
  if (n <= 0) return 0;
  size_t per = size_t(n) * MAP_TEXELS;
  R* scratch = nullptr;
  DRCB_CUDA(cudaMallocAsync((void**)&scratch, per * 7 * sizeof(R) + 64 + size_t(n) * 8, st));
  R* rad = scratch;
  R* dist = scratch + 3 * per;
  R* nloc = scratch + 4 * per;
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(scratch + 7 * per);
  uint64_t* pre2 = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(scratch + 7 * per) + 64);
  DRCB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  k_point_frames<R><<<nblocks(n), TPB, 0, st>>>(S, nrm, n, frames, keys, cfg.seed, pre2);
  LAUNCH_CHECK();
  // the table is filled once, synchronously, outside any graph capture (the
  // path kernel evaluates texel_local itself until then: frames on other
  // streams must never see a half-written table)
  // per precision (one instantiation each) and per device (each device has
  // its own copy of the __device__ table)
  static DeviceFlags dirs_flags;
  const int dev = current_device();
  bool dirs_ready = dirs_flags.test(dev);
  if (!dirs_ready) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      k_texel_dirs<R><<<nblocks(MAP_TEXELS), TPB, 0, st>>>();
      LAUNCH_CHECK();
      DRCB_CUDA(cudaStreamSynchronize(st));
      dirs_flags.set(dev);
      dirs_ready = true;
    }
  }
  // persistent grid: resident CTAs per SM x SMs of this device
  static std::atomic<int> grid_dev[64];
  int grid = grid_dev[dev & 63].load(std::memory_order_relaxed);
  if (!grid) {
    int per_sm = 0;
    // the casting kernels use no shared memory and live on L1 hits: ask for
    // the largest L1 (maps 3.58 ms at 0 % shared, 3.71 at 50 %, 4.27 at 100 %)
    cudaFuncSetAttribute(k_map_paths<R>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaFuncSetAttribute(k_gbuffer_direct1<R>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_map_paths<R>, MAP_TPB, 0);
    if (const char* e = getenv("DRCB_MAP_PER_SM")) per_sm = std::min(per_sm, std::max(1, atoi(e)));
    grid = sm_count() * (per_sm > 0 ? per_sm : 1);
    grid_dev[dev & 63].store(grid, std::memory_order_relaxed);
  }
  int64_t total = int64_t(per);
  int g = int(std::min<int64_t>(grid, (total + MAP_TPB - 1) / MAP_TPB));
  k_map_paths<R><<<g, MAP_TPB, 0, st>>>(S, cfg, pos, nrm, keys, live, total, counter, rad, dist,
                                         nloc, nonfinite, dirs_ready ? 1 : 0, frames, pre2);
  LAUNCH_CHECK();
  k_stack_normalize<R><<<int(n), 256, 0, st>>>(rad, dist, nloc, live, n, stacks, s_r, s_d, nhwc,
                                                nhwc_kind, cpad);
  LAUNCH_CHECK();
  DRCB_CUDA(cudaFreeAsync(scratch, st));
  return 0;
}

template <typename R>
int launch_shade(const DevScene& S, const DrcbRenderCfg& cfg, const float* pred, const R* s_r,
                 const R* frames, const R* wo, const int32_t* mat, const uint64_t* keys,
                 const uint8_t* live, int64_t n, R* L, cudaStream_t st) {
  if (n <= 0) return 0;
  if (cfg.mis_samples < 2 || cfg.mis_samples > 64)
    return fail(DRCB_ECONFIG, "mis_samples must be in [2, 64]");
  constexpr int wpb = shade_warps<R>();
  k_shade<R><<<int((n + wpb - 1) / wpb), 32 * wpb, 0, st>>>(S, cfg, pred, s_r, frames, wo, mat,
                                                          keys, live, n, L);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_interp_composite(const DevScene& S, int W, int H, const DrcbGBuffer& gb,
                            const int32_t* e_px, const int32_t* e_py, const R* e_n,
                            const R* e_rad, int64_t m, const int* m_dev, int r, const R* direct,
                            R* image, cudaStream_t st) {
  int nbx = (W + BUCKET - 1) / BUCKET, nby = (H + BUCKET - 1) / BUCKET;
  int nb = nbx * nby;
  int* buf = nullptr;
  size_t mm = size_t(m > 0 ? m : 1);
  DRCB_CUDA(cudaMallocAsync((void**)&buf, sizeof(int) * (3 * size_t(nb) + 2 + mm), st));
  int* counts = buf;
  int* offsets = buf + nb + 1;     // nb + 1
  int* cursor = offsets + nb + 1;  // nb
  int* items = cursor + nb;        // m
  DRCB_CUDA(cudaMemsetAsync(buf, 0, sizeof(int) * (3 * size_t(nb) + 2), st));
  if (m > 0) {
    k_bucket_count<<<nblocks(m), TPB, 0, st>>>(e_px, e_py, m, m_dev, nbx, counts);
    LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, nb + 1, st);
    void* tmp = nullptr;
    DRCB_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offsets, nb + 1, st);
    count_launch(2);
    DRCB_CUDA(cudaFreeAsync(tmp, st));
    k_bucket_fill<<<nblocks(m), TPB, 0, st>>>(e_px, e_py, m, m_dev, nbx, offsets, cursor, items);
    LAUNCH_CHECK();
    k_bucket_sort<<<nblocks(nb), TPB, 0, st>>>(offsets, nb, items);
    LAUNCH_CHECK();
  }
  Rec4<R>* recs = nullptr;  // inrm (m), irad (m), then ipx (m)
  DRCB_CUDA(cudaMallocAsync((void**)&recs, (2 * sizeof(Rec4<R>) + sizeof(int2)) * mm, st));
  Rec4<R>* inrm = recs;
  Rec4<R>* irad = recs + mm;
  int2* ipx = reinterpret_cast<int2*>(recs + 2 * mm);
  if (m > 0) {
    k_bucket_gather<R><<<nblocks(m), TPB, 0, st>>>(items, m, m_dev, e_px, e_py, e_n, e_rad, ipx, inrm,
                                                    irad);
    LAUNCH_CHECK();
  }
  const dim3 igrid(unsigned(nbx), unsigned((H + TPB / BUCKET - 1) / (TPB / BUCKET)));
  k_interp<R><<<igrid, TPB, 0, st>>>(S, W, H, gb, ipx, inrm, irad, m, m_dev, r, nbx, nby, offsets,
                                     direct, image);
  LAUNCH_CHECK();
  DRCB_CUDA(cudaFreeAsync(recs, st));
  DRCB_CUDA(cudaFreeAsync(buf, st));
  return 0;
}

template <typename R>
int launch_pt_frame(const DevScene& S, const DevCamera& C, const DrcbRenderCfg& cfg, int spp,
                    int tile, R* image, int64_t* nonfinite, cudaStream_t st) {
  int64_t n = int64_t(C.W) * C.H;
  if (n <= 0) return 0;
  k_pt_frame<R><<<nblocks(n), TPB, 0, st>>>(S, C, cfg, spp, tile, image, nonfinite);
  LAUNCH_CHECK();
  return 0;
}

template <typename R>
int launch_reference_map(const DevScene& S, const DrcbRenderCfg& cfg, const R* pos, const R* nrm,
                         uint64_t key, int ref_spp, R* out, int64_t* nonfinite, cudaStream_t st) {
  const int chunk = std::max(1, (1 << 14) / MAP_TEXELS);  // dataset.py:114
  const int nchunks = (ref_spp + chunk - 1) / chunk;
  // groups of whole chunks whose per-path radiance fits 256 MB
  const int64_t per_chunk = int64_t(chunk) * MAP_TEXELS * 3 * int64_t(sizeof(R));
  const int gchunks = int(std::max<int64_t>(1, std::min<int64_t>(nchunks, (int64_t(256) << 20) / per_chunk)));
  const int gs = std::min(ref_spp, gchunks * chunk);
  R* paths = nullptr;
  DRCB_CUDA(cudaMallocAsync((void**)&paths, sizeof(R) * 3 * (size_t(gs) + 1) * MAP_TEXELS, st));
  R* tot = paths + 3 * size_t(gs) * MAP_TEXELS;
  for (int c0 = 0; c0 < nchunks; c0 += gchunks) {
    const int c1 = std::min(nchunks, c0 + gchunks);
    const int s0 = c0 * chunk, s1 = std::min(ref_spp, c1 * chunk);
    k_reference_paths<R><<<nblocks(int64_t(s1 - s0) * MAP_TEXELS), TPB, 0, st>>>(
        S, cfg, pos, nrm, key, ref_spp, s0, s1 - s0, paths, nonfinite);
    LAUNCH_CHECK();
    k_reference_reduce<R><<<nblocks(MAP_TEXELS), TPB, 0, st>>>(paths, s0, chunk, c0, c1, ref_spp,
                                                               tot, out, c1 == nchunks ? 1 : 0);
    LAUNCH_CHECK();
  }
  DRCB_CUDA(cudaFreeAsync(paths, st));
  return 0;
}

#define INST(R)                                                                                  \
  template int launch_intersect<R>(const DevScene&, const R*, const R*, int64_t, const R*,      \
                                   const R*, int, uint8_t*, R*, int64_t*, int32_t*, R*, R*,     \
                                   cudaStream_t);                                                \
  template int launch_primary_chain<R>(const DevScene&, const R*, const R*, int64_t,            \
                                       const DrcbGBuffer&, cudaStream_t);                        \
  template int launch_li_direct<R>(const DevScene&, const DrcbRenderCfg&, const R*, const R*,   \
                                   const uint64_t*, const uint64_t*, int64_t, int, R*, int64_t*, \
                                   cudaStream_t);                                                \
  template int launch_trace_radiance<R>(const DevScene&, const DrcbRenderCfg&, const R*,        \
                                        const R*, const uint64_t*, const uint64_t*, int64_t,    \
                                        int, int, int, R*, int64_t*, cudaStream_t);              \
  template int launch_gbuffer_direct<R>(const DevScene&, const DevCamera&,                      \
                                        const DrcbRenderCfg&, int, const DrcbGBuffer&, R*,      \
                                        int64_t*, cudaStream_t);                                 \
  template int launch_render_stacks<R>(const DevScene&, const DrcbRenderCfg&, const R*,         \
                                       const R*, const uint64_t*, const uint8_t*, int64_t,      \
                                       float*, R*, R*, R*, int64_t*, cudaStream_t, void*, int,  \
                                       int);                                                     \
  template int launch_shade<R>(const DevScene&, const DrcbRenderCfg&, const float*, const R*,   \
                               const R*, const R*, const int32_t*, const uint64_t*,             \
                               const uint8_t*, int64_t, R*, cudaStream_t);                       \
  template int launch_interp_composite<R>(const DevScene&, int, int, const DrcbGBuffer&,        \
                                          const int32_t*, const int32_t*, const R*, const R*,   \
                                          int64_t, const int*, int, const R*, R*, cudaStream_t);

// One source, two objects (Makefile): the fp64 parity build with -fmad=false
// (numpy's unfused arithmetic, bit-exact against the reference) and the fp32
// build with the compiler's FMA contraction.
#if DRCB_RENDER_PREC == 32
INST(float)
template int launch_pt_frame<float>(const DevScene&, const DevCamera&, const DrcbRenderCfg&, int,
                                    int, float*, int64_t*, cudaStream_t);
template int launch_reference_map<float>(const DevScene&, const DrcbRenderCfg&, const float*,
                                         const float*, uint64_t, int, float*, int64_t*,
                                         cudaStream_t);

int launch_intersect_mixed(const DevScene& S, const double* O, const double* D, int64_t n,
                           const double* tmin, const double* tmax, int record, uint8_t* hit,
                           double* t, int64_t* prim, int32_t* mat, double* pos, double* nrm,
                           cudaStream_t st) {
  if (n <= 0) return 0;
  DRCB_RENDER_NS::k_intersect_mixed<<<DRCB_RENDER_NS::nblocks(n), DRCB_RENDER_NS::TPB, 0, st>>>(
      S, O, D, n, tmin, tmax, record, hit, t, prim, mat, pos, nrm);
  LAUNCH_CHECK();
  return 0;
}

// the fp32 module's copy of the traversal-counter pointer
int set_trav_stats_f32(unsigned long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_trav_stats, &buf, sizeof(buf));
  return e == cudaSuccess ? 0 : cuda_fail(e, "drcb_trav_stats");
}
}  // namespace drcb
#else
INST(double)
template int launch_pt_frame<double>(const DevScene&, const DevCamera&, const DrcbRenderCfg&, int,
                                     int, double*, int64_t*, cudaStream_t);
template int launch_reference_map<double>(const DevScene&, const DrcbRenderCfg&, const double*,
                                          const double*, uint64_t, int, double*, int64_t*,
                                          cudaStream_t);
int set_trav_stats_f32(unsigned long long* buf);
}  // namespace drcb

// arm (buf != NULL, device u64[12] counters) or disarm the traversal counters
// of both arithmetic builds
extern "C" int drcb_trav_stats(unsigned long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(drcb::g_trav_stats, &buf, sizeof(buf));
  if (e != cudaSuccess) return drcb::cuda_fail(e, "drcb_trav_stats");
  return drcb::set_trav_stats_f32(buf);
}
#endif
