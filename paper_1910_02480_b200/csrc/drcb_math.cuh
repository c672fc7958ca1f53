// drcb_math.cuh — Real-templated 3-vector arithmetic and the keyed sampler.
//
// Operation order mirrors the reference's numpy expressions so that the
// fp64 build reproduces them up to libm last-ulp differences; this TU is
// compiled with -fmad=false so no FMA contraction changes rounding.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define DRCB_HD __host__ __device__ __forceinline__

namespace drcb {

constexpr double T_EPS = 1e-4;                 // drc/geometry.py:22
constexpr int SPECULAR_CHAIN_BOUND = 16;       // drc/integrators.py:35
constexpr double SPECULAR_THROUGHPUT_CUTOFF = 1e-4;  // integrators.py:36
constexpr double RR_FLOOR = 0.05;              // integrators.py:37
constexpr uint64_t SHADE_DIM_BASE = 1ull << 20;  // integrators.py:38
constexpr double UP_DEGENERACY = 1.0 - 1e-4;   // drc/bsdf.py:27
constexpr double PI = 3.141592653589793;
constexpr int MAP_RES = 32;
constexpr int MAP_TEXELS = MAP_RES * MAP_RES;

template <typename R>
struct V3 {
  R x, y, z;
};

template <typename R>
DRCB_HD V3<R> mk(R x, R y, R z) { return V3<R>{x, y, z}; }
template <typename R>
DRCB_HD V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <typename R>
DRCB_HD V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <typename R>
DRCB_HD V3<R> operator-(V3<R> a) { return {-a.x, -a.y, -a.z}; }
template <typename R>
DRCB_HD V3<R> operator*(R s, V3<R> a) { return {s * a.x, s * a.y, s * a.z}; }
template <typename R>
DRCB_HD V3<R> operator*(V3<R> a, V3<R> b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
template <typename R>
DRCB_HD V3<R> divs(V3<R> a, R s) { return {a.x / s, a.y / s, a.z / s}; }
// (a0*b0 + a1*b1) + a2*b2 — the _dot3 / _dot_rows order (geometry.py:193)
template <typename R>
DRCB_HD R dot(V3<R> a, V3<R> b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
// np.cross component formulas
template <typename R>
DRCB_HD V3<R> cross(V3<R> a, V3<R> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <typename R>
DRCB_HD R norm(V3<R> a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
template <typename R>
DRCB_HD bool any_pos(V3<R> a) { return a.x > R(0) || a.y > R(0) || a.z > R(0); }
template <typename R>
DRCB_HD bool all_finite(V3<R> a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
template <typename R>
DRCB_HD R maxc(V3<R> a) {
  // numpy max propagates nan
  R m = a.x;
  if (!(m >= a.y)) m = (isnan(m) ? m : a.y);
  if (!(m >= a.z)) m = (isnan(m) ? m : a.z);
  return m;
}
template <typename R, typename S>
DRCB_HD V3<R> cvt(V3<S> a) { return {R(a.x), R(a.y), R(a.z)}; }
template <typename R>
DRCB_HD V3<R> ld3(const double* p) { return {R(p[0]), R(p[1]), R(p[2])}; }
template <typename R>
DRCB_HD V3<R> ldr3(const R* p) { return {p[0], p[1], p[2]}; }
template <typename R>
DRCB_HD void st3(R* p, V3<R> v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }

// ---------------------------------------------------------------------------
// keyed stateless sampler (drc/sampler.py:17-78): splitmix-style uint64 mix
constexpr uint64_t M1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t M2 = 0x94D049BB133111EBull;
constexpr uint64_t SEED0 = 0x853C49E6748FEA9Bull;

DRCB_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * M1;
  z = (z ^ (z >> 27)) * M2;
  return z ^ (z >> 31);
}
DRCB_HD uint64_t hash_step(uint64_t h, uint64_t k) { return mix64((h * M2) ^ k); }
DRCB_HD double u53(uint64_t h) { return double(h >> 11) * 1.1102230246251565e-16; }  // 2^-53

// Sampler bound to (seed, pixel key, sample index); prefix of the hash chain
// is cached so each dimension costs one mix (sampler.py:31-37).
struct PathRng {
  uint64_t seed, pix, smp, prefix;
  uint32_t spp;
  int kind;  // 0 independent, 1 stratified
  DRCB_HD void init(uint64_t seed_, uint64_t pix_, uint64_t smp_, int kind_, uint32_t spp_) {
    seed = seed_; pix = pix_; smp = smp_; kind = kind_; spp = spp_;
    prefix = hash_step(hash_step(hash_step(SEED0, seed), pix), smp);
  }
  // the same, with hash_step(hash_step(SEED0, seed), pix) precomputed
  DRCB_HD void init_pre(uint64_t pre2, uint64_t seed_, uint64_t pix_, uint64_t smp_, int kind_,
                        uint32_t spp_) {
    seed = seed_; pix = pix_; smp = smp_; kind = kind_; spp = spp_;
    prefix = hash_step(pre2, smp);
  }
  DRCB_HD double sample(uint64_t dim) const {
    double jitter = u53(hash_step(prefix, dim));
    if (kind == 0 || spp == 1) return jitter;
    uint64_t n = spp;
    uint64_t off = hash_step(hash_step(hash_step(hash_step(SEED0, seed), pix), dim), 0xD1Full) % n;
    uint64_t stratum = (smp + off) % n;
    return (double(stratum) + jitter) / double(spp);
  }
};

// fp64 uniform -> R, never rounding up to 1
template <typename R>
DRCB_HD R to_unit(double u) { return R(u); }
template <>
DRCB_HD float to_unit<float>(double u) {
  float f = float(u);
  return f < 1.0f ? f : 0x1.fffffep-1f;
}

}  // namespace drcb
