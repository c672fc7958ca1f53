// drcb_trace.cuh — per-ray device code: BVH traversal, primitive tests,
// BSDFs, light sampling and the three path estimators, templated on the
// arithmetic type R (double = parity build, float = fast build).
//
// The reference runs these as numpy wavefronts over ray batches
// (drc/integrators.py, drc/geometry.py, drc/bsdf.py); here each CUDA thread
// walks one path to completion (a persistent "megakernel" loop), which keeps
// per-path state in registers instead of compacting HBM arrays per segment.
#pragma once
#include <type_traits>

#include "drcb_math.cuh"
#include "drcb_scene.cuh"

namespace drcb {

// fp64 with every operation explicitly rounded (no FMA contraction): the
// fp32 build's near-tie re-tests compute exactly what the -fmad=false fp64
// build (and numpy) computes, although their translation unit contracts
struct Dn {
  double v;
  __device__ __forceinline__ Dn() = default;
  __device__ __forceinline__ constexpr Dn(double x) : v(x) {}
};
__device__ __forceinline__ Dn operator+(Dn a, Dn b) { return Dn(__dadd_rn(a.v, b.v)); }
__device__ __forceinline__ Dn operator-(Dn a, Dn b) { return Dn(__dsub_rn(a.v, b.v)); }
__device__ __forceinline__ Dn operator-(Dn a) { return Dn(-a.v); }
__device__ __forceinline__ Dn operator*(Dn a, Dn b) { return Dn(__dmul_rn(a.v, b.v)); }
__device__ __forceinline__ Dn operator/(Dn a, Dn b) { return Dn(__ddiv_rn(a.v, b.v)); }
__device__ __forceinline__ bool operator<(Dn a, Dn b) { return a.v < b.v; }
__device__ __forceinline__ bool operator>(Dn a, Dn b) { return a.v > b.v; }
__device__ __forceinline__ bool operator<=(Dn a, Dn b) { return a.v <= b.v; }
__device__ __forceinline__ bool operator>=(Dn a, Dn b) { return a.v >= b.v; }
using ::fabs;  // the Dn overloads below must not hide the float / double ones
using ::sqrt;
__device__ __forceinline__ Dn fabs(Dn a) { return Dn(::fabs(a.v)); }
__device__ __forceinline__ Dn sqrt(Dn a) { return Dn(__dsqrt_rn(a.v)); }

template <typename R>
struct HitRec {
  R t;
  int prim;  // -1 = miss
};

// ---------------------------------------------------------------------------
// primitive tests (drc/geometry.py:233-286 batch form, 468-523 scalar form)

template <typename R>
__device__ __forceinline__ bool sphere_t(const DevScene& S, int i, V3<R> O, V3<R> D, R tmin,
                                         R tmax, R& tout) {
  const double* s = S.sph + 5 * i;
  V3<R> oc = O - ld3<R>(s);
  R b = dot(oc, D);
  R c = dot(oc, oc) - R(s[4]);
  R disc = b * b - c;
  if (!(disc >= R(0))) return false;
  R sq = sqrt(disc);
  R t0 = -b - sq, t1 = -b + sq;
  R t = (t0 > tmin) ? t0 : t1;
  if (t > tmin && t <= tmax) { tout = t; return true; }
  return false;
}

template <typename R>
__device__ __forceinline__ bool quad_t(const DevScene& S, int i, V3<R> O, V3<R> D, R tmin,
                                       R tmax, R& tout) {
  const double* q = S.quad + 18 * i;
  V3<R> n = ld3<R>(q + 9);
  R denom = dot(D, n);
  if (!(fabs(denom) > R(1e-12))) return false;
  R t = (R(q[15]) - dot(O, n)) / denom;
  if (!(t > tmin && t <= tmax)) return false;
  V3<R> eu = ld3<R>(q + 3), ev = ld3<R>(q + 6);
  R meu = (dot(O, eu) - R(q[16])) + t * dot(D, eu);
  R mev = (dot(O, ev) - R(q[17])) + t * dot(D, ev);
  R iuu = R(q[12]), iuv = R(q[13]), ivv = R(q[14]);
  R a = iuu * meu + iuv * mev;
  R b2 = iuv * meu + ivv * mev;
  if (a >= R(0) && a <= R(1) && b2 >= R(0) && b2 <= R(1)) { tout = t; return true; }
  return false;
}

// Moller-Trumbore exactly as geometry.py:271-286
template <typename R>
__device__ __forceinline__ bool tri_t(V3<R> v0, V3<R> e1, V3<R> e2, V3<R> O, V3<R> D, R tmin,
                                      R tmax, R& tout) {
  V3<R> pv = cross(D, e2);
  R det = dot(pv, e1);
  if (!(fabs(det) > R(1e-14))) return false;
  R inv = R(1) / det;
  V3<R> tv = O - v0;
  R u = dot(tv, pv) * inv;
  if (!(u >= R(0) && u <= R(1))) return false;
  V3<R> qv = cross(tv, e1);
  R v = dot(qv, D) * inv;
  if (!(v >= R(0) && u + v <= R(1))) return false;
  R t = dot(qv, e2) * inv;
  if (t > tmin && t <= tmax) { tout = t; return true; }
  return false;
}

template <typename R>
__device__ __forceinline__ void leaf_tri(const DevScene& S, int slot, V3<R>& v0, V3<R>& e1,
                                         V3<R>& e2, int& id);
template <>
__device__ __forceinline__ void leaf_tri<float>(const DevScene& S, int slot, V3<float>& v0,
                                                V3<float>& e1, V3<float>& e2, int& id) {
  float4 a = __ldg(S.leaf_f + 3 * slot), b = __ldg(S.leaf_f + 3 * slot + 1),
         c = __ldg(S.leaf_f + 3 * slot + 2);
  v0 = {a.x, a.y, a.z};
  id = __float_as_int(a.w);
  e1 = {b.x, b.y, b.z};
  e2 = {c.x, c.y, c.z};
}
template <>
__device__ __forceinline__ void leaf_tri<Dn>(const DevScene& S, int slot, V3<Dn>& v0, V3<Dn>& e1,
                                             V3<Dn>& e2, int& id) {
  const double* p = S.leaf_d + 9 * slot;
  id = __ldg(S.leaf_id + slot);
  v0 = {__ldg(p + 0), __ldg(p + 1), __ldg(p + 2)};
  e1 = {__ldg(p + 3), __ldg(p + 4), __ldg(p + 5)};
  e2 = {__ldg(p + 6), __ldg(p + 7), __ldg(p + 8)};
}
template <>
__device__ __forceinline__ void leaf_tri<double>(const DevScene& S, int slot, V3<double>& v0,
                                                 V3<double>& e1, V3<double>& e2, int& id) {
  const double* p = S.leaf_d + 9 * slot;
  id = __ldg(S.leaf_id + slot);
  v0 = {__ldg(p + 0), __ldg(p + 1), __ldg(p + 2)};
  e1 = {__ldg(p + 3), __ldg(p + 4), __ldg(p + 5)};
  e2 = {__ldg(p + 6), __ldg(p + 7), __ldg(p + 8)};
}

// nearest wins; exact ties -> lowest prim id (geometry.py:199-202)
template <typename R>
__device__ __forceinline__ bool improves(R t, int prim, R best_t, int best_prim) {
  return t < best_t || (t == best_t && (best_prim < 0 || prim < best_prim));
}

constexpr int TRAV_STACK = 64;

// traversal counters (nodes visited, primitives tested, casts) for the
// roofline's algorithmic-bytes figure; flushed only when a counting run
// armed g_trav_stats (drcb_trav_stats), one predicated branch per cast.
__device__ unsigned long long* g_trav_stats = nullptr;

__device__ __forceinline__ float f_ru(double x) { return __double2float_ru(x); }
__device__ __forceinline__ float f_ru(float x) { return x; }

constexpr int TRAV_SENTINEL = 0x76543210;

// one primitive test; returns whether it hit inside (tmin, bound)
template <typename R>
__device__ __forceinline__ bool test_prim(const DevScene& S, int slot, V3<R> O, V3<R> D, R tmin,
                                          R bound, R& t, int& id) {
  V3<R> v0, e1, e2;
  leaf_tri<R>(S, slot, v0, e1, e2, id);
  if (id >= S.n_s + S.n_q) return tri_t(v0, e1, e2, O, D, tmin, bound, t);
  if (id >= S.n_s) return quad_t(S, id - S.n_s, O, D, tmin, bound, t);
  return sphere_t(S, id, O, D, tmin, bound, t);
}

// ---------------------------------------------------------------------------
// fp32 build: near-tie refinement. The fp32 triangle test carries a bound on
// its own rounding error (the ray and the triangle rounded to fp32, and the
// fp32 arithmetic of Moller-Trumbore): a candidate whose inside/outside or
// t-range decision lies within that bound, or whose t lies within the bound
// of the current nearest hit, is re-tested in fp64 against the fp64 leaf
// records and the fp64 ray (the reference's arithmetic, geometry.py:271-286,
// with its nearest-t / lowest-id rule, geometry.py:199-214). Every other
// decision is provably the one fp64 makes.
//   Ray64 references: Plain (no refinement: the fp32 decisions as they
//   come — bounce, shadow and map-path casts, whose flip rate the tests
//   report), Promote (the fp32 ray itself in fp64, for later links of a
//   primary chain), Ray64Ptr (fp64 rays in memory: drcb_intersect's mixed
//   mode), CameraRay64 (the pixel's fp64 camera ray, recomputed on demand:
//   the G-buffer's primary casts).
struct Plain {};
struct Promote {
  template <typename R>
  __device__ __forceinline__ void get(V3<R> O, V3<R> D, V3<Dn>& o, V3<Dn>& d) const {
    o = {double(O.x), double(O.y), double(O.z)};
    d = {double(D.x), double(D.y), double(D.z)};
  }
};
struct Ray64Ptr {
  const double* o;
  const double* d;
  template <typename R>
  __device__ __forceinline__ void get(V3<R>, V3<R>, V3<Dn>& oo, V3<Dn>& dd) const {
    oo = ld3<Dn>(o);
    dd = ld3<Dn>(d);
  }
};

// 0 = certain miss, 1 = certain hit (t, error bound mt), 2 = undecided in fp32
__device__ __forceinline__ int tri_t_margin(V3<float> v0, V3<float> e1, V3<float> e2, V3<float> O,
                                            V3<float> D, float tmin, float tmax, float& tout,
                                            float& mt) {
  V3<float> pv = cross(D, e2);
  float det = dot(pv, e1);
  if (!(fabsf(det) > 1e-12f)) return fabsf(det) > 0.f ? 2 : 0;  // fp64 decides |det| vs 1e-14
  // 16 ulps of every operand magnitude that enters a result
  constexpr float EPS = 16.f * 5.9604645e-8f;
  const float inv = 1.f / det, ainv = fabsf(inv);
  V3<float> tv = O - v0;
  auto l1 = [](V3<float> a) { return fabsf(a.x) + fabsf(a.y) + fabsf(a.z); };
  // |O - v0| carries the rounding of both points: bound it by their sizes
  const float T = fmaxf(l1(O), l1(v0)) + l1(tv);
  // |D||e2| bounds pv = D x e2 and its error even when D is nearly parallel to
  // e2 (the rounding of D and e2 perturbs pv by eps |D||e2|, not eps |pv|)
  const float de2 = l1(D) * l1(e2);
  const float pe1 = de2 * l1(e1) * ainv;  // condition of det (>= 1)
  const float u = dot(tv, pv) * inv;
  const float mu = EPS * (T * de2 * ainv + fabsf(u) * pe1 + 1.f);
  if (u < -mu || u > 1.f + mu) return 0;
  const V3<float> qv = cross(tv, e1);
  const float te1 = T * l1(e1);
  const float v = dot(qv, D) * inv;
  const float mv = EPS * (te1 * l1(D) * ainv + fabsf(v) * pe1 + 1.f);
  if (v < -mv || u + v > 1.f + mu + mv) return 0;
  const float t = dot(qv, e2) * inv;
  const float m_t = EPS * (te1 * l1(e2) * ainv + fabsf(t) * pe1);
  if (t <= tmin - m_t || t > tmax + m_t) return 0;
  tout = t;
  mt = m_t;
  const bool sure = u >= mu && u <= 1.f - mu && v >= mv && u + v <= 1.f - mu - mv &&
                    t > tmin + m_t && t <= tmax - m_t;
  return sure ? 1 : 2;
}

// fp32 candidate test: 0 miss, 1 certain hit, 2 undecided (refine in fp64)
__device__ __forceinline__ int test_prim32(const DevScene& S, int slot, V3<float> O, V3<float> D,
                                           float tmin, float bound, float& t, float& mt, int& id) {
  V3<float> v0, e1, e2;
  leaf_tri<float>(S, slot, v0, e1, e2, id);
  if (id >= S.n_s + S.n_q) return tri_t_margin(v0, e1, e2, O, D, tmin, bound, t, mt);
  // spheres / quads: the plain fp32 test with a relative t bound (their
  // near-ties with other primitives still go to fp64)
  bool h = id >= S.n_s ? quad_t(S, id - S.n_s, O, D, tmin, bound, t) : sphere_t(S, id, O, D, tmin, bound, t);
  mt = 1e-5f * fabsf(t) + 1e-6f;
  return h ? 1 : 0;
}

// the fp64 re-test of one leaf slot (uncontracted: the fp64 build's bits)
template <class Ref>
__device__ __noinline__ bool refine64(const DevScene& S, int slot, const Ref& ref, V3<float> O,
                                      V3<float> D, float tmin, float tmax, double& t) {
  V3<Dn> o, d;
  ref.get(O, D, o, d);
  const Dn lo = tmin == float(T_EPS) ? T_EPS : double(tmin);
  const Dn hi = isinf(tmax) ? double(INFINITY) : double(tmax);
  int id;
  Dn tt;
  const bool h = test_prim<Dn>(S, slot, o, d, lo, hi, tt, id);
  t = tt.v;
  return h;
}

// Closest hit (ANY=false) or any hit in (tmin, tmax] (ANY=true) over the BVH.
// Warp-synchronous while-while traversal with speculative leaf postponement
// (Aila & Laine 2009): every lane that entered runs every iteration of ONE
// loop whose phase is warp-uniform. INNER phase: lanes step one node; a lane
// reaching a leaf postpones it and keeps descending speculatively until it
// meets a second leaf. The warp switches to the LEAF phase when no lane is
// still searching for its first leaf, and stays there while any lane has
// primitives left: each iteration tests ONE primitive per lane, so leaf work
// of different lanes is done side by side instead of lane after lane. The
// result is traversal-order independent (nearest t, ties -> lowest prim id).
template <typename R, bool ANY, class Ref = Plain>
__device__ HitRec<R> traverse(const DevScene& S, V3<R> O, V3<R> D, R tmin, R tmax,
                              const Ref& ref = Ref()) {
  constexpr bool F32 = std::is_same<R, float>::value && !std::is_same<Ref, Plain>::value;
  HitRec<R> best{tmax, -1};
  if (S.n_prims == 0) return best;
  const unsigned tmask = __activemask();
  const int entry_lanes = __popc(tmask);
  const float ox = float(O.x), oy = float(O.y), oz = float(O.z);
  auto safe_inv = [](R d) -> float {
    float f = float(d);
    if (fabsf(f) < 1e-30f) f = copysignf(1e-30f, f);
    return 1.0f / f;
  };
  const float ix = safe_inv(D.x), iy = safe_inv(D.y), iz = safe_inv(D.z);
  const float oix = ox * ix, oiy = oy * iy, oiz = oz * iz;
  constexpr float ROB = 1.0f + 4.0f * 5.97e-8f;  // conservative slab (2*gamma(3))
  int stack[TRAV_STACK];
  int sp = 0;
  stack[0] = TRAV_SENTINEL;
  int node = 0;        // >= 0 inner node, < 0 leaf code, SENTINEL = stack empty
  int postponed = 0;   // < 0: a leaf found while searching
  int pcur = 0, pend = 0;  // primitive cursor of the leaf under test
  bool leaf_phase = false;
  unsigned n_nodes = 0, n_prims = 0;
  // fp32 build: the nearest hit's leaf slot and its t error bound (0 once the
  // hit is exact, i.e. came from the fp64 re-test)
  int best_slot = -1;
  float best_mt = 0.f;
  float tbest = isinf(float(tmax)) ? INFINITY : f_ru(tmax) * ROB;
  while (true) {
    const bool inner = node >= 0 && node != TRAV_SENTINEL;
    const bool leafwork = pcur < pend || postponed < 0 || node < 0;
    const bool searching = inner && postponed >= 0 && pcur >= pend;
    const unsigned any_search = __ballot_sync(tmask, searching);
    const unsigned any_leaf = __ballot_sync(tmask, leafwork);
    if (!any_search && !any_leaf) break;
    leaf_phase = any_leaf && (leaf_phase || !any_search);
    if (!leaf_phase) {
      if (inner && pcur >= pend) {
        ++n_nodes;
        const float4* nd = S.nodes + 4 * node;
        float4 a = __ldg(nd), b = __ldg(nd + 1), c = __ldg(nd + 2), d = __ldg(nd + 3);
        // explicit FMAs (this TU builds with -fmad=false for the fp64 parity
        // path; one rounding instead of two stays inside the ROB slack)
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
        // packed pairs (FFMA2: per lane the same correctly rounded fma)
        const float2 tx = __ffma2_rn(make_float2(a.x, a.y), make_float2(ix, ix), make_float2(-oix, -oix));
        const float2 ty = __ffma2_rn(make_float2(a.z, a.w), make_float2(iy, iy), make_float2(-oiy, -oiy));
        const float2 tz = __ffma2_rn(make_float2(c.x, c.y), make_float2(iz, iz), make_float2(-oiz, -oiz));
        const float2 sx = __ffma2_rn(make_float2(b.x, b.y), make_float2(ix, ix), make_float2(-oix, -oix));
        const float2 sy = __ffma2_rn(make_float2(b.z, b.w), make_float2(iy, iy), make_float2(-oiy, -oiy));
        const float2 sz = __ffma2_rn(make_float2(c.z, c.w), make_float2(iz, iz), make_float2(-oiz, -oiz));
        float tx0 = tx.x, tx1 = tx.y, ty0 = ty.x, ty1 = ty.y, tz0 = tz.x, tz1 = tz.y;
        float sx0 = sx.x, sx1 = sx.y, sy0 = sy.x, sy1 = sy.y, sz0 = sz.x, sz1 = sz.y;
#else
        float tx0 = __fmaf_rn(a.x, ix, -oix), tx1 = __fmaf_rn(a.y, ix, -oix);
        float ty0 = __fmaf_rn(a.z, iy, -oiy), ty1 = __fmaf_rn(a.w, iy, -oiy);
        float tz0 = __fmaf_rn(c.x, iz, -oiz), tz1 = __fmaf_rn(c.y, iz, -oiz);
        float sx0 = __fmaf_rn(b.x, ix, -oix), sx1 = __fmaf_rn(b.y, ix, -oix);
        float sy0 = __fmaf_rn(b.z, iy, -oiy), sy1 = __fmaf_rn(b.w, iy, -oiy);
        float sz0 = __fmaf_rn(c.z, iz, -oiz), sz1 = __fmaf_rn(c.w, iz, -oiz);
#endif
        float n0 = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
        float f0 = fminf(fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fmaxf(tz0, tz1)) * ROB, tbest);
        float n1 = fmaxf(fmaxf(fminf(sx0, sx1), fminf(sy0, sy1)), fmaxf(fminf(sz0, sz1), 0.0f));
        float f1 = fminf(fminf(fminf(fmaxf(sx0, sx1), fmaxf(sy0, sy1)), fmaxf(sz0, sz1)) * ROB, tbest);
        bool h0 = n0 <= f0, h1 = n1 <= f1;
        int c0 = __float_as_int(d.x), c1 = __float_as_int(d.y);
        if (!h0 && !h1) {
          node = stack[sp--];
        } else {
          node = h0 ? c0 : c1;
          if (h0 && h1) {
            int other = c1;
            if (n1 < n0) {
              node = c1;
              other = c0;
            }
            if (sp + 1 < TRAV_STACK) stack[++sp] = other;
          }
        }
        if (node < 0 && postponed >= 0) {  // first leaf: postpone, keep descending
          postponed = node;
          node = stack[sp--];
        }
      }
    } else if (leafwork) {
      if (pcur >= pend) {  // next leaf: the postponed one, then the current node
        int code;
        if (postponed < 0) {
          code = ~postponed;
          postponed = 0;
        } else {
          code = ~node;
          node = stack[sp--];
        }
        pcur = code >> 3;
        pend = pcur + (code & 7) + 1;
        n_prims += pend - pcur;
      }
      R t;
      int id;
      if constexpr (F32) {
        static_assert(std::is_same<R, float>::value, "refinement is the fp32 build's");
        float mt;
        const int res = test_prim32(S, pcur, O, D, tmin, ANY ? tmax : best.t + best_mt, t, mt, id);
        if (ANY) {
          double t64;
          if (res == 1 || (res == 2 && refine64(S, pcur, ref, O, D, tmin, tmax, t64))) {
            best.t = t;
            best.prim = id;
            node = TRAV_SENTINEL;
            postponed = 0;
            pend = pcur;
          }
        } else if (res) {
          const bool near = best.prim >= 0 && fabsf(t - best.t) <= mt + best_mt;
          if (res == 1 && !near) {
            if (t < best.t) {
              best.t = t;
              best.prim = id;
              best_slot = pcur;
              best_mt = mt;
              tbest = f_ru(t + mt) * ROB;
            }
          } else {
            // undecided candidate or a near-tie with the current nearest hit:
            // both in fp64, the reference's comparison (nearest, then lowest id)
            double tc, tb = 0.0;
            if (refine64(S, pcur, ref, O, D, tmin, tmax, tc)) {
              bool take = best.prim < 0;
              if (!take) {
                const bool bhit = refine64(S, best_slot, ref, O, D, tmin, tmax, tb);
                take = !bhit || tc < tb || (tc == tb && id < best.prim);
              }
              if (take) {
                const float tf = float(tc);
                best.t = tf;
                best.prim = id;
                best_slot = pcur;
                best_mt = fabsf(tf) * 1.2e-7f;  // exact up to its fp32 rounding
                tbest = f_ru(tc) * ROB;
              }
            }
          }
        }
      } else {
        if (test_prim<R>(S, pcur, O, D, tmin, ANY ? tmax : best.t, t, id)) {
          if (ANY) {
            best.t = t;
            best.prim = id;
            node = TRAV_SENTINEL;
            postponed = 0;
            pend = pcur;
          } else if (improves(t, id, best.t, best.prim)) {
            best.t = t;
            best.prim = id;
            tbest = f_ru(t) * ROB;
          }
        }
      }
      ++pcur;
    }
  }
  (void)best_slot;
  (void)best_mt;
  if (g_trav_stats) {
    atomicAdd(g_trav_stats + 0, n_nodes);
    atomicAdd(g_trav_stats + 1, n_prims);
    atomicAdd(g_trav_stats + 2, 1ull);
    atomicMax(g_trav_stats + 3, (unsigned long long)n_nodes);
    atomicMax(g_trav_stats + 4, (unsigned long long)n_prims);
    // histogram of prims tested: [0,8) [8,32) [32,128) [128,512) [512,inf)
    int b = n_prims < 8 ? 0 : n_prims < 32 ? 1 : n_prims < 128 ? 2 : n_prims < 512 ? 3 : 4;
    atomicAdd(g_trav_stats + 5 + b, 1ull);
    atomicAdd(g_trav_stats + 10, (unsigned long long)entry_lanes);
    if (ANY) atomicAdd(g_trav_stats + 11, 1ull);
  }
  return best;
}

template <typename R>
struct SurfHit {
  bool hit;
  R t;
  int prim, mat;
  V3<R> pos, normal;  // geometric, unflipped (geometry.py:296-322)
};

template <typename R, class Ref = Plain>
__device__ __forceinline__ SurfHit<R> intersect(const DevScene& S, V3<R> O, V3<R> D,
                                                R tmin = R(T_EPS), R tmax = R(INFINITY),
                                                const Ref& ref = Ref()) {
  HitRec<R> h = traverse<R, false, Ref>(S, O, D, tmin, tmax, ref);
  SurfHit<R> r;
  r.hit = h.prim >= 0;
  r.prim = h.prim;
  r.t = r.hit ? h.t : R(INFINITY);
  r.mat = -1;
  r.normal = {R(0), R(0), R(0)};
  r.pos = O + (r.hit ? h.t : R(0)) * D;
  if (r.hit) {
    int p = h.prim;
    if (p < S.n_s) {
      const double* s = S.sph + 5 * p;
      R rad = R(s[3]);
      V3<R> d = r.pos - ld3<R>(s);
      r.normal = {d.x / rad, d.y / rad, d.z / rad};
      r.mat = S.sph_mat[p];
    } else if (p < S.n_s + S.n_q) {
      int i = p - S.n_s;
      r.normal = ld3<R>(S.quad + 18 * i + 9);
      r.mat = S.quad_mat[i];
    } else {
      int i = p - S.n_s - S.n_q;
      r.normal = ld3<R>(S.tri + 13 * i + 9);
      r.mat = S.tri_mat[i];
    }
  }
  return r;
}

template <typename R>
__device__ __forceinline__ bool occluded(const DevScene& S, V3<R> O, V3<R> D, R tmax) {
  return traverse<R, true>(S, O, D, R(T_EPS), tmax).prim >= 0;
}

// ---------------------------------------------------------------------------
// frames (drc/bsdf.py:78-96 batch; 63-75 scalar build_frame)
template <typename R>
struct Frame {
  V3<R> t, b, n;
  __device__ __forceinline__ V3<R> to_local(V3<R> v) const {
    return {dot(v, t), dot(v, b), dot(v, n)};
  }
  __device__ __forceinline__ V3<R> to_world(V3<R> l) const {
    return (l.x * t + l.y * b) + l.z * n;
  }
};

template <typename R>
__device__ __forceinline__ Frame<R> frame_batch(const DevScene& S, V3<R> n) {
  V3<R> up = ld3<R>(S.up);
  V3<R> ref = up;
  if (fabs(dot(n, up)) > R(UP_DEGENERACY)) ref = ld3<R>(S.rot_up);
  V3<R> t = cross(ref, n);
  R nr = norm(t);
  if (nr < R(1e-9)) {
    t = cross(mk<R>(R(1), R(0), R(0)), n);
    nr = norm(t);
  }
  t = divs(t, nr);
  return Frame<R>{t, cross(n, t), n};
}

// scalar build_frame: the fallback re-derives the reference up from the X axis
// (bsdf.py:52-75); used for cache-point frames (hemimap.py:238)
template <typename R>
__device__ __forceinline__ V3<R> rotated_up_of(V3<R> up) {
  V3<R> axes[2] = {mk<R>(R(0), R(1), R(0)), mk<R>(R(1), R(0), R(0))};
  for (int k = 0; k < 2; ++k) {
    V3<R> w = axes[k] - dot(axes[k], up) * up;
    R nw = norm(w);
    if (nw > R(1e-6)) return divs(w, nw);
  }
  return mk<R>(R(0), R(0), R(1));
}

template <typename R>
__device__ __forceinline__ Frame<R> frame_scalar(const DevScene& S, V3<R> n) {
  V3<R> up = ld3<R>(S.up);
  V3<R> ref = (fabs(dot(n, up)) <= R(UP_DEGENERACY)) ? up : ld3<R>(S.rot_up);
  V3<R> t = cross(ref, n);
  R nr = norm(t);
  if (nr < R(1e-9)) {
    V3<R> xa = mk<R>(R(1), R(0), R(0));
    ref = (fabs(dot(n, xa)) <= R(UP_DEGENERACY)) ? xa : rotated_up_of(xa);
    t = cross(ref, n);
    nr = norm(t);
  }
  t = divs(t, nr);
  return Frame<R>{t, cross(n, t), n};
}

// ---------------------------------------------------------------------------
// BSDFs (drc/bsdf.py:223-327)
template <typename R>
__device__ __forceinline__ R schlick1(R f0, R c) {
  c = fmin(fmax(c, R(0)), R(1));
  return f0 + (R(1) - f0) * pow(R(1) - c, R(5));
}

template <typename R>
__device__ __forceinline__ R power_heuristic(R a, R b) {
  R a2 = a * a;
  return a2 / (a2 + b * b);
}

// eval_batch (bsdf.py:234-254): f and sampling pdf for one row
template <typename R>
__device__ __forceinline__ void bsdf_eval(const DevScene& S, int mat, V3<R> lo, V3<R> li,
                                          V3<R>& f, R& pdf) {
  int kind = S.mat_kind[mat];
  V3<R> alb = ld3<R>(S.mat_albedo + 3 * mat);
  bool above = lo.z > R(0) && li.z > R(0);
  f = {R(0), R(0), R(0)};
  pdf = R(0);
  const R inv_pi = R(1) / R(PI);
  if (kind == 0) {
    if (above) f = {alb.x / R(PI), alb.y / R(PI), alb.z / R(PI)};
    pdf = fmax(li.z, R(0)) / R(PI);
    (void)inv_pi;
  } else if (kind == 1) {
    R e = R(S.mat_exp[mat]);
    R cos_a = fmax((-lo.x * li.x - lo.y * li.y) + lo.z * li.z, R(0));
    R lobe = pow(cos_a, e);
    R s = (e + R(2)) / (R(2) * R(PI)) * lobe;
    if (above) f = {alb.x * s, alb.y * s, alb.z * s};
    pdf = (e + R(1)) / (R(2) * R(PI)) * lobe;
  }
}

// _frames_around (bsdf.py:322-327)
template <typename R>
__device__ __forceinline__ void frames_around(V3<R> axis, V3<R>& t, V3<R>& b) {
  V3<R> a = (fabs(axis.x) > R(0.9)) ? mk<R>(R(0), R(1), R(0)) : mk<R>(R(1), R(0), R(0));
  t = cross(a, axis);
  R nr = fmax(norm(t), R(1e-12));
  t = divs(t, nr);
  b = cross(axis, t);
}

template <typename R>
struct BsdfSample {
  V3<R> li, value;
  R pdf;
  bool spec;
};

// sample_batch (bsdf.py:257-319)
template <typename R>
__device__ __forceinline__ BsdfSample<R> bsdf_sample(const DevScene& S, int mat, V3<R> lo, R u1,
                                                     R u2, bool entering) {
  BsdfSample<R> s;
  int kind = S.mat_kind[mat];
  V3<R> alb = ld3<R>(S.mat_albedo + 3 * mat);
  s.pdf = R(1);
  s.value = {R(0), R(0), R(0)};
  s.spec = (kind == 2 || kind == 3);
  if (kind == 0) {
    R r = sqrt(u1);
    R phi = R(2.0 * PI) * u2;
    R z = sqrt(fmax(R(1) - u1, R(0)));
    s.li = {r * cos(phi), r * sin(phi), z};
    s.pdf = fmax(z / R(PI), R(1e-12));
    if (lo.z > R(0)) s.value = {alb.x / R(PI), alb.y / R(PI), alb.z / R(PI)};
  } else if (kind == 1) {
    R e = R(S.mat_exp[mat]);
    R cos_a = pow(u1, R(1) / (e + R(1)));
    R sin_a = sqrt(fmax(R(1) - cos_a * cos_a, R(0)));
    R phi = R(2.0 * PI) * u2;
    V3<R> lobe = {sin_a * cos(phi), sin_a * sin(phi), cos_a};
    V3<R> r = {-lo.x, -lo.y, lo.z};
    V3<R> ft, fb;
    frames_around(r, ft, fb);
    V3<R> wig = (lobe.x * ft + lobe.y * fb) + lobe.z * r;
    s.li = wig;
    R lobe_d = pow(cos_a, e);
    s.pdf = fmax((e + R(1)) / (R(2) * R(PI)) * lobe_d, R(1e-12));
    if (wig.z > R(0) && lo.z > R(0)) {
      R k = (e + R(2)) / (R(2) * R(PI)) * lobe_d;
      s.value = {alb.x * k, alb.y * k, alb.z * k};
    }
  } else if (kind == 2) {
    s.li = {-lo.x, -lo.y, lo.z};
    s.value = {schlick1(alb.x, lo.z), schlick1(alb.y, lo.z), schlick1(alb.z, lo.z)};
  } else {
    R ior = R(S.mat_ior[mat]);
    R eta = entering ? R(1) / ior : ior;
    R cos_i = lo.z;
    R sin2_t = eta * eta * fmax(R(1) - cos_i * cos_i, R(0));
    R q = (ior - R(1)) / (ior + R(1));
    R f0 = q * q;
    R fr = schlick1(f0, cos_i);
    bool refl = (sin2_t >= R(1)) || (u1 < fr);
    R cos_t = sqrt(fmax(R(1) - sin2_t, R(0)));
    s.li = refl ? mk<R>(-lo.x, -lo.y, cos_i) : mk<R>(-eta * lo.x, -eta * lo.y, -cos_t);
    s.value = alb;
  }
  return s;
}

// ---------------------------------------------------------------------------
// next-event estimation (drc/integrators.py:86-169)
template <typename R>
struct LightSample {
  V3<R> wl, ratio;
  R dist, pdf_sa;
  bool is_delta, valid;
};

template <typename R>
__device__ __forceinline__ LightSample<R> sample_lights(const DevScene& S, V3<R> pos, R u_sel,
                                                        R ua, R ub) {
  LightSample<R> L;
  int nl = S.n_lights;
  long long pk = (long long)(u_sel * R(nl));
  int pick = int(pk < nl - 1 ? pk : nl - 1);
  L.is_delta = pick < S.n_point;
  L.wl = {R(0), R(0), R(0)};
  L.ratio = {R(0), R(0), R(0)};
  L.dist = R(INFINITY);
  L.pdf_sa = R(INFINITY);
  if (L.is_delta) {
    V3<R> vec = ld3<R>(S.point_pos + 3 * pick) - pos;
    R d2 = dot(vec, vec);
    R d = sqrt(d2);
    L.wl = divs(vec, d);
    L.dist = d;
    R k = R(nl) / d2;
    V3<R> I = ld3<R>(S.point_int + 3 * pick);
    L.ratio = {I.x * k, I.y * k, I.z * k};
    L.valid = d > R(4 * T_EPS);
    return L;
  }
  int k = pick - S.n_point;
  int prim = S.area_prim[k];
  R area = R(S.area_area[k]);
  V3<R> le = ld3<R>(S.mat_emis + 3 * S.area_mat[k]);
  V3<R> y, nl3;
  if (prim < S.n_s) {
    const double* s = S.sph + 5 * prim;
    R z = R(1) - R(2) * ua;
    R r = sqrt(fmax(R(1) - z * z, R(0)));
    R phi = R(2.0 * PI) * ub;
    V3<R> dsph = {r * cos(phi), r * sin(phi), z};
    y = ld3<R>(s) + R(s[3]) * dsph;
    nl3 = dsph;
  } else if (prim < S.n_s + S.n_q) {
    const double* q = S.quad + 18 * (prim - S.n_s);
    y = (ld3<R>(q) + ua * ld3<R>(q + 3)) + ub * ld3<R>(q + 6);
    nl3 = ld3<R>(q + 9);
  } else {
    const double* t = S.tri + 13 * (prim - S.n_s - S.n_q);
    R su = sqrt(ua);
    R b1 = R(1) - su;
    R b2 = ub * su;
    y = (ld3<R>(t) + b1 * ld3<R>(t + 3)) + b2 * ld3<R>(t + 6);
    nl3 = ld3<R>(t + 9);
  }
  V3<R> vec = y - pos;
  R d2 = fmax(dot(vec, vec), R(1e-24));
  R d = sqrt(d2);
  V3<R> w = divs(vec, d);
  R cos_l = -dot(nl3, w);
  bool ok = (cos_l > R(1e-9)) && (d > R(4 * T_EPS));
  R pdf = ok ? d2 / fmax(cos_l, R(1e-12)) / area / R(nl) : R(INFINITY);
  L.wl = w;
  L.dist = d;
  if (ok) L.ratio = {le.x / pdf, le.y / pdf, le.z / pdf};
  L.pdf_sa = pdf;
  L.valid = ok;
  return L;
}

// _nee_pdf_for_hit (integrators.py:164-169)
template <typename R>
__device__ __forceinline__ R nee_pdf_for_hit(const DevScene& S, int prim, R t, R cos_l) {
  int li = S.prim_light[prim];
  if (li < 0) return R(0);
  R area = R(S.area_area[li]);
  int nl = S.n_lights > 1 ? S.n_lights : 1;
  return t * t / fmax(cos_l, R(1e-12)) / area / R(nl);
}

template <typename R>
__device__ __forceinline__ R sample_dim(const PathRng& rng, uint64_t dim) {
  return to_unit<R>(rng.sample(dim));
}

// NEE at a non-specular vertex (integrators.py:242-269 / 364-396); returns
// the unoccluded contribution (before beta) or zero.
template <typename R>
__device__ __forceinline__ V3<R> nee(const DevScene& S, const PathRng& rng, uint64_t base,
                                     V3<R> pos, V3<R> n_front, const Frame<R>& fr, int mat,
                                     V3<R> wo_local) {
  V3<R> zero = {R(0), R(0), R(0)};
  R u_sel = sample_dim<R>(rng, base + 0);
  R ua = sample_dim<R>(rng, base + 1);
  R ub = sample_dim<R>(rng, base + 2);
  LightSample<R> ls = sample_lights(S, pos, u_sel, ua, ub);
  V3<R> wl_local = fr.to_local(ls.wl);
  R cos_s = wl_local.z;
  if (!(ls.valid && cos_s > R(0))) return zero;
  V3<R> f;
  R pdf_b;
  bsdf_eval(S, mat, wo_local, wl_local, f, pdf_b);
  V3<R> contrib = f * mk<R>(ls.ratio.x * cos_s, ls.ratio.y * cos_s, ls.ratio.z * cos_s);
  R w = ls.is_delta ? R(1) : power_heuristic(ls.pdf_sa, pdf_b);
  contrib = contrib * mk<R>(w, w, w);
  if (!any_pos(contrib)) return zero;
  V3<R> so = pos + R(T_EPS) * n_front;
  if (occluded(S, so, ls.wl, ls.dist - R(2 * T_EPS))) return zero;
  return contrib;
}

// ---------------------------------------------------------------------------
// trace_radiance_batch for one path (integrators.py:175-302). `first` is the
// segment-0 intersection when the caller already cast it (map rays).
template <typename R>
__device__ V3<R> trace_path(const DevScene& S, V3<R> O, V3<R> D, const PathRng& rng,
                            int max_depth, bool skip_first_emission, int rr_start,
                            const SurfHit<R>* first, int& nonfinite) {
  V3<R> L = {R(0), R(0), R(0)};
  V3<R> beta = {R(1), R(1), R(1)};
  R prev_pdf = R(0);
  bool prev_delta = true;
  V3<R> env = ld3<R>(S.env);
  for (int seg = 0; seg <= max_depth; ++seg) {
    SurfHit<R> h = (seg == 0 && first) ? *first : intersect(S, O, D);
    bool skip = (seg == 0 && skip_first_emission);
    if (!h.hit) {
      if (S.has_env && !skip) L = L + beta * env;
      break;
    }
    int mat = h.mat;
    bool facing = dot(h.normal, D) < R(0);
    if (S.mat_emitter[mat] && facing && !skip) {
      R w = R(1);
      if (seg > 0 && !prev_delta) {
        R cos_l = -dot(h.normal, D);
        R pdf_nee = nee_pdf_for_hit(S, h.prim, h.t, cos_l);
        w = power_heuristic(prev_pdf, pdf_nee);
      }
      V3<R> e = ld3<R>(S.mat_emis + 3 * mat);
      L = L + (beta * e) * mk<R>(w, w, w);
    }
    if (seg == max_depth) break;
    bool entering = facing;
    V3<R> n_front = entering ? h.normal : -h.normal;
    Frame<R> fr = frame_batch(S, n_front);
    V3<R> wo_local = fr.to_local(-D);
    uint64_t base = 2 + 8 * (uint64_t)seg;
    bool spec = S.mat_spec[mat];
    if (S.n_lights > 0 && !spec) {
      V3<R> c = nee(S, rng, base, h.pos, n_front, fr, mat, wo_local);
      L = L + beta * c;
    }
    R u1 = sample_dim<R>(rng, base + 3), u2 = sample_dim<R>(rng, base + 4);
    BsdfSample<R> bs = bsdf_sample(S, mat, wo_local, u1, u2, entering);
    R cos_i = fabs(bs.li.z);
    V3<R> weight = bs.spec ? bs.value : bs.value * mk<R>(cos_i / bs.pdf, cos_i / bs.pdf, cos_i / bs.pdf);
    beta = beta * weight;
    V3<R> wi = fr.to_world(bs.li);
    R side = bs.li.z >= R(0) ? R(1) : R(-1);
    O = h.pos + (R(T_EPS) * side) * n_front;
    D = wi;
    prev_pdf = bs.pdf;
    prev_delta = bs.spec;
    bool alive = any_pos(beta) && all_finite(beta);
    if (seg + 1 >= rr_start) {
      R q = fmin(fmax(maxc(beta), R(RR_FLOOR)), R(1));
      R u_rr = sample_dim<R>(rng, base + 5);
      bool survive = u_rr < q;
      beta = divs(beta, q);
      alive = alive && survive;
    }
    if (!alive) break;
  }
  if (!all_finite(L)) {
    L = {R(0), R(0), R(0)};
    ++nonfinite;
  }
  return L;
}

// li_direct_batch for one path (integrators.py:305-424)
template <typename R>
__device__ V3<R> direct_path(const DevScene& S, V3<R> O, V3<R> D, const PathRng& rng,
                             bool include_background, int& nonfinite) {
  V3<R> L = {R(0), R(0), R(0)};
  V3<R> beta = {R(1), R(1), R(1)};
  bool phase1 = false, mis_live = false;
  R mis_pdf = R(0);
  V3<R> env = ld3<R>(S.env);
  for (int seg = 0; seg < SPECULAR_CHAIN_BOUND; ++seg) {
    SurfHit<R> h = intersect(S, O, D);
    if (!h.hit) {
      if (S.has_env && (phase1 || include_background)) L = L + beta * env;
      break;
    }
    int mat = h.mat;
    bool facing = dot(h.normal, D) < R(0);
    if (S.mat_emitter[mat] && facing) {
      R w = R(1);
      if (mis_live) {
        R cos_l = -dot(h.normal, D);
        R pdf_nee = nee_pdf_for_hit(S, h.prim, h.t, cos_l);
        w = power_heuristic(mis_pdf, pdf_nee);
      }
      V3<R> e = ld3<R>(S.mat_emis + 3 * mat);
      L = L + (beta * e) * mk<R>(w, w, w);
    }
    bool spec = S.mat_spec[mat];
    if (!(spec || !phase1)) break;
    bool entering = facing;
    V3<R> n_front = entering ? h.normal : -h.normal;
    Frame<R> fr = frame_batch(S, n_front);
    V3<R> wo_local = fr.to_local(-D);
    uint64_t base = 2 + 8 * (uint64_t)seg;
    bool shade = !spec && !phase1;
    if (shade && S.n_lights > 0) {
      V3<R> c = nee(S, rng, base, h.pos, n_front, fr, mat, wo_local);
      L = L + beta * c;
    }
    R u1 = sample_dim<R>(rng, base + 3), u2 = sample_dim<R>(rng, base + 4);
    BsdfSample<R> bs = bsdf_sample(S, mat, wo_local, u1, u2, entering);
    R cos_i = fabs(bs.li.z);
    V3<R> weight = bs.spec ? bs.value : bs.value * mk<R>(cos_i / bs.pdf, cos_i / bs.pdf, cos_i / bs.pdf);
    beta = beta * weight;
    R side = bs.li.z >= R(0) ? R(1) : R(-1);
    O = h.pos + (R(T_EPS) * side) * n_front;
    D = fr.to_world(bs.li);
    mis_live = shade && !bs.spec;
    mis_pdf = mis_live ? bs.pdf : R(0);
    phase1 = phase1 || shade;
    bool alive = (beta.x > R(SPECULAR_THROUGHPUT_CUTOFF) || beta.y > R(SPECULAR_THROUGHPUT_CUTOFF) ||
                  beta.z > R(SPECULAR_THROUGHPUT_CUTOFF)) && all_finite(beta);
    if (!alive) break;
  }
  if (!all_finite(L)) {
    L = {R(0), R(0), R(0)};
    ++nonfinite;
  }
  return L;
}

// primary_chain_batch for one ray (integrators.py:427-518)
template <typename R>
struct ChainOut {
  bool found, escaped;
  V3<R> pos, normal, thr, dir;
  int mat;
  R t_total;
};

// the fp64 twin of the chain's FIRST cast only (later links are fp32-born)
template <class Ref0>
struct FirstCast {
  Ref0 r0;
  bool first;
  template <typename R>
  __device__ __forceinline__ void get(V3<R> O, V3<R> D, V3<Dn>& o, V3<Dn>& d) const {
    if (first)
      r0.get(O, D, o, d);
    else
      Promote().get(O, D, o, d);
  }
};

template <typename R, class Ref0 = Plain>
__device__ ChainOut<R> primary_chain(const DevScene& S, V3<R> O, V3<R> D, const Ref0& ref0 = Ref0()) {
  ChainOut<R> out;
  out.found = out.escaped = false;
  out.pos = out.normal = {R(0), R(0), R(0)};
  out.thr = {R(1), R(1), R(1)};
  out.dir = D;
  out.mat = -1;
  out.t_total = R(0);
  V3<R> beta = {R(1), R(1), R(1)};
  using RefT = typename std::conditional<std::is_same<Ref0, Plain>::value, Plain, FirstCast<Ref0>>::type;
  RefT ref;
  if constexpr (!std::is_same<Ref0, Plain>::value) ref = RefT{ref0, true};
  for (int it = 0; it < SPECULAR_CHAIN_BOUND; ++it) {
    SurfHit<R> h = intersect(S, O, D, R(T_EPS), R(INFINITY), ref);
    if constexpr (!std::is_same<Ref0, Plain>::value) ref.first = false;
    if (!h.hit) {
      out.escaped = true;
      out.thr = beta;
      out.dir = D;
      break;
    }
    out.t_total = out.t_total + h.t;
    int mat = h.mat;
    bool entering = dot(h.normal, D) < R(0);
    if (!S.mat_spec[mat]) {
      out.found = true;
      out.pos = h.pos;
      out.normal = entering ? h.normal : -h.normal;
      out.mat = mat;
      out.thr = beta;
      out.dir = D;
      break;
    }
    V3<R> n_front = entering ? h.normal : -h.normal;
    R cos_i = -dot(n_front, D);
    int kind = S.mat_kind[mat];
    V3<R> alb = ld3<R>(S.mat_albedo + 3 * mat);
    V3<R> refl = D + (R(2) * cos_i) * n_front;
    V3<R> nd = refl;
    V3<R> factor;
    if (kind == 2) {
      factor = {schlick1(alb.x, cos_i), schlick1(alb.y, cos_i), schlick1(alb.z, cos_i)};
    } else {
      R ior = R(S.mat_ior[mat]);
      R eta = entering ? R(1) / ior : ior;
      R ci = cos_i;
      R sin2_t = eta * eta * fmax(R(1) - ci * ci, R(0));
      bool tir = sin2_t >= R(1);
      R q = (ior - R(1)) / (ior + R(1));
      R fr = schlick1(q * q, ci);
      R cos_t = sqrt(fmax(R(1) - sin2_t, R(0)));
      V3<R> refr = eta * D + (eta * ci - cos_t) * n_front;
      nd = tir ? refl : refr;
      R k = tir ? R(1) : R(1) - fr;
      factor = {alb.x * k, alb.y * k, alb.z * k};
    }
    beta = beta * factor;
    R to_side = dot(nd, n_front) >= R(0) ? R(1) : R(-1);
    O = h.pos + (R(T_EPS) * to_side) * n_front;
    D = divs(nd, norm(nd));
    if (beta.x < R(SPECULAR_THROUGHPUT_CUTOFF) && beta.y < R(SPECULAR_THROUGHPUT_CUTOFF) &&
        beta.z < R(SPECULAR_THROUGHPUT_CUTOFF))
      break;
  }
  return out;
}

// Camera.ray_directions for one image-plane point (scene.py:76-93)
template <typename R>
__device__ __forceinline__ V3<R> camera_dir(const DevCamera& C, R px, R py) {
  R w = R(C.W), hh = R(C.H);
  R th = R(C.tan_half);
  R aspect = R(C.aspect);
  R ndc_x = (px / w * R(2) - R(1)) * th * aspect;
  R ndc_y = (R(1) - py / hh * R(2)) * th;
  V3<R> d = (ld3<R>(C.fwd) + ndc_x * ld3<R>(C.right)) + ndc_y * ld3<R>(C.up);
  return divs(d, norm(d));
}

// texel_to_direction local part (hemimap.py:74-84)
template <typename R>
__device__ __forceinline__ V3<R> texel_local(int u, int v) {
  R phi = R(2.0 * PI) * (R(u) + R(0.5)) / R(MAP_RES);
  R theta = R(PI / 2.0) * (R(v) + R(0.5)) / R(MAP_RES);
  R st = sin(theta);
  return {st * cos(phi), st * sin(phi), cos(theta)};
}

}  // namespace drcb
