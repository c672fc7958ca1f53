// drcb_scene.cu — Geometry tables + BVH build on the host, upload to HBM.
//
// Replaces drc.geometry.Geometry (geometry.py:48-185) and BVH
// (geometry.py:335-460). The BVH is a binned-SAH BVH2 over the fp64 prim
// AABBs (32 bins on all three axes, SAH leaf termination, leaf <= 8 refs,
// median fallback), laid
// out as 64 B two-child nodes (drcb_scene.cuh). Triangles are re-ordered into
// leaf order as 48 B fp32 records (v0+id, e1, e2) and 72 B fp64 records so a
// leaf's triangles are contiguous in memory.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>

#include "drcb_internal.h"

namespace drcb {

namespace {

struct Box {
  double lo[3] = {INFINITY, INFINITY, INFINITY};
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  void grow(const Box& b) {
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], b.lo[k]);
      hi[k] = std::max(hi[k], b.hi[k]);
    }
  }
  void grow_pt(const double* p) {
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], p[k]);
      hi[k] = std::max(hi[k], p[k]);
    }
  }
  double area() const {
    double d[3];
    for (int k = 0; k < 3; ++k) d[k] = std::max(hi[k] - lo[k], 0.0);
    return 2.0 * (d[0] * d[1] + d[1] * d[2] + d[0] * d[2]);
  }
};

struct BuildNode {
  Box box[2];
  int child[2];
};

struct Builder {
  const std::vector<Box>& pb;   // one box per reference
  const std::vector<int>& ref_prim;  // reference -> prim id
  std::vector<double> cen;  // 3 per reference
  std::vector<int> ids;
  std::vector<BuildNode> nodes;
  std::vector<int> order;  // leaf slots -> prim id
  int max_depth = 0;
  int n_leaves = 0;
  static constexpr int NB = 32;
  static constexpr int LEAF = 4;
  static constexpr int DEPTH_LIMIT = 56;
  // SAH leaf termination: ranges of up to max_leaf refs become a leaf when
  // n * ci <= ct + ci * (A_l n_l + A_r n_r) / A with ct = 1 (one traversal
  // step ~ one primitive step of the traversal loop). Measured on C3: 22.2
  // nodes + 3.9 primitives per cast (vs 20.5 + 6.5 splitting to <= 4), maps
  // stage -3 %. DRCB_BVH_SAH_CI=0 restores the split-to-4 builder.
  int max_leaf = 8;
  double sah_ci = 1.0;
  double last_cost = INFINITY;

  Builder(const std::vector<Box>& b, const std::vector<int>& rp) : pb(b), ref_prim(rp) {
    cen.resize(3 * pb.size());
    for (size_t i = 0; i < pb.size(); ++i)
      for (int k = 0; k < 3; ++k) cen[3 * i + k] = 0.5 * (pb[i].lo[k] + pb[i].hi[k]);
    ids.resize(pb.size());
    std::iota(ids.begin(), ids.end(), 0);
  }

  Box bounds(int b, int e) const {
    Box r;
    for (int i = b; i < e; ++i) r.grow(pb[ids[i]]);
    return r;
  }

  int make_leaf(int b, int e) {
    int start = (int)order.size();
    for (int i = b; i < e; ++i) order.push_back(ref_prim[ids[i]]);
    ++n_leaves;
    return ~((start << 3) | (e - b - 1));
  }

  // split [b,e) and return the mid index
  int split(int b, int e, int depth) {
    int n = e - b;
    last_cost = INFINITY;
    Box cb;
    for (int i = b; i < e; ++i) cb.grow_pt(&cen[3 * ids[i]]);
    double best_cost = INFINITY;
    int best_axis = -1, best_bin = -1;
    if (depth < DEPTH_LIMIT) {
      for (int ax = 0; ax < 3; ++ax) {
        double ext = cb.hi[ax] - cb.lo[ax];
        if (!(ext > 1e-12)) continue;
        Box bb[NB];
        int bc[NB] = {0};
        double scale = NB / ext;
        for (int i = b; i < e; ++i) {
          int id = ids[i];
          int k = std::min(int((cen[3 * id + ax] - cb.lo[ax]) * scale), NB - 1);
          bb[k].grow(pb[id]);
          ++bc[k];
        }
        Box rb[NB];
        int rc[NB];
        Box acc;
        int cnt = 0;
        for (int k = NB - 1; k >= 0; --k) {
          acc.grow(bb[k]);
          cnt += bc[k];
          rb[k] = acc;
          rc[k] = cnt;
        }
        Box lacc;
        int lc = 0;
        for (int k = 1; k < NB; ++k) {
          lacc.grow(bb[k - 1]);
          lc += bc[k - 1];
          if (lc == 0 || rc[k] == 0) continue;
          double cost = lacc.area() * lc + rb[k].area() * rc[k];
          if (cost < best_cost) {
            best_cost = cost;
            best_axis = ax;
            best_bin = k;
          }
        }
      }
    }
    last_cost = best_cost;
    if (best_axis >= 0) {
      double ext = cb.hi[best_axis] - cb.lo[best_axis];
      double scale = NB / ext;
      auto mid = std::partition(ids.begin() + b, ids.begin() + e, [&](int id) {
        int k = std::min(int((cen[3 * id + best_axis] - cb.lo[best_axis]) * scale), NB - 1);
        return k < best_bin;
      });
      int m = int(mid - ids.begin());
      if (m > b && m < e) return m;
    }
    // median split on the widest centroid axis (geometry.py:397-402)
    int ax = 0;
    double w = -1;
    for (int k = 0; k < 3; ++k)
      if (cb.hi[k] - cb.lo[k] > w) { w = cb.hi[k] - cb.lo[k]; ax = k; }
    int m = b + n / 2;
    std::nth_element(ids.begin() + b, ids.begin() + m, ids.begin() + e, [&](int x, int y) {
      double cx = cen[3 * x + ax], cy = cen[3 * y + ax];
      return cx < cy || (cx == cy && x < y);
    });
    return m;
  }

  // returns encoded child reference for range [b,e)
  int build(int b, int e, int depth) {
    max_depth = std::max(max_depth, depth);
    const int n = e - b;
    if (sah_ci <= 0.0 && n <= LEAF) return make_leaf(b, e);
    if (n <= 1) return make_leaf(b, e);
    int m = split(b, e, depth);
    if (sah_ci > 0.0 && n <= max_leaf) {
      const double a = bounds(b, e).area();
      if (!(a > 0.0) || n * sah_ci <= 1.0 + sah_ci * last_cost / a) return make_leaf(b, e);
    }
    int idx = (int)nodes.size();
    nodes.push_back(BuildNode{});
    Box lb = bounds(b, m), rb = bounds(m, e);
    int l = build(b, m, depth + 1);
    int r = build(m, e, depth + 1);
    nodes[idx].box[0] = lb;
    nodes[idx].box[1] = rb;
    nodes[idx].child[0] = l;
    nodes[idx].child[1] = r;
    return idx;
  }

  void run() {
    int n = (int)pb.size();
    nodes.reserve(std::max(1, n / 2));
    if (n == 0) return;
    // the root is always an inner node; small scenes get two leaves
    nodes.push_back(BuildNode{});
    int m = (n <= LEAF) ? std::max(1, n / 2) : split(0, n, 0);
    Box lb = bounds(0, m), rb = bounds(m, n);
    int l = (n <= LEAF) ? make_leaf(0, m) : build(0, m, 1);
    int r;
    if (m < n)
      r = (n <= LEAF) ? make_leaf(m, n) : build(m, n, 1);
    else {
      r = l;
      rb = lb;
    }
    nodes[0].box[0] = lb;
    nodes[0].box[1] = rb;
    nodes[0].child[0] = l;
    nodes[0].child[1] = r;
  }
};

float round_down(double x, double pad) {
  float f = float(x - pad);
  if (double(f) > x - pad) f = std::nextafter(f, -INFINITY);
  return f;
}
float round_up(double x, double pad) {
  float f = float(x + pad);
  if (double(f) < x + pad) f = std::nextafter(f, INFINITY);
  return f;
}

template <typename T>
int upload(DrcbScene* s, const std::vector<T>& v, const T** out) {
  if (v.empty()) {
    *out = nullptr;
    return 0;
  }
  void* p = nullptr;
  DRCB_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
  s->allocs.push_back(p);
  s->stats.bytes += int64_t(v.size() * sizeof(T));
  DRCB_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<const T*>(p);
  return 0;
}

// Sutherland-Hodgman clip of a convex polygon to x[axis] <= pos (keep_le)
// or >= pos
void clip_poly(const std::vector<std::array<double, 3>>& in, int axis, double pos, bool keep_le,
               std::vector<std::array<double, 3>>& out) {
  out.clear();
  size_t n = in.size();
  for (size_t i = 0; i < n; ++i) {
    const auto& a = in[i];
    const auto& b = in[(i + 1) % n];
    double da = keep_le ? pos - a[axis] : a[axis] - pos;
    double db = keep_le ? pos - b[axis] : b[axis] - pos;
    if (da >= 0) out.push_back(a);
    if ((da >= 0) != (db >= 0)) {
      double t = da / (da - db);
      std::array<double, 3> c;
      for (int k = 0; k < 3; ++k) c[k] = a[k] + t * (b[k] - a[k]);
      c[axis] = pos;
      out.push_back(c);
    }
  }
}

void split_rec(const std::vector<std::array<double, 3>>& poly, const Box& box, double target,
               int depth, int prim, std::vector<Box>& rb, std::vector<int>& rp) {
  int ax = 0;
  double ext[3];
  for (int k = 0; k < 3; ++k) ext[k] = box.hi[k] - box.lo[k];
  for (int k = 1; k < 3; ++k)
    if (ext[k] > ext[ax]) ax = k;
  if (ext[ax] <= target || depth >= 7 || poly.size() < 3) {
    rb.push_back(box);
    rp.push_back(prim);
    return;
  }
  double mid = 0.5 * (box.lo[ax] + box.hi[ax]);
  std::vector<std::array<double, 3>> half;
  for (int side = 0; side < 2; ++side) {
    clip_poly(poly, ax, mid, side == 0, half);
    if (half.size() < 3) continue;
    Box hb;
    for (const auto& v : half) hb.grow_pt(v.data());
    // never let rounding shrink a piece outside the parent box
    for (int k = 0; k < 3; ++k) {
      hb.lo[k] = std::max(hb.lo[k], box.lo[k]);
      hb.hi[k] = std::min(hb.hi[k], box.hi[k]);
    }
    split_rec(half, hb, target, depth + 1, prim, rb, rp);
  }
}

void split_references(const std::vector<Box>& pb, const std::vector<double>& tri, int ns, int nq,
                      int nt, std::vector<Box>& rb, std::vector<int>& rp) {
  const int np = int(pb.size());
  rb.reserve(np);
  rp.reserve(np);
  std::vector<double> ext(np);
  for (int p = 0; p < np; ++p) {
    double e = 0;
    for (int k = 0; k < 3; ++k) e = std::max(e, pb[p].hi[k] - pb[p].lo[k]);
    ext[p] = e;
  }
  double target = INFINITY;
  if (nt >= 1024) {
    std::vector<double> te(ext.begin() + ns + nq, ext.end());
    std::nth_element(te.begin(), te.begin() + te.size() / 2, te.end());
    target = 4.0 * te[te.size() / 2];
  }
  for (int p = 0; p < np; ++p) {
    if (p < ns + nq || !(ext[p] > target)) {
      rb.push_back(pb[p]);
      rp.push_back(p);
      continue;
    }
    const double* t = &tri[13 * (p - ns - nq)];
    std::vector<std::array<double, 3>> poly(3);
    for (int k = 0; k < 3; ++k) {
      poly[0][k] = t[k];
      poly[1][k] = t[k] + t[3 + k];
      poly[2][k] = t[k] + t[6 + k];
    }
    split_rec(poly, pb[p], target, 0, p, rb, rp);
  }
}

inline void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

}  // namespace

DevCamera make_camera(const DrcbCamera& c) {
  DevCamera d;
  for (int k = 0; k < 3; ++k) {
    d.pos[k] = c.position[k];
    d.fwd[k] = c.forward[k];
    d.right[k] = c.right[k];
    d.up[k] = c.up[k];
  }
  d.tan_half = c.tan_half;
  d.W = c.width;
  d.H = c.height;
  d.aspect = double(c.width) / double(c.height);
  return d;
}

}  // namespace drcb

using namespace drcb;

extern "C" int drcb_scene_create(const DrcbSceneDesc* desc, DrcbScene** out) {
  if (!desc || !out) return fail(DRCB_ECONTRACT, "drcb_scene_create: null argument");
  *out = nullptr;
  const int ns = desc->n_spheres, nq = desc->n_quads, nt = desc->n_tris;
  const int nm = desc->n_materials, npl = desc->n_point_lights;
  if (ns < 0 || nq < 0 || nt < 0 || nm < 1 || npl < 0)
    return fail(DRCB_EVALIDATION, "scene: negative counts or no materials");
  auto check_mat = [&](const int32_t* m, int n) {
    for (int i = 0; i < n; ++i)
      if (m[i] < 0 || m[i] >= nm) return false;
    return true;
  };
  if (!check_mat(desc->sph_mat, ns) || !check_mat(desc->quad_mat, nq) ||
      !check_mat(desc->tri_mat, nt))
    return fail(DRCB_EVALIDATION, "scene: material index out of range");

  DrcbScene* s = new DrcbScene();
  cudaGetDevice(&s->device);
  DevScene& D = s->dev;
  std::memset(&D, 0, sizeof(D));
  D.n_s = ns;
  D.n_q = nq;
  D.n_t = nt;
  D.n_prims = ns + nq + nt;
  D.n_mat = nm;
  D.n_point = npl;

  // --- per-type tables (geometry.py:67-98), derived quantities in fp64
  std::vector<double> sph(5 * size_t(ns)), quad(18 * size_t(nq)), tri(13 * size_t(nt));
  std::vector<Box> pb(D.n_prims);
  for (int i = 0; i < ns; ++i) {
    const double* c = desc->sph_center + 3 * i;
    double r = desc->sph_radius[i];
    double* o = &sph[5 * i];
    o[0] = c[0]; o[1] = c[1]; o[2] = c[2]; o[3] = r; o[4] = r * r;
    for (int k = 0; k < 3; ++k) { pb[i].lo[k] = c[k] - r; pb[i].hi[k] = c[k] + r; }
  }
  std::vector<double> quad_area(nq);
  for (int i = 0; i < nq; ++i) {
    const double *c = desc->quad_corner + 3 * i, *eu = desc->quad_eu + 3 * i,
                 *ev = desc->quad_ev + 3 * i;
    double* o = &quad[18 * i];
    double n[3];
    cross3(eu, ev, n);
    double area = std::sqrt((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
    quad_area[i] = area;
    double den = std::max(area, 1e-300);
    for (int k = 0; k < 3; ++k) {
      o[k] = c[k]; o[3 + k] = eu[k]; o[6 + k] = ev[k]; o[9 + k] = n[k] / den;
    }
    double g11 = dot3(eu, eu), g22 = dot3(ev, ev), g12 = dot3(eu, ev);
    double det = std::max(g11 * g22 - g12 * g12, 1e-300);
    o[12] = g22 / det; o[13] = -g12 / det; o[14] = g11 / det;
    o[15] = dot3(c, o + 9); o[16] = dot3(c, eu); o[17] = dot3(c, ev);
    Box& b = pb[ns + i];
    double p[3];
    b.grow_pt(c);
    for (int k = 0; k < 3; ++k) p[k] = c[k] + eu[k];
    b.grow_pt(p);
    for (int k = 0; k < 3; ++k) p[k] = c[k] + ev[k];
    b.grow_pt(p);
    for (int k = 0; k < 3; ++k) p[k] = c[k] + eu[k] + ev[k];
    b.grow_pt(p);
  }
  for (int i = 0; i < nt; ++i) {
    const double *v0 = desc->tri_v0 + 3 * i, *v1 = desc->tri_v1 + 3 * i,
                 *v2 = desc->tri_v2 + 3 * i;
    double* o = &tri[13 * i];
    double e1[3], e2[3], n[3];
    for (int k = 0; k < 3; ++k) { e1[k] = v1[k] - v0[k]; e2[k] = v2[k] - v0[k]; }
    cross3(e1, e2, n);
    double ln = std::sqrt((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
    double den = std::max(ln, 1e-300);
    for (int k = 0; k < 3; ++k) {
      o[k] = v0[k]; o[3 + k] = e1[k]; o[6 + k] = e2[k]; o[9 + k] = n[k] / den;
    }
    o[12] = 0.5 * ln;
    Box& b = pb[ns + nq + i];
    double p[3];
    b.grow_pt(v0);
    for (int k = 0; k < 3; ++k) p[k] = v0[k] + e1[k];
    b.grow_pt(p);
    for (int k = 0; k < 3; ++k) p[k] = v0[k] + e2[k];
    b.grow_pt(p);
  }

  // --- lights (geometry.py:121-150)
  std::vector<int> mat_of(D.n_prims);
  for (int i = 0; i < ns; ++i) mat_of[i] = desc->sph_mat[i];
  for (int i = 0; i < nq; ++i) mat_of[ns + i] = desc->quad_mat[i];
  for (int i = 0; i < nt; ++i) mat_of[ns + nq + i] = desc->tri_mat[i];
  std::vector<uint8_t> emitter(nm), spec(nm);
  for (int m = 0; m < nm; ++m) {
    const double* e = desc->mat_emission + 3 * m;
    emitter[m] = (e[0] > 0 || e[1] > 0 || e[2] > 0);
    spec[m] = (desc->mat_kind[m] == DRCB_MIRROR || desc->mat_kind[m] == DRCB_TRANSMISSION);
  }
  std::vector<int> area_prim, area_mat, prim_light(std::max(D.n_prims, 1), -1);
  std::vector<double> area_area;
  for (int p = 0; p < D.n_prims; ++p) {
    if (!emitter[mat_of[p]]) continue;
    prim_light[p] = (int)area_prim.size();
    area_prim.push_back(p);
    area_mat.push_back(mat_of[p]);
    if (p < ns) {
      double r = desc->sph_radius[p];
      area_area.push_back(4.0 * M_PI * (r * r));
    } else if (p < ns + nq) {
      area_area.push_back(quad_area[p - ns]);
    } else {
      area_area.push_back(tri[13 * (p - ns - nq) + 12]);
    }
  }
  D.n_area = (int)area_prim.size();
  D.n_lights = npl + D.n_area;

  // --- BVH over primitive references. Early split clipping (Ernst &
  // Greiner 2007): primitives whose box is much larger than the typical one
  // (config 3/4's random triangles span the scene) are recursively cut at the
  // mid-plane of their box's longest axis, the triangle is clipped to each
  // half and each piece's tight box becomes a reference to the SAME prim.
  // Duplicate references cannot change the result (same t, same id).
  std::vector<Box> rb;
  std::vector<int> rp;
  split_references(pb, tri, ns, nq, nt, rb, rp);
  Builder B(rb, rp);
  if (const char* e = getenv("DRCB_BVH_SAH_CI")) B.sah_ci = atof(e);
  if (const char* e = getenv("DRCB_BVH_MAX_LEAF")) B.max_leaf = std::min(8, std::max(1, atoi(e)));
  B.run();
  s->stats.n_prims = D.n_prims;
  s->stats.n_refs = (int64_t)rb.size();
  s->stats.n_nodes = (int64_t)B.nodes.size();
  s->stats.n_leaves = B.n_leaves;
  s->stats.max_depth = B.max_depth;
  s->stats.n_lights = D.n_lights;
  if (B.max_depth + 2 > 64) {
    drcb_scene_destroy(s);
    return fail(DRCB_ECONFIG, "BVH deeper than the traversal stack");
  }
  double scale = 1.0;
  for (const Box& b : pb)
    for (int k = 0; k < 3; ++k)
      if (std::isfinite(b.lo[k]) && std::isfinite(b.hi[k]))
        scale = std::max(scale, std::max(std::fabs(b.lo[k]), std::fabs(b.hi[k])));
  const double pad = 4e-6 * scale;
  std::vector<float4> nodes(4 * B.nodes.size());
  for (size_t i = 0; i < B.nodes.size(); ++i) {
    const BuildNode& n = B.nodes[i];
    float lo[2][3], hi[2][3];
    for (int c = 0; c < 2; ++c)
      for (int k = 0; k < 3; ++k) {
        lo[c][k] = round_down(n.box[c].lo[k], pad);
        hi[c][k] = round_up(n.box[c].hi[k], pad);
      }
    nodes[4 * i + 0] = make_float4(lo[0][0], hi[0][0], lo[0][1], hi[0][1]);
    nodes[4 * i + 1] = make_float4(lo[1][0], hi[1][0], lo[1][1], hi[1][1]);
    nodes[4 * i + 2] = make_float4(lo[0][2], hi[0][2], lo[1][2], hi[1][2]);
    float c0, c1;
    std::memcpy(&c0, &n.child[0], 4);
    std::memcpy(&c1, &n.child[1], 4);
    nodes[4 * i + 3] = make_float4(c0, c1, 0.f, 0.f);
  }
  D.n_nodes = (int)B.nodes.size();
  size_t nslots = B.order.size();
  std::vector<float4> leaf_f(3 * nslots);
  std::vector<double> leaf_d(9 * nslots, 0.0);
  std::vector<int> leaf_id(nslots);
  for (size_t sl = 0; sl < nslots; ++sl) {
    int id = B.order[sl];
    leaf_id[sl] = id;
    float idf;
    std::memcpy(&idf, &id, 4);
    if (id >= ns + nq) {
      const double* t = &tri[13 * (id - ns - nq)];
      leaf_f[3 * sl + 0] = make_float4(float(t[0]), float(t[1]), float(t[2]), idf);
      leaf_f[3 * sl + 1] = make_float4(float(t[3]), float(t[4]), float(t[5]), 0.f);
      leaf_f[3 * sl + 2] = make_float4(float(t[6]), float(t[7]), float(t[8]), 0.f);
      for (int k = 0; k < 9; ++k) leaf_d[9 * sl + k] = t[k];
    } else {
      leaf_f[3 * sl + 0] = make_float4(0.f, 0.f, 0.f, idf);
      leaf_f[3 * sl + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      leaf_f[3 * sl + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }

  // --- materials
  std::vector<int> mk(desc->mat_kind, desc->mat_kind + nm);
  std::vector<double> malb(desc->mat_albedo, desc->mat_albedo + 3 * nm);
  std::vector<double> mexp(desc->mat_exponent, desc->mat_exponent + nm);
  std::vector<double> mior(desc->mat_ior, desc->mat_ior + nm);
  std::vector<double> memi(desc->mat_emission, desc->mat_emission + 3 * nm);
  std::vector<int> smat(desc->sph_mat, desc->sph_mat + ns), qmat(desc->quad_mat, desc->quad_mat + nq),
      tmat(desc->tri_mat, desc->tri_mat + nt);
  std::vector<double> ppos, pint;
  if (npl) {
    ppos.assign(desc->point_pos, desc->point_pos + 3 * npl);
    pint.assign(desc->point_intensity, desc->point_intensity + 3 * npl);
  }

  int rc = 0;
  rc |= upload(s, sph, &D.sph);
  rc |= upload(s, smat, &D.sph_mat);
  rc |= upload(s, quad, &D.quad);
  rc |= upload(s, qmat, &D.quad_mat);
  rc |= upload(s, tri, &D.tri);
  rc |= upload(s, tmat, &D.tri_mat);
  rc |= upload(s, nodes, &D.nodes);
  rc |= upload(s, leaf_f, &D.leaf_f);
  rc |= upload(s, leaf_d, &D.leaf_d);
  rc |= upload(s, leaf_id, &D.leaf_id);
  rc |= upload(s, mk, &D.mat_kind);
  rc |= upload(s, malb, &D.mat_albedo);
  rc |= upload(s, mexp, &D.mat_exp);
  rc |= upload(s, mior, &D.mat_ior);
  rc |= upload(s, memi, &D.mat_emis);
  rc |= upload(s, emitter, &D.mat_emitter);
  rc |= upload(s, spec, &D.mat_spec);
  rc |= upload(s, ppos, &D.point_pos);
  rc |= upload(s, pint, &D.point_int);
  rc |= upload(s, area_prim, &D.area_prim);
  rc |= upload(s, area_area, &D.area_area);
  rc |= upload(s, area_mat, &D.area_mat);
  rc |= upload(s, prim_light, &D.prim_light);
  if (rc) {
    drcb_scene_destroy(s);
    return rc;
  }
  for (int k = 0; k < 3; ++k) {
    D.env[k] = desc->environment[k];
    D.up[k] = desc->global_up[k];
    D.rot_up[k] = desc->rotated_up[k];
  }
  D.has_env = (D.env[0] > 0 || D.env[1] > 0 || D.env[2] > 0);
  *out = s;
  return 0;
}

extern "C" void drcb_scene_destroy(DrcbScene* s) {
  if (!s) return;
  for (void* p : s->allocs) cudaFree(p);
  delete s;
}

extern "C" int drcb_scene_stats(const DrcbScene* s, int64_t* out) {
  if (!s || !out) return fail(DRCB_ECONTRACT, "drcb_scene_stats: null argument");
  out[0] = s->stats.n_prims;
  out[1] = s->stats.n_nodes;
  out[2] = s->stats.n_leaves;
  out[3] = s->stats.max_depth;
  out[4] = s->stats.n_lights;
  out[5] = s->stats.bytes;
  out[6] = s->stats.n_refs;
  out[7] = 0;
  return 0;
}
