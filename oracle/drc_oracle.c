/*
 * drc_oracle.c — TEST INFRASTRUCTURE ONLY (see drc_oracle.h).
 *
 * Scalar fp64 restatement of the reference renderer, one ray at a time, in
 * the reference's operation order (compiled with -ffp-contract=off). OpenMP
 * parallelises over independent rays / maps only; every sample is keyed, so
 * results do not depend on the thread count (sampler.py:1-7).
 */
#include "drc_oracle.h"

#include <float.h>
#include <stdio.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TEPS 1e-4                 /* geometry.py:22 */
#define CHAIN_BOUND 16            /* integrators.py:35 */
#define THR_CUTOFF 1e-4           /* integrators.py:36 */
#define RRFLOOR 0.05              /* integrators.py:37 */
#define SHADE_BASE (1ull << 20)   /* integrators.py:38 */
#define UPDEG (1.0 - 1e-4)        /* bsdf.py:27 */
#define RES 32
#define NT (RES * RES)
static const double OPI = 3.141592653589793;

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ----------------------------------------------------------------- vectors */
typedef struct { double x, y, z; } v3;
static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, v3 b) { return V(a.x * b.x, a.y * b.y, a.z * b.z); }
static v3 vsc(double s, v3 a) { return V(s * a.x, s * a.y, s * a.z); }
static v3 vdivs(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static v3 vneg(v3 a) { return V(-a.x, -a.y, -a.z); }
static double vdot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
  return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vlen(v3 a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); }
static v3 L3(const double *p) { return V(p[0], p[1], p[2]); }
static void S3(double *p, v3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }
static int vfinite(v3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

/* ----------------------------------------------------------------- sampler */
/* sampler.py:25-78 */
static uint64_t mixz(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t hkeys(const uint64_t *k, int n) {
  uint64_t h = 0x853C49E6748FEA9Bull;
  for (int i = 0; i < n; ++i) h = mixz((h * 0x94D049BB133111EBull) ^ k[i]);
  return h;
}
typedef struct { int kind; uint64_t seed; uint64_t spp; } Smp;
static double smp_get(const Smp *s, uint64_t pix, uint64_t idx, uint64_t dim) {
  uint64_t k4[4] = {s->seed, pix, idx, dim};
  double jit = (double)(hkeys(k4, 4) >> 11) * 1.1102230246251565e-16;
  if (s->kind == 0 || s->spp == 1) return jit;
  uint64_t k5[4] = {s->seed, pix, dim, 0xD1Full};
  uint64_t off = hkeys(k5, 4) % s->spp;
  uint64_t stratum = (idx + off) % s->spp;
  return ((double)stratum + jit) / (double)s->spp;
}

/* ------------------------------------------------------------------- scene */
typedef struct { int node_or_leaf; } Unused;
typedef struct {
  double lo[3], hi[3];
  int left, right; /* right < 0: leaf with start=left, count=-right */
} ONode;

struct OrScene {
  int ns, nq, nt, np, nm, npl, narea, nl;
  double *sph;   /* c3, r, r2 */
  int *sph_mat;
  double *quad;  /* corner3 eu3 ev3 n3 inv3 d ceu cev area */
  int *quad_mat;
  double *tri;   /* v0 e1 e2 n area */
  int *tri_mat;
  int *mkind;
  double *malb, *mexp, *mior, *memi;
  unsigned char *memit, *mspec;
  double *ppos, *pint;
  int *aprim, *amat, *plight;
  double *aarea;
  double up[3], rup[3], env[3];
  int has_env;
  ONode *nodes;
  int nnodes;
  int *order;
};

static void prim_box(const OrScene *s, int p, double *lo, double *hi) {
  for (int k = 0; k < 3; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
  if (p < s->ns) {
    const double *q = s->sph + 5 * p;
    for (int k = 0; k < 3; ++k) { lo[k] = q[k] - q[3]; hi[k] = q[k] + q[3]; }
    return;
  }
  double pts[4][3];
  int npts;
  if (p < s->ns + s->nq) {
    const double *q = s->quad + 19 * (p - s->ns);
    for (int k = 0; k < 3; ++k) {
      pts[0][k] = q[k]; pts[1][k] = q[k] + q[3 + k]; pts[2][k] = q[k] + q[6 + k];
      pts[3][k] = q[k] + q[3 + k] + q[6 + k];
    }
    npts = 4;
  } else {
    const double *t = s->tri + 13 * (p - s->ns - s->nq);
    for (int k = 0; k < 3; ++k) { pts[0][k] = t[k]; pts[1][k] = t[k] + t[3 + k]; pts[2][k] = t[k] + t[6 + k]; }
    npts = 3;
  }
  for (int i = 0; i < npts; ++i)
    for (int k = 0; k < 3; ++k) {
      if (pts[i][k] < lo[k]) lo[k] = pts[i][k];
      if (pts[i][k] > hi[k]) hi[k] = pts[i][k];
    }
}

/* median-split BVH; results are tree-independent by the tie rule */
typedef struct { double *cen; int axis; } SortCtx;
static SortCtx g_sort;
static int cmp_cen(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  double cx = g_sort.cen[3 * x + g_sort.axis], cy = g_sort.cen[3 * y + g_sort.axis];
  if (cx < cy) return -1;
  if (cx > cy) return 1;
  return (x > y) - (x < y);
}

static int build_rec(OrScene *s, int *ids, int n, double *plo, double *phi, double *cen,
                     double pad) {
  int me = s->nnodes++;
  ONode *nd = &s->nodes[me];
  for (int k = 0; k < 3; ++k) { nd->lo[k] = INFINITY; nd->hi[k] = -INFINITY; }
  double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < n; ++i) {
    int p = ids[i];
    for (int k = 0; k < 3; ++k) {
      if (plo[3 * p + k] < nd->lo[k]) nd->lo[k] = plo[3 * p + k];
      if (phi[3 * p + k] > nd->hi[k]) nd->hi[k] = phi[3 * p + k];
      if (cen[3 * p + k] < clo[k]) clo[k] = cen[3 * p + k];
      if (cen[3 * p + k] > chi[k]) chi[k] = cen[3 * p + k];
    }
  }
  for (int k = 0; k < 3; ++k) { nd->lo[k] -= pad; nd->hi[k] += pad; }
  if (n <= 4) {
    nd->left = (int)(ids - s->order);
    nd->right = -n;
    return me;
  }
  int ax = 0;
  for (int k = 1; k < 3; ++k)
    if (chi[k] - clo[k] > chi[ax] - clo[ax]) ax = k;
  g_sort.cen = cen;
  g_sort.axis = ax;
  qsort(ids, (size_t)n, sizeof(int), cmp_cen);
  int h = n / 2;
  int l = build_rec(s, ids, h, plo, phi, cen, pad);
  int r = build_rec(s, ids + h, n - h, plo, phi, cen, pad);
  s->nodes[me].left = l;
  s->nodes[me].right = r;
  return me;
}

OrScene *or_scene_create(const OrSceneDesc *d) {
  OrScene *s = (OrScene *)calloc(1, sizeof(OrScene));
  s->ns = d->n_spheres; s->nq = d->n_quads; s->nt = d->n_tris;
  s->np = s->ns + s->nq + s->nt; s->nm = d->n_materials; s->npl = d->n_point_lights;
  s->sph = (double *)calloc((size_t)5 * s->ns + 1, sizeof(double));
  s->sph_mat = (int *)calloc((size_t)s->ns + 1, sizeof(int));
  for (int i = 0; i < s->ns; ++i) {
    double r = d->sph_radius[i];
    for (int k = 0; k < 3; ++k) s->sph[5 * i + k] = d->sph_center[3 * i + k];
    s->sph[5 * i + 3] = r;
    s->sph[5 * i + 4] = r * r;
    s->sph_mat[i] = d->sph_mat[i];
  }
  /* geometry.py:74-88 */
  s->quad = (double *)calloc((size_t)19 * s->nq + 1, sizeof(double));
  s->quad_mat = (int *)calloc((size_t)s->nq + 1, sizeof(int));
  for (int i = 0; i < s->nq; ++i) {
    double *q = s->quad + 19 * i;
    v3 c = L3(d->quad_corner + 3 * i), eu = L3(d->quad_eu + 3 * i), ev = L3(d->quad_ev + 3 * i);
    v3 n = vcross(eu, ev);
    double area = vlen(n);
    v3 nn = vdivs(n, area > 1e-300 ? area : 1e-300);
    S3(q, c); S3(q + 3, eu); S3(q + 6, ev); S3(q + 9, nn);
    double g11 = vdot(eu, eu), g22 = vdot(ev, ev), g12 = vdot(eu, ev);
    double det = g11 * g22 - g12 * g12;
    if (det < 1e-300) det = 1e-300;
    q[12] = g22 / det; q[13] = -g12 / det; q[14] = g11 / det;
    q[15] = vdot(c, nn); q[16] = vdot(c, eu); q[17] = vdot(c, ev); q[18] = area;
    s->quad_mat[i] = d->quad_mat[i];
  }
  /* geometry.py:90-98 */
  s->tri = (double *)calloc((size_t)13 * s->nt + 1, sizeof(double));
  s->tri_mat = (int *)calloc((size_t)s->nt + 1, sizeof(int));
  for (int i = 0; i < s->nt; ++i) {
    double *t = s->tri + 13 * i;
    v3 a = L3(d->tri_v0 + 3 * i);
    v3 e1 = vsub(L3(d->tri_v1 + 3 * i), a), e2 = vsub(L3(d->tri_v2 + 3 * i), a);
    v3 n = vcross(e1, e2);
    double ln = vlen(n);
    S3(t, a); S3(t + 3, e1); S3(t + 6, e2); S3(t + 9, vdivs(n, ln > 1e-300 ? ln : 1e-300));
    t[12] = 0.5 * ln;
    s->tri_mat[i] = d->tri_mat[i];
  }
  int nm = s->nm;
  s->mkind = (int *)malloc(sizeof(int) * nm);
  s->malb = (double *)malloc(sizeof(double) * 3 * nm);
  s->mexp = (double *)malloc(sizeof(double) * nm);
  s->mior = (double *)malloc(sizeof(double) * nm);
  s->memi = (double *)malloc(sizeof(double) * 3 * nm);
  s->memit = (unsigned char *)malloc(nm);
  s->mspec = (unsigned char *)malloc(nm);
  for (int m = 0; m < nm; ++m) {
    s->mkind[m] = d->mat_kind[m];
    s->mexp[m] = d->mat_exponent[m];
    s->mior[m] = d->mat_ior[m];
    for (int k = 0; k < 3; ++k) {
      s->malb[3 * m + k] = d->mat_albedo[3 * m + k];
      s->memi[3 * m + k] = d->mat_emission[3 * m + k];
    }
    s->memit[m] = s->memi[3 * m] > 0 || s->memi[3 * m + 1] > 0 || s->memi[3 * m + 2] > 0;
    s->mspec[m] = d->mat_kind[m] == 2 || d->mat_kind[m] == 3;
  }
  s->ppos = (double *)calloc((size_t)3 * s->npl + 1, sizeof(double));
  s->pint = (double *)calloc((size_t)3 * s->npl + 1, sizeof(double));
  for (int i = 0; i < 3 * s->npl; ++i) { s->ppos[i] = d->point_pos[i]; s->pint[i] = d->point_intensity[i]; }
  /* emitter table, geometry.py:121-150 */
  s->plight = (int *)malloc(sizeof(int) * (s->np > 0 ? s->np : 1));
  s->aprim = (int *)malloc(sizeof(int) * (s->np > 0 ? s->np : 1));
  s->amat = (int *)malloc(sizeof(int) * (s->np > 0 ? s->np : 1));
  s->aarea = (double *)malloc(sizeof(double) * (s->np > 0 ? s->np : 1));
  s->narea = 0;
  for (int p = 0; p < s->np; ++p) {
    int m = p < s->ns ? s->sph_mat[p] : p < s->ns + s->nq ? s->quad_mat[p - s->ns] : s->tri_mat[p - s->ns - s->nq];
    s->plight[p] = -1;
    if (!s->memit[m]) continue;
    s->plight[p] = s->narea;
    s->aprim[s->narea] = p;
    s->amat[s->narea] = m;
    if (p < s->ns) { double r = s->sph[5 * p + 3]; s->aarea[s->narea] = 4.0 * OPI * (r * r); }
    else if (p < s->ns + s->nq) s->aarea[s->narea] = s->quad[19 * (p - s->ns) + 18];
    else s->aarea[s->narea] = s->tri[13 * (p - s->ns - s->nq) + 12];
    s->narea++;
  }
  s->nl = s->npl + s->narea;
  for (int k = 0; k < 3; ++k) { s->up[k] = d->global_up[k]; s->rup[k] = d->rotated_up[k]; s->env[k] = d->environment[k]; }
  s->has_env = s->env[0] > 0 || s->env[1] > 0 || s->env[2] > 0;
  /* BVH */
  if (s->np > 0) {
    double *plo = (double *)malloc(sizeof(double) * 3 * s->np), *phi = (double *)malloc(sizeof(double) * 3 * s->np);
    double *cen = (double *)malloc(sizeof(double) * 3 * s->np);
    double scale = 1.0;
    for (int p = 0; p < s->np; ++p) {
      prim_box(s, p, plo + 3 * p, phi + 3 * p);
      for (int k = 0; k < 3; ++k) {
        cen[3 * p + k] = 0.5 * (plo[3 * p + k] + phi[3 * p + k]);
        if (fabs(plo[3 * p + k]) > scale) scale = fabs(plo[3 * p + k]);
        if (fabs(phi[3 * p + k]) > scale) scale = fabs(phi[3 * p + k]);
      }
    }
    s->order = (int *)malloc(sizeof(int) * s->np);
    for (int p = 0; p < s->np; ++p) s->order[p] = p;
    s->nodes = (ONode *)malloc(sizeof(ONode) * (size_t)(2 * s->np + 1));
    s->nnodes = 0;
    build_rec(s, s->order, s->np, plo, phi, cen, 1e-9 * scale);
    free(plo); free(phi); free(cen);
  }
  return s;
}

void or_scene_destroy(OrScene *s) {
  if (!s) return;
  free(s->sph); free(s->sph_mat); free(s->quad); free(s->quad_mat); free(s->tri); free(s->tri_mat);
  free(s->mkind); free(s->malb); free(s->mexp); free(s->mior); free(s->memi); free(s->memit);
  free(s->mspec); free(s->ppos); free(s->pint); free(s->plight); free(s->aprim); free(s->amat);
  free(s->aarea); free(s->nodes); free(s->order);
  free(s);
}

/* ------------------------------------------------------ primitive tests */
/* geometry.py:468-523 (scalar path, bit-identical to the batch kernels) */
static int hit_sphere(const OrScene *s, int i, v3 O, v3 D, double tmin, double tbest, double *out) {
  const double *q = s->sph + 5 * i;
  v3 oc = vsub(O, L3(q));
  double b = vdot(oc, D);
  double c = vdot(oc, oc) - q[4];
  double disc = b * b - c;
  if (disc < 0.0) return 0;
  double sq = sqrt(disc);
  double t = -b - sq;
  if (t <= tmin) t = -b + sq;
  if (tmin < t && t <= tbest) { *out = t; return 1; }
  return 0;
}
static int hit_quad(const OrScene *s, int i, v3 O, v3 D, double tmin, double tbest, double *out) {
  const double *q = s->quad + 19 * i;
  v3 n = L3(q + 9);
  double den = vdot(D, n);
  if (fabs(den) <= 1e-12) return 0;
  double t = (q[15] - vdot(O, n)) / den;
  if (!(tmin < t && t <= tbest)) return 0;
  v3 eu = L3(q + 3), ev = L3(q + 6);
  double meu = (vdot(O, eu) - q[16]) + t * vdot(D, eu);
  double mev = (vdot(O, ev) - q[17]) + t * vdot(D, ev);
  double a = q[12] * meu + q[13] * mev;
  double b2 = q[13] * meu + q[14] * mev;
  if (0.0 <= a && a <= 1.0 && 0.0 <= b2 && b2 <= 1.0) { *out = t; return 1; }
  return 0;
}
static int hit_tri(const OrScene *s, int i, v3 O, v3 D, double tmin, double tbest, double *out) {
  const double *q = s->tri + 13 * i;
  v3 e1 = L3(q + 3), e2 = L3(q + 6);
  v3 pv = vcross(D, e2);
  double det = vdot(pv, e1);
  if (fabs(det) <= 1e-14) return 0;
  double inv = 1.0 / det;
  v3 tv = vsub(O, L3(q));
  double u = vdot(tv, pv) * inv;
  if (u < 0.0 || u > 1.0) return 0;
  v3 qv = vcross(tv, e1);
  double v = vdot(qv, D) * inv;
  if (v < 0.0 || u + v > 1.0) return 0;
  double t = vdot(qv, e2) * inv;
  if (tmin < t && t <= tbest) { *out = t; return 1; }
  return 0;
}

/* nearest hit, ties -> lowest prim id (geometry.py:199-214, 422-460);
 * any_hit stops at the first hit in range (shadow rays). */
static int cast(const OrScene *s, v3 O, v3 D, double tmin, double tmax, int any_hit, double *tout) {
  int best = -1;
  double bt = tmax;
  if (s->np == 0) return -1;
  double inv[3];
  const double dd[3] = {D.x, D.y, D.z}, oo[3] = {O.x, O.y, O.z};
  for (int k = 0; k < 3; ++k) inv[k] = 1.0 / (fabs(dd[k]) > 1e-300 ? dd[k] : 1e-300);
  int stack[128];
  int sp = 0;
  stack[sp++] = 0;
  while (sp) {
    const ONode *nd = &s->nodes[stack[--sp]];
    double tn = 0.0, tf = bt * (1.0 + 1e-12);
    int miss = 0;
    for (int k = 0; k < 3; ++k) {
      double a = (nd->lo[k] - oo[k]) * inv[k], b = (nd->hi[k] - oo[k]) * inv[k];
      double lo = a < b ? a : b, hi = a < b ? b : a;
      if (lo > tn) tn = lo;
      if (hi < tf) tf = hi;
      if (tn > tf) { miss = 1; break; }
    }
    if (miss) continue;
    if (nd->right < 0) {
      for (int j = nd->left; j < nd->left - nd->right; ++j) {
        int p = s->order[j];
        double t;
        double lim = any_hit ? tmax : bt;
        int ok = p < s->ns ? hit_sphere(s, p, O, D, tmin, lim, &t)
                 : p < s->ns + s->nq ? hit_quad(s, p - s->ns, O, D, tmin, lim, &t)
                                     : hit_tri(s, p - s->ns - s->nq, O, D, tmin, lim, &t);
        if (!ok) continue;
        if (any_hit) { *tout = t; return p; }
        if (t < bt || (t == bt && (best < 0 || p < best))) { bt = t; best = p; }
      }
    } else {
      stack[sp++] = nd->right;
      stack[sp++] = nd->left;
    }
  }
  *tout = best >= 0 ? bt : INFINITY;
  return best;
}

typedef struct { int hit, prim, mat; double t; v3 pos, n; } Isect;
static Isect trace1(const OrScene *s, v3 O, v3 D, double tmin, double tmax) {
  Isect h;
  double t;
  h.prim = cast(s, O, D, tmin, tmax, 0, &t);
  h.hit = h.prim >= 0;
  h.t = h.hit ? t : INFINITY;
  h.pos = vadd(O, vsc(h.hit ? t : 0.0, D));
  h.n = V(0, 0, 0);
  h.mat = -1;
  if (h.hit) {
    int p = h.prim;
    if (p < s->ns) {
      double r = s->sph[5 * p + 3];
      v3 dd = vsub(h.pos, L3(s->sph + 5 * p));
      h.n = V(dd.x / r, dd.y / r, dd.z / r);
      h.mat = s->sph_mat[p];
    } else if (p < s->ns + s->nq) {
      h.n = L3(s->quad + 19 * (p - s->ns) + 9);
      h.mat = s->quad_mat[p - s->ns];
    } else {
      h.n = L3(s->tri + 13 * (p - s->ns - s->nq) + 9);
      h.mat = s->tri_mat[p - s->ns - s->nq];
    }
  }
  return h;
}

void or_intersect(const OrScene *s, const double *O, const double *D, int64_t n, const double *tmin,
                  const double *tmax, int record, uint8_t *hit, double *t, int64_t *prim,
                  int32_t *mat, double *pos, double *nrm) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    Isect h = trace1(s, L3(O + 3 * i), L3(D + 3 * i), tmin ? tmin[i] : TEPS, tmax ? tmax[i] : INFINITY);
    hit[i] = (uint8_t)h.hit;
    if (t) t[i] = h.t;
    if (prim) prim[i] = h.prim;
    if (record) {
      if (mat) mat[i] = h.mat;
      if (pos) S3(pos + 3 * i, h.pos);
      if (nrm) S3(nrm + 3 * i, h.n);
    }
  }
}

/* ------------------------------------------------------------- frames/BSDF */
typedef struct { v3 t, b, n; } Frm;
static v3 to_loc(const Frm *f, v3 v) { return V(vdot(v, f->t), vdot(v, f->b), vdot(v, f->n)); }
static v3 to_wld(const Frm *f, v3 l) { return vadd(vadd(vsc(l.x, f->t), vsc(l.y, f->b)), vsc(l.z, f->n)); }

/* build_frames_batch, bsdf.py:78-96 */
static Frm frame_b(const OrScene *s, v3 n) {
  v3 up = L3(s->up);
  v3 ref = fabs(vdot(n, up)) > UPDEG ? L3(s->rup) : up;
  v3 t = vcross(ref, n);
  double nr = vlen(t);
  if (nr < 1e-9) { t = vcross(V(1, 0, 0), n); nr = vlen(t); }
  Frm f;
  f.t = vdivs(t, nr);
  f.b = vcross(n, f.t);
  f.n = n;
  return f;
}
/* _rotated_up / build_frame, bsdf.py:45-75 */
static v3 rot_up(v3 up) {
  v3 ax[2] = {{0, 1, 0}, {1, 0, 0}};
  for (int k = 0; k < 2; ++k) {
    v3 w = vsub(ax[k], vsc(vdot(ax[k], up), up));
    double nw = vlen(w);
    if (nw > 1e-6) return vdivs(w, nw);
  }
  return V(0, 0, 1);
}
static Frm frame_s(const OrScene *s, v3 n) {
  v3 up = L3(s->up);
  v3 ref = fabs(vdot(n, up)) <= UPDEG ? up : L3(s->rup);
  v3 t = vcross(ref, n);
  double nr = vlen(t);
  if (nr < 1e-9) {
    v3 xa = V(1, 0, 0);
    ref = fabs(vdot(n, xa)) <= UPDEG ? xa : rot_up(xa);
    t = vcross(ref, n);
    nr = vlen(t);
  }
  Frm f;
  f.t = vdivs(t, nr);
  f.b = vcross(n, f.t);
  f.n = n;
  return f;
}

static double schl(double f0, double c) {
  c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
  return f0 + (1.0 - f0) * pow(1.0 - c, 5.0);
}
static double powh(double a, double b) { double a2 = a * a; return a2 / (a2 + b * b); }

/* eval_batch, bsdf.py:234-254 */
static void bsdf_f(const OrScene *s, int m, v3 lo, v3 li, v3 *f, double *pdf) {
  int above = lo.z > 0.0 && li.z > 0.0;
  v3 alb = L3(s->malb + 3 * m);
  *f = V(0, 0, 0);
  *pdf = 0.0;
  if (s->mkind[m] == 0) {
    if (above) *f = V(alb.x / OPI, alb.y / OPI, alb.z / OPI);
    *pdf = (li.z > 0.0 ? li.z : 0.0) / OPI;
  } else if (s->mkind[m] == 1) {
    double e = s->mexp[m];
    double ca = (-lo.x * li.x - lo.y * li.y) + lo.z * li.z;
    if (ca < 0.0) ca = 0.0;
    double lobe = pow(ca, e);
    double k = (e + 2.0) / (2.0 * OPI) * lobe;
    if (above) *f = V(alb.x * k, alb.y * k, alb.z * k);
    *pdf = (e + 1.0) / (2.0 * OPI) * lobe;
  }
}

typedef struct { v3 li, val; double pdf; int spec; } BS;
/* sample_batch, bsdf.py:257-327 */
static BS bsdf_s(const OrScene *s, int m, v3 lo, double u1, double u2, int entering) {
  BS r;
  int kind = s->mkind[m];
  v3 alb = L3(s->malb + 3 * m);
  r.pdf = 1.0;
  r.val = V(0, 0, 0);
  r.spec = kind >= 2;
  if (kind == 0) {
    double rr = sqrt(u1), ph = 2.0 * OPI * u2, z = sqrt(1.0 - u1 > 0.0 ? 1.0 - u1 : 0.0);
    r.li = V(rr * cos(ph), rr * sin(ph), z);
    r.pdf = z / OPI > 1e-12 ? z / OPI : 1e-12;
    if (lo.z > 0.0) r.val = V(alb.x / OPI, alb.y / OPI, alb.z / OPI);
  } else if (kind == 1) {
    double e = s->mexp[m];
    double ca = pow(u1, 1.0 / (e + 1.0));
    double sa2 = 1.0 - ca * ca;
    double sa = sqrt(sa2 > 0.0 ? sa2 : 0.0), ph = 2.0 * OPI * u2;
    v3 lobe = V(sa * cos(ph), sa * sin(ph), ca);
    v3 ax = V(-lo.x, -lo.y, lo.z);
    v3 a = fabs(ax.x) > 0.9 ? V(0, 1, 0) : V(1, 0, 0);
    v3 t = vcross(a, ax);
    double nt = vlen(t);
    t = vdivs(t, nt > 1e-12 ? nt : 1e-12);
    v3 b = vcross(ax, t);
    v3 w = vadd(vadd(vsc(lobe.x, t), vsc(lobe.y, b)), vsc(lobe.z, ax));
    r.li = w;
    double ld = pow(ca, e);
    double pd = (e + 1.0) / (2.0 * OPI) * ld;
    r.pdf = pd > 1e-12 ? pd : 1e-12;
    if (w.z > 0.0 && lo.z > 0.0) {
      double k = (e + 2.0) / (2.0 * OPI) * ld;
      r.val = V(alb.x * k, alb.y * k, alb.z * k);
    }
  } else if (kind == 2) {
    r.li = V(-lo.x, -lo.y, lo.z);
    r.val = V(schl(alb.x, lo.z), schl(alb.y, lo.z), schl(alb.z, lo.z));
  } else {
    double ior = s->mior[m];
    double eta = entering ? 1.0 / ior : ior;
    double ci = lo.z;
    double c2 = 1.0 - ci * ci;
    double s2t = eta * eta * (c2 > 0.0 ? c2 : 0.0);
    double q = (ior - 1.0) / (ior + 1.0);
    double fr = schl(q * q, ci);
    int refl = s2t >= 1.0 || u1 < fr;
    double ct2 = 1.0 - s2t;
    double ct = sqrt(ct2 > 0.0 ? ct2 : 0.0);
    r.li = refl ? V(-lo.x, -lo.y, ci) : V(-eta * lo.x, -eta * lo.y, -ct);
    r.val = alb;
  }
  return r;
}

/* ------------------------------------------------------------------ lights */
typedef struct { v3 wl, ratio; double dist, pdf; int delta, valid; } LS;
/* _sample_lights, integrators.py:86-161 */
static LS sample_light(const OrScene *s, v3 pos, double us, double ua, double ub) {
  LS L;
  int nl = s->nl;
  int64_t pk = (int64_t)(us * (double)nl);
  int pick = (int)(pk < nl - 1 ? pk : nl - 1);
  L.delta = pick < s->npl;
  L.wl = V(0, 0, 0);
  L.ratio = V(0, 0, 0);
  L.dist = INFINITY;
  L.pdf = INFINITY;
  if (L.delta) {
    v3 vec = vsub(L3(s->ppos + 3 * pick), pos);
    double d2 = vdot(vec, vec), d = sqrt(d2);
    L.wl = vdivs(vec, d);
    L.dist = d;
    double f = (double)nl / d2;
    v3 I = L3(s->pint + 3 * pick);
    L.ratio = V(I.x * f, I.y * f, I.z * f);
    L.valid = d > 4 * TEPS;
    return L;
  }
  int k = pick - s->npl, p = s->aprim[k];
  double area = s->aarea[k];
  v3 le = L3(s->memi + 3 * s->amat[k]), y, nl3;
  if (p < s->ns) {
    double z = 1.0 - 2.0 * ua, rr2 = 1.0 - z * z;
    double rr = sqrt(rr2 > 0.0 ? rr2 : 0.0), ph = 2.0 * OPI * ub;
    v3 ds = V(rr * cos(ph), rr * sin(ph), z);
    y = vadd(L3(s->sph + 5 * p), vsc(s->sph[5 * p + 3], ds));
    nl3 = ds;
  } else if (p < s->ns + s->nq) {
    const double *q = s->quad + 19 * (p - s->ns);
    y = vadd(vadd(L3(q), vsc(ua, L3(q + 3))), vsc(ub, L3(q + 6)));
    nl3 = L3(q + 9);
  } else {
    const double *t = s->tri + 13 * (p - s->ns - s->nq);
    double su = sqrt(ua);
    y = vadd(vadd(L3(t), vsc(1.0 - su, L3(t + 3))), vsc(ub * su, L3(t + 6)));
    nl3 = L3(t + 9);
  }
  v3 vec = vsub(y, pos);
  double d2 = vdot(vec, vec);
  if (d2 < 1e-24) d2 = 1e-24;
  double d = sqrt(d2);
  v3 w = vdivs(vec, d);
  double cl = -vdot(nl3, w);
  int ok = cl > 1e-9 && d > 4 * TEPS;
  double pdf = ok ? d2 / (cl > 1e-12 ? cl : 1e-12) / area / (double)nl : INFINITY;
  L.wl = w;
  L.dist = d;
  if (ok) L.ratio = V(le.x / pdf, le.y / pdf, le.z / pdf);
  L.pdf = pdf;
  L.valid = ok;
  return L;
}
/* _nee_pdf_for_hit, integrators.py:164-169 */
static double nee_pdf(const OrScene *s, int prim, double t, double cl) {
  int li = s->plight[prim];
  if (li < 0) return 0.0;
  return t * t / (cl > 1e-12 ? cl : 1e-12) / s->aarea[li] / (double)(s->nl > 1 ? s->nl : 1);
}

static v3 do_nee(const OrScene *s, const Smp *sm, uint64_t pix, uint64_t idx, uint64_t base,
                 v3 pos, v3 nf, const Frm *fr, int m, v3 wol) {
  LS ls = sample_light(s, pos, smp_get(sm, pix, idx, base), smp_get(sm, pix, idx, base + 1),
                       smp_get(sm, pix, idx, base + 2));
  v3 wll = to_loc(fr, ls.wl);
  if (!(ls.valid && wll.z > 0.0)) return V(0, 0, 0);
  v3 f;
  double pb;
  bsdf_f(s, m, wol, wll, &f, &pb);
  v3 c = vmul(f, V(ls.ratio.x * wll.z, ls.ratio.y * wll.z, ls.ratio.z * wll.z));
  double w = ls.delta ? 1.0 : powh(ls.pdf, pb);
  c = vmul(c, V(w, w, w));
  if (!(c.x > 0 || c.y > 0 || c.z > 0)) return V(0, 0, 0);
  double tt;
  if (cast(s, vadd(pos, vsc(TEPS, nf)), ls.wl, TEPS, ls.dist - 2 * TEPS, 1, &tt) >= 0) return V(0, 0, 0);
  return c;
}

/* -------------------------------------------------------------- estimators */
/* trace_radiance_batch for one path, integrators.py:175-302 */
static v3 path_li(const OrScene *s, const Smp *sm, v3 O, v3 D, uint64_t pix, uint64_t idx, int maxd,
                  int skip0, int rrs, int *nonfin) {
  v3 L = V(0, 0, 0), beta = V(1, 1, 1), env = L3(s->env);
  double ppdf = 0.0;
  int pdelta = 1;
  for (int seg = 0; seg <= maxd; ++seg) {
    Isect h = trace1(s, O, D, TEPS, INFINITY);
    int skip = seg == 0 && skip0;
    if (!h.hit) {
      if (s->has_env && !skip) L = vadd(L, vmul(beta, env));
      break;
    }
    int face = vdot(h.n, D) < 0.0;
    if (s->memit[h.mat] && face && !skip) {
      double w = 1.0;
      if (seg > 0 && !pdelta) w = powh(ppdf, nee_pdf(s, h.prim, h.t, -vdot(h.n, D)));
      L = vadd(L, vmul(vmul(beta, L3(s->memi + 3 * h.mat)), V(w, w, w)));
    }
    if (seg == maxd) break;
    v3 nf = face ? h.n : vneg(h.n);
    Frm fr = frame_b(s, nf);
    v3 wol = to_loc(&fr, vneg(D));
    uint64_t base = 2 + 8 * (uint64_t)seg;
    if (s->nl > 0 && !s->mspec[h.mat]) L = vadd(L, vmul(beta, do_nee(s, sm, pix, idx, base, h.pos, nf, &fr, h.mat, wol)));
    BS b = bsdf_s(s, h.mat, wol, smp_get(sm, pix, idx, base + 3), smp_get(sm, pix, idx, base + 4), face);
    double ci = fabs(b.li.z);
    v3 wgt = b.spec ? b.val : vmul(b.val, V(ci / b.pdf, ci / b.pdf, ci / b.pdf));
    beta = vmul(beta, wgt);
    O = vadd(h.pos, vsc(TEPS * (b.li.z >= 0.0 ? 1.0 : -1.0), nf));
    D = to_wld(&fr, b.li);
    ppdf = b.pdf;
    pdelta = b.spec;
    int alive = (beta.x > 0 || beta.y > 0 || beta.z > 0) && vfinite(beta);
    if (seg + 1 >= rrs) {
      double mx = beta.x;
      if (beta.y > mx) mx = beta.y;
      if (beta.z > mx) mx = beta.z;
      double q = mx < RRFLOOR ? RRFLOOR : (mx > 1.0 ? 1.0 : mx);
      int surv = smp_get(sm, pix, idx, base + 5) < q;
      beta = vdivs(beta, q);
      alive = alive && surv;
    }
    if (!alive) break;
  }
  if (!vfinite(L)) { L = V(0, 0, 0); ++*nonfin; }
  return L;
}

/* li_direct_batch for one path, integrators.py:305-424 */
static v3 direct_li(const OrScene *s, const Smp *sm, v3 O, v3 D, uint64_t pix, uint64_t idx, int incbg,
                    int *nonfin) {
  v3 L = V(0, 0, 0), beta = V(1, 1, 1), env = L3(s->env);
  int ph1 = 0, mlive = 0;
  double mpdf = 0.0;
  for (int seg = 0; seg < CHAIN_BOUND; ++seg) {
    Isect h = trace1(s, O, D, TEPS, INFINITY);
    if (!h.hit) {
      if (s->has_env && (ph1 || incbg)) L = vadd(L, vmul(beta, env));
      break;
    }
    int face = vdot(h.n, D) < 0.0;
    if (s->memit[h.mat] && face) {
      double w = mlive ? powh(mpdf, nee_pdf(s, h.prim, h.t, -vdot(h.n, D))) : 1.0;
      L = vadd(L, vmul(vmul(beta, L3(s->memi + 3 * h.mat)), V(w, w, w)));
    }
    int spec = s->mspec[h.mat];
    if (!(spec || !ph1)) break;
    v3 nf = face ? h.n : vneg(h.n);
    Frm fr = frame_b(s, nf);
    v3 wol = to_loc(&fr, vneg(D));
    uint64_t base = 2 + 8 * (uint64_t)seg;
    int shade = !spec && !ph1;
    if (shade && s->nl > 0) L = vadd(L, vmul(beta, do_nee(s, sm, pix, idx, base, h.pos, nf, &fr, h.mat, wol)));
    BS b = bsdf_s(s, h.mat, wol, smp_get(sm, pix, idx, base + 3), smp_get(sm, pix, idx, base + 4), face);
    double ci = fabs(b.li.z);
    v3 wgt = b.spec ? b.val : vmul(b.val, V(ci / b.pdf, ci / b.pdf, ci / b.pdf));
    beta = vmul(beta, wgt);
    O = vadd(h.pos, vsc(TEPS * (b.li.z >= 0.0 ? 1.0 : -1.0), nf));
    D = to_wld(&fr, b.li);
    mlive = shade && !b.spec;
    mpdf = mlive ? b.pdf : 0.0;
    ph1 = ph1 || shade;
    if (!((beta.x > THR_CUTOFF || beta.y > THR_CUTOFF || beta.z > THR_CUTOFF) && vfinite(beta))) break;
  }
  if (!vfinite(L)) { L = V(0, 0, 0); ++*nonfin; }
  return L;
}

int64_t or_li_direct(const OrScene *s, const OrCfg *cfg, const double *O, const double *D,
                     const uint64_t *pix, const uint64_t *smp, int64_t n, int include_bg, double *L) {
  Smp sm = {cfg->sampler_kind, cfg->seed, (uint64_t)(cfg->direct_spp > 1 ? cfg->direct_spp : 1)};
  int64_t nf = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : nf)
  for (int64_t i = 0; i < n; ++i) {
    int c = 0;
    S3(L + 3 * i, direct_li(s, &sm, L3(O + 3 * i), L3(D + 3 * i), pix[i], smp[i], include_bg, &c));
    nf += c;
  }
  return nf;
}

int64_t or_trace_radiance(const OrScene *s, const OrCfg *cfg, const double *O, const double *D,
                          const uint64_t *pix, const uint64_t *smp, int64_t n, int max_depth,
                          int skip_first, int rr_start, double *L) {
  Smp sm = {cfg->sampler_kind, cfg->seed, (uint64_t)(cfg->direct_spp > 1 ? cfg->direct_spp : 1)};
  int64_t nf = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : nf)
  for (int64_t i = 0; i < n; ++i) {
    int c = 0;
    S3(L + 3 * i, path_li(s, &sm, L3(O + 3 * i), L3(D + 3 * i), pix[i], smp[i], max_depth, skip_first, rr_start, &c));
    nf += c;
  }
  return nf;
}

/* primary_chain_batch for one ray, integrators.py:427-518 */
static void chain1(const OrScene *s, v3 O, v3 D, uint8_t *found, uint8_t *esc, double *pos, double *nrm,
                   int32_t *mat, double *thr, double *dir, double *tt) {
  v3 beta = V(1, 1, 1);
  *found = 0; *esc = 0; S3(pos, V(0, 0, 0)); S3(nrm, V(0, 0, 0)); *mat = -1;
  S3(thr, beta); S3(dir, D); *tt = 0.0;
  for (int it = 0; it < CHAIN_BOUND; ++it) {
    Isect h = trace1(s, O, D, TEPS, INFINITY);
    if (!h.hit) { *esc = 1; S3(thr, beta); S3(dir, D); return; }
    *tt = *tt + h.t;
    int ent = vdot(h.n, D) < 0.0;
    if (!s->mspec[h.mat]) {
      *found = 1; S3(pos, h.pos); S3(nrm, ent ? h.n : vneg(h.n)); *mat = h.mat; S3(thr, beta); S3(dir, D);
      return;
    }
    v3 nf = ent ? h.n : vneg(h.n);
    double ci = -vdot(nf, D);
    v3 alb = L3(s->malb + 3 * h.mat);
    v3 refl = vadd(D, vsc(2.0 * ci, nf)), nd = refl, fac;
    if (s->mkind[h.mat] == 2) {
      fac = V(schl(alb.x, ci), schl(alb.y, ci), schl(alb.z, ci));
    } else {
      double ior = s->mior[h.mat], eta = ent ? 1.0 / ior : ior;
      double c2 = 1.0 - ci * ci;
      double s2t = eta * eta * (c2 > 0.0 ? c2 : 0.0);
      int tir = s2t >= 1.0;
      double q = (ior - 1.0) / (ior + 1.0);
      double fr = schl(q * q, ci);
      double ct2 = 1.0 - s2t;
      double ct = sqrt(ct2 > 0.0 ? ct2 : 0.0);
      v3 refr = vadd(vsc(eta, D), vsc(eta * ci - ct, nf));
      if (!tir) nd = refr;
      double k = tir ? 1.0 : 1.0 - fr;
      fac = V(alb.x * k, alb.y * k, alb.z * k);
    }
    beta = vmul(beta, fac);
    O = vadd(h.pos, vsc(TEPS * (vdot(nd, nf) >= 0.0 ? 1.0 : -1.0), nf));
    D = vdivs(nd, vlen(nd));
    if (beta.x < THR_CUTOFF && beta.y < THR_CUTOFF && beta.z < THR_CUTOFF) return;
  }
}

void or_primary_chain(const OrScene *s, const double *O, const double *D, int64_t n, uint8_t *found,
                      uint8_t *escaped, double *pos, double *nrm, int32_t *mat, double *thr, double *dir,
                      double *t_total) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i)
    chain1(s, L3(O + 3 * i), L3(D + 3 * i), found + i, escaped + i, pos + 3 * i, nrm + 3 * i, mat + i,
           thr + 3 * i, dir + 3 * i, t_total + i);
}

/* Camera.ray_directions, scene.py:76-93 */
static v3 cam_dir(const OrCamera *c, double px, double py) {
  double w = c->width, h = c->height;
  double nx = (px / w * 2.0 - 1.0) * c->tan_half * (w / h);
  double ny = (1.0 - py / h * 2.0) * c->tan_half;
  v3 d = vadd(vadd(L3(c->forward), vsc(nx, L3(c->right))), vsc(ny, L3(c->up)));
  return vdivs(d, vlen(d));
}

int64_t or_gbuffer_direct(const OrScene *s, const OrCamera *cam, const OrCfg *cfg, int64_t p0, int64_t p1,
                          uint8_t *found, uint8_t *escaped, double *pos, double *nrm, int32_t *mat,
                          double *thr, double *dir, double *t_total, double *direct) {
  int spp = cfg->direct_spp;
  Smp sm = {cfg->sampler_kind, cfg->seed, (uint64_t)(spp > 1 ? spp : 1)};
  int64_t nf = 0;
  int W = cam->width, H = cam->height, tile = cfg->tile;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : nf)
  for (int64_t i = p0; i < p1; ++i) {
    int x = (int)(i % W), y = (int)(i / W);
    v3 o = L3(cam->position);
    chain1(s, o, cam_dir(cam, x + 0.5, y + 0.5), found + i, escaped + i, pos + 3 * i, nrm + 3 * i, mat + i,
           thr + 3 * i, dir + 3 * i, t_total + i);
    /* direct pass: per-tile wave chunks of the reference (cache.py:399-413) */
    int tx0 = (x / tile) * tile, ty0 = (y / tile) * tile;
    int tw = W - tx0 < tile ? W - tx0 : tile, th = H - ty0 < tile ? H - ty0 : tile;
    int chunk = 16384 / (tw * th);
    if (chunk < 1) chunk = 1;
    v3 acc = V(0, 0, 0);
    for (int s0 = 0; s0 < spp; s0 += chunk) {
      int ns = spp - s0 < chunk ? spp - s0 : chunk;
      v3 part = V(0, 0, 0);
      for (int sidx = s0; sidx < s0 + ns; ++sidx) {
        int c = 0;
        double jx = smp_get(&sm, (uint64_t)i, (uint64_t)sidx, 0), jy = smp_get(&sm, (uint64_t)i, (uint64_t)sidx, 1);
        v3 l = direct_li(s, &sm, o, cam_dir(cam, x + jx, y + jy), (uint64_t)i, (uint64_t)sidx, 0, &c);
        nf += c;
        part = sidx == s0 ? l : vadd(part, l);
      }
      acc = vadd(acc, part);
    }
    S3(direct + 3 * i, vdivs(acc, (double)spp));
  }
  return nf;
}

/* --------------------------------------------------------------- map stacks */
/* numpy pairwise summation (contiguous, n > 0) */
static double pw_sum(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

static const double LR = 0.2126, LG = 0.7152, LB = 0.0722; /* hemimap.py:26 */

static v3 texel_dir_local(int u, int v) {
  double phi = 2.0 * OPI * (u + 0.5) / RES;
  double th = (OPI / 2.0) * (v + 0.5) / RES;
  double st = sin(th);
  return V(st * cos(phi), st * sin(phi), cos(th));
}

/* render_input_stacks_batch, hemimap.py:229-281 */
int64_t or_render_stacks(const OrScene *s, const OrCfg *cfg, const double *pos, const double *nrm,
                         const uint64_t *keys, int64_t n, float *stacks, double *s_r, double *s_d,
                         double *frames) {
  Smp sm = {cfg->sampler_kind, cfg->seed, 1};
  int64_t nf = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : nf)
  for (int64_t p = 0; p < n; ++p) {
    double *rad = (double *)malloc(sizeof(double) * 3 * NT), *dist = (double *)malloc(sizeof(double) * NT);
    double *nl = (double *)malloc(sizeof(double) * 3 * NT), *lum = (double *)malloc(sizeof(double) * NT);
    v3 hp = L3(pos + 3 * p), hn = L3(nrm + 3 * p);
    Frm fr = frame_s(s, hn);
    S3(frames + 9 * p, fr.t); S3(frames + 9 * p + 3, fr.b); S3(frames + 9 * p + 6, fr.n);
    v3 o = vadd(hp, vsc(TEPS, hn));
    for (int tex = 0; tex < NT; ++tex) {
      v3 d = to_wld(&fr, texel_dir_local(tex % RES, tex / RES));
      Isect h = trace1(s, o, d, TEPS, INFINITY);
      dist[tex] = h.hit ? h.t : 0.0;
      int facing = vdot(h.n, d) > 0.0;
      v3 nfr = facing ? vneg(h.n) : h.n;
      v3 l = h.hit ? to_loc(&fr, nfr) : V(0, 0, 0);
      S3(nl + 3 * tex, l);
      int c = 0;
      v3 L = path_li(s, &sm, o, d, keys[p], (uint64_t)tex, cfg->max_path_depth, 1, cfg->rr_start, &c);
      nf += c;
      S3(rad + 3 * tex, L);
      lum[tex] = (L.x * LR + L.y * LG) + L.z * LB;
    }
    double sr = pw_sum(lum, NT) / NT + 1e-3;
    double mx = 0.0;
    for (int t = 0; t < NT; ++t) if (dist[t] > mx) mx = dist[t];
    double sd = mx > 0.0 ? mx : 1.0;
    float *o7 = stacks + p * 7 * NT;
    for (int t = 0; t < NT; ++t) {
      for (int c = 0; c < 3; ++c) o7[c * NT + t] = (float)(rad[3 * t + c] / sr);
      for (int c = 0; c < 3; ++c) o7[(3 + c) * NT + t] = (float)nl[3 * t + c];
      o7[6 * NT + t] = (float)(dist[t] / sd);
    }
    s_r[p] = sr;
    s_d[p] = sd;
    free(rad); free(dist); free(nl); free(lum);
  }
  return nf;
}

/* ------------------------------------------------------------------ shading */
static double fmod_py(double x, double y) {
  double m = fmod(x, y);
  if (m != 0.0) { if ((m < 0.0) != (y < 0.0)) m += y; }
  else m = copysign(0.0, y);
  return m;
}
static double sin_theta_v(int v) { return sin((OPI / 2.0) * (v + 0.5) / RES); }

/* build_map_distribution + shade_indirect, hemimap.py:156-197 and
 * integrators.py:564-614 */
void or_shade(const OrScene *s, const OrCfg *cfg, const float *pred, const double *s_r,
              const double *frames, const double *wo, const int32_t *mat, const uint64_t *keys,
              int64_t n, double *Lout) {
  Smp sm = {cfg->sampler_kind, cfg->seed, 1};
  const double omega0 = (2.0 * OPI / RES) * (OPI / (2.0 * RES));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t p = 0; p < n; ++p) {
    double prob[NT], ccdf[NT], rcdf[RES], rows[RES];
    const float *pd = pred + p * 3 * NT;
    double sc = s_r[p];
    for (int t = 0; t < NT; ++t) {
      double r = (double)pd[t] * sc, g = (double)pd[NT + t] * sc, b = (double)pd[2 * NT + t] * sc;
      prob[t] = ((r * LR + g * LG) + b * LB) * sin_theta_v(t / RES) + 1e-8;
    }
    double tot = pw_sum(prob, NT);
    for (int t = 0; t < NT; ++t) prob[t] = prob[t] / tot;
    for (int v = 0; v < RES; ++v) rows[v] = pw_sum(prob + RES * v, RES);
    for (int v = 0; v < RES; ++v) {
      rcdf[v] = v == 0 ? rows[0] : rcdf[v - 1] + rows[v];
      for (int u = 0; u < RES; ++u) {
        double c = prob[v * RES + u] / rows[v];
        ccdf[v * RES + u] = u == 0 ? c : ccdf[v * RES + u - 1] + c;
      }
      ccdf[v * RES + RES - 1] = 1.0;
    }
    rcdf[RES - 1] = 1.0;
    Frm fr = {L3(frames + 9 * p), L3(frames + 9 * p + 3), L3(frames + 9 * p + 6)};
    v3 wol = to_loc(&fr, L3(wo + 3 * p));
    int m = mat[p];
    int nmap = cfg->mis_samples / 2, nbs = cfg->mis_samples - nmap;
    v3 smap = V(0, 0, 0), sbs = V(0, 0, 0);
    for (int i = 0; i < nmap; ++i) {
      double u1 = smp_get(&sm, keys[p], (uint64_t)i, SHADE_BASE), u2 = smp_get(&sm, keys[p], (uint64_t)i, SHADE_BASE + 1);
      int v = 0;
      while (v < RES && rcdf[v] <= u1) ++v;
      if (v > RES - 1) v = RES - 1;
      int u = 0;
      for (int k = 0; k < RES; ++k) u += ccdf[v * RES + k] <= u2;
      if (u > RES - 1) u = RES - 1;
      int q = v * RES + u;
      double pdf = prob[q] / (omega0 * sin_theta_v(v));
      v3 rad = V((double)pd[q] * sc, (double)pd[NT + q] * sc, (double)pd[2 * NT + q] * sc);
      v3 li = to_loc(&fr, to_wld(&fr, texel_dir_local(u, v)));
      v3 f;
      double pb;
      bsdf_f(s, m, wol, li, &f, &pb);
      double ci = li.z > 0.0 ? li.z : 0.0;
      double k = (powh(pdf, pb) * ci) / pdf;
      v3 c = vmul(vmul(f, rad), V(k, k, k));
      smap = i == 0 ? c : vadd(smap, c);
    }
    for (int i = 0; i < nbs; ++i) {
      double u1 = smp_get(&sm, keys[p], (uint64_t)i, SHADE_BASE + 2), u2 = smp_get(&sm, keys[p], (uint64_t)i, SHADE_BASE + 3);
      BS b = bsdf_s(s, m, wol, u1, u2, 1);
      double z = b.li.z < -1.0 ? -1.0 : (b.li.z > 1.0 ? 1.0 : b.li.z);
      int valid = z >= 0.0;
      v3 rad = V(0, 0, 0);
      double pm = 0.0;
      if (valid) {
        double th = acos(z), ph = fmod_py(atan2(b.li.y, b.li.x), 2.0 * OPI);
        int64_t uu = (int64_t)(ph / (2.0 * OPI) * RES), vv = (int64_t)(th / (OPI / 2.0) * RES);
        int u = (int)(uu < RES - 1 ? uu : RES - 1), v = (int)(vv < RES - 1 ? vv : RES - 1);
        int q = v * RES + u;
        rad = V((double)pd[q] * sc, (double)pd[NT + q] * sc, (double)pd[2 * NT + q] * sc);
        pm = prob[q] / (omega0 * sin_theta_v(v));
      }
      double ci = b.li.z > 0.0 ? b.li.z : 0.0;
      double k = (powh(b.pdf, pm) * ci) / b.pdf;
      v3 c = vmul(vmul(b.val, rad), V(k, k, k));
      sbs = i == 0 ? c : vadd(sbs, c);
    }
    v3 total = vadd(vdivs(smap, (double)nmap), vdivs(sbs, (double)nbs));
    if (!vfinite(total)) total = V(0, 0, 0);
    S3(Lout + 3 * p, total);
  }
}

/* --------------------------------------------------------- interpolation */
/* _interpolate_layer + composite, cache.py:283-345, 463 (brute force over
 * entries in ascending index, the cKDTree/np.add.at order) */
void or_interp_composite(int32_t W, int32_t H, const uint8_t *found, const uint8_t *escaped,
                         const double *nrm, const double *thr, const double *env, const int32_t *epx,
                         const int32_t *epy, const double *en, const double *erad, int64_t m, int32_t r,
                         const double *direct, double *image) {
  int has_env = env[0] > 0 || env[1] > 0 || env[2] > 0;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < (int64_t)W * H; ++i) {
    int x = (int)(i % W), y = (int)(i / W);
    v3 lay = V(0, 0, 0), th = L3(thr + 3 * i);
    if (escaped[i] && has_env) lay = vmul(th, L3(env));
    if (found[i] && m > 0) {
      int64_t best = INT64_MAX;
      for (int64_t e = 0; e < m; ++e) {
        int64_t dx = epx[e] - x, dy = epy[e] - y, d2 = dx * dx + dy * dy;
        if (d2 < best) best = d2;
      }
      double d1 = sqrt((double)best);
      double reff = (double)r > 1.5 * d1 ? (double)r : 1.5 * d1;
      double R = 2.0 * reff, R2 = R * R;
      v3 num = V(0, 0, 0);
      double den = 0.0;
      v3 np_ = L3(nrm + 3 * i);
      for (int64_t e = 0; e < m; ++e) {
        double dx = (double)(epx[e] - x), dy = (double)(epy[e] - y);
        double d2 = dx * dx + dy * dy;
        if (!(d2 <= R2)) continue;
        double wp = 1.0 - sqrt(d2) / reff;
        if (wp < 0.0) wp = 0.0;
        double wn = vdot(L3(en + 3 * e), np_);
        if (wn < 0.0) wn = 0.0;
        double w = (wp * wn + wp) + 1e-4;
        num = vadd(num, vsc(w, L3(erad + 3 * e)));
        den += w;
      }
      if (den > 0.0) lay = vmul(th, vdivs(num, den));
    }
    v3 out = direct ? vadd(L3(direct + 3 * i), lay) : lay;
    S3(image + 3 * i, out);
  }
}

/* --------------------------------------------------------------- network */
/* cnn.py:39-215 restated in fp32 with direct loops */
typedef struct { float *w, *b, *sc, *sh; int cin, cout, ks, hw, act; } OLayer;
struct OrNet { int k; float slope; OLayer L[17]; };

typedef struct { const uint8_t *p; int64_t len, off; } Rd;
static int rd(Rd *r, void *d, int64_t n) {
  if (r->off + n > r->len) return 0;
  memcpy(d, r->p + r->off, (size_t)n);
  r->off += n;
  return 1;
}

typedef struct { char name[64]; uint32_t dims[4]; int rank; float *data; } OTensor;

static OTensor *find_t(OTensor *ts, int n, const char *name) {
  for (int i = 0; i < n; ++i) if (strcmp(ts[i].name, name) == 0) return &ts[i];
  return NULL;
}

OrNet *or_net_create(const uint8_t *drcw, int64_t len) {
  Rd r = {drcw, len, 0};
  char magic[4];
  uint32_t ver, slb, cnt;
  if (!rd(&r, magic, 4) || memcmp(magic, "DRCW", 4) || !rd(&r, &ver, 4) || !rd(&r, &slb, 4) || !rd(&r, &cnt, 4))
    return NULL;
  OTensor *ts = (OTensor *)calloc(cnt, sizeof(OTensor));
  for (uint32_t i = 0; i < cnt; ++i) {
    uint16_t nl;
    uint8_t rk;
    if (!rd(&r, &nl, 2) || nl >= 64 || !rd(&r, ts[i].name, nl) || !rd(&r, &rk, 1) || rk > 4) return NULL;
    ts[i].rank = rk;
    if (!rd(&r, ts[i].dims, 4 * rk)) return NULL;
    int64_t c = 1;
    for (int k = 0; k < rk; ++k) c *= ts[i].dims[k];
    ts[i].data = (float *)malloc(sizeof(float) * (size_t)c);
    if (!rd(&r, ts[i].data, 4 * c)) return NULL;
  }
  OrNet *net = (OrNet *)calloc(1, sizeof(OrNet));
  memcpy(&net->slope, &slb, 4);
  OTensor *w0 = find_t(ts, (int)cnt, "enc1.conv1.weight");
  int k = net->k = (int)w0->dims[0];
  struct { const char *n, *bn; int cin, cout, hw, ks, de; } sp[17] = {
      {"enc1.conv1", "enc1.bn1", 7, k, 32, 3, 0}, {"enc1.conv2", "enc1.bn2", k, k, 32, 3, 0},
      {"enc2.conv1", "enc2.bn1", k, 2 * k, 16, 3, 0}, {"enc2.conv2", "enc2.bn2", 2 * k, 2 * k, 16, 3, 0},
      {"enc3.conv1", "enc3.bn1", 2 * k, 4 * k, 8, 3, 0}, {"enc3.conv2", "enc3.bn2", 4 * k, 4 * k, 8, 3, 0},
      {"bott.conv1", "bott.bn1", 4 * k, 8 * k, 4, 3, 0}, {"bott.conv2", "bott.bn2", 8 * k, 8 * k, 4, 3, 0},
      {"dec3.deconv1", "dec3.bn1", 12 * k, 4 * k, 8, 3, 1}, {"dec3.deconv2", "dec3.bn2", 4 * k, 4 * k, 8, 3, 1},
      {"dec2.deconv1", "dec2.bn1", 6 * k, 2 * k, 16, 3, 1}, {"dec2.deconv2", "dec2.bn2", 2 * k, 2 * k, 16, 3, 1},
      {"dec1.deconv1", "dec1.bn1", 3 * k, k, 32, 3, 1}, {"dec1.deconv2", "dec1.bn2", k, k, 32, 3, 1},
      {"head.deconv1", "head.bn1", k, k / 2, 32, 3, 1}, {"head.deconv2", "head.bn2", k / 2, k / 4, 32, 3, 1},
      {"head.conv_out", "", k / 4, 3, 32, 1, 0}};
  char buf[96];
  for (int l = 0; l < 17; ++l) {
    OLayer *L = &net->L[l];
    L->cin = sp[l].cin; L->cout = sp[l].cout; L->ks = sp[l].ks; L->hw = sp[l].hw; L->act = sp[l].bn[0] != 0;
    snprintf(buf, sizeof buf, "%s.weight", sp[l].n);
    OTensor *W = find_t(ts, (int)cnt, buf);
    snprintf(buf, sizeof buf, "%s.bias", sp[l].n);
    OTensor *B = find_t(ts, (int)cnt, buf);
    if (!W || !B) return NULL;
    int ks = L->ks;
    size_t nw = (size_t)L->cout * L->cin * ks * ks;
    L->w = (float *)malloc(sizeof(float) * nw);
    /* deconv2d == conv with flipped kernel and swapped channel axes (cnn.py:124-131) */
    for (int co = 0; co < L->cout; ++co)
      for (int ci = 0; ci < L->cin; ++ci)
        for (int a = 0; a < ks; ++a)
          for (int b = 0; b < ks; ++b)
            L->w[((size_t)(co * L->cin + ci) * ks + a) * ks + b] =
                sp[l].de ? W->data[((size_t)(ci * L->cout + co) * 3 + (2 - a)) * 3 + (2 - b)]
                         : W->data[((size_t)(co * L->cin + ci) * ks + a) * ks + b];
    L->b = (float *)malloc(sizeof(float) * L->cout);
    memcpy(L->b, B->data, sizeof(float) * L->cout);
    L->sc = (float *)malloc(sizeof(float) * L->cout);
    L->sh = (float *)malloc(sizeof(float) * L->cout);
    for (int c = 0; c < L->cout; ++c) { L->sc[c] = 1.f; L->sh[c] = 0.f; }
    if (L->act) {
      const char *fld[4] = {"gamma", "beta", "running_mean", "running_var"};
      OTensor *T[4];
      for (int q = 0; q < 4; ++q) { snprintf(buf, sizeof buf, "%s.%s", sp[l].bn, fld[q]); T[q] = find_t(ts, (int)cnt, buf); if (!T[q]) return NULL; }
      /* batchnorm_infer, cnn.py:134-141 (float32 arithmetic) */
      for (int c = 0; c < L->cout; ++c) {
        float var = T[3]->data[c] + 1e-5f;
        float s = T[0]->data[c] / sqrtf(var);
        L->sc[c] = s;
        L->sh[c] = T[1]->data[c] - T[2]->data[c] * s;
      }
    }
  }
  for (uint32_t i = 0; i < cnt; ++i) free(ts[i].data);
  free(ts);
  return net;
}

void or_net_destroy(OrNet *net) {
  if (!net) return;
  for (int l = 0; l < 17; ++l) { free(net->L[l].w); free(net->L[l].b); free(net->L[l].sc); free(net->L[l].sh); }
  free(net);
}

/* conv2d + bias + (BN + LeakyReLU | ReLU) on one map; out may point into a
 * wider concat buffer (channel offset handled by the caller) */
static void oconv(const OLayer *L, const float *in, float *out, float slope) {
  int hw = L->hw, np = hw * hw, ks = L->ks, R = ks / 2;
  float *acc = (float *)malloc(sizeof(float) * np);
  for (int co = 0; co < L->cout; ++co) {
    for (int q = 0; q < np; ++q) acc[q] = 0.f;
    for (int ci = 0; ci < L->cin; ++ci) {
      const float *ip = in + (size_t)ci * np;
      for (int a = 0; a < ks; ++a)
        for (int b = 0; b < ks; ++b) {
          float wv = L->w[((size_t)(co * L->cin + ci) * ks + a) * ks + b];
          for (int y = 0; y < hw; ++y) {
            int yy = y + a - R;
            if (yy < 0 || yy >= hw) continue;
            for (int x = 0; x < hw; ++x) {
              int xx = x + b - R;
              if (xx < 0 || xx >= hw) continue;
              acc[y * hw + x] += wv * ip[yy * hw + xx];
            }
          }
        }
    }
    float *op = out + (size_t)co * np;
    for (int q = 0; q < np; ++q) {
      float v = acc[q] + L->b[co];
      if (L->act) {
        v = v * L->sc[co] + L->sh[co];
        v = v >= 0.f ? v : slope * v;
      } else {
        v = v > 0.f ? v : 0.f;
      }
      op[q] = v;
    }
  }
  free(acc);
}

static void opool(const float *in, int c, int hw, float *out) {
  int ho = hw / 2;
  for (int ch = 0; ch < c; ++ch)
    for (int y = 0; y < ho; ++y)
      for (int x = 0; x < ho; ++x) {
        const float *p = in + ((size_t)ch * hw + 2 * y) * hw + 2 * x;
        float m = p[0];
        if (p[1] > m) m = p[1];
        if (p[hw] > m) m = p[hw];
        if (p[hw + 1] > m) m = p[hw + 1];
        out[((size_t)ch * ho + y) * ho + x] = m;
      }
}

/* upsample_bilinear2x2, cnn.py:159-174 */
static void oup(const float *in, int c, int hw, float *out) {
  int ho = 2 * hw;
  int i0[64], i1[64];
  float fr[64];
  for (int o = 0; o < ho; ++o) {
    double src = (o + 0.5) / 2.0 - 0.5;
    if (src < 0.0) src = 0.0;
    int a = (int)src;
    i0[o] = a < hw - 1 ? a : hw - 1;
    i1[o] = i0[o] + 1 < hw - 1 ? i0[o] + 1 : hw - 1;
    fr[o] = (float)(src - i0[o]);
  }
  for (int ch = 0; ch < c; ++ch) {
    const float *p = in + (size_t)ch * hw * hw;
    for (int y = 0; y < ho; ++y)
      for (int x = 0; x < ho; ++x) {
        float omr = 1.f - fr[y], omc = 1.f - fr[x];
        float t0 = p[i0[y] * hw + i0[x]] * omr + p[i1[y] * hw + i0[x]] * fr[y];
        float t1 = p[i0[y] * hw + i1[x]] * omr + p[i1[y] * hw + i1[x]] * fr[y];
        out[((size_t)ch * ho + y) * ho + x] = t0 * omc + t1 * fr[x];
      }
  }
}

void or_net_forward(const OrNet *net, const float *x, float *y, int64_t n) {
  int k = net->k;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < n; ++i) {
    const OLayer *L = net->L;
    float sl = net->slope;
    float *c1 = (float *)malloc(sizeof(float) * 3 * k * 1024), *t32 = (float *)malloc(sizeof(float) * k * 1024);
    float *p1 = (float *)malloc(sizeof(float) * k * 256), *c2 = (float *)malloc(sizeof(float) * 6 * k * 256);
    float *t16 = (float *)malloc(sizeof(float) * 2 * k * 256), *p2 = (float *)malloc(sizeof(float) * 2 * k * 64);
    float *c3 = (float *)malloc(sizeof(float) * 12 * k * 64), *t8 = (float *)malloc(sizeof(float) * 4 * k * 64);
    float *p3 = (float *)malloc(sizeof(float) * 4 * k * 16), *b0 = (float *)malloc(sizeof(float) * 8 * k * 16);
    float *b1 = (float *)malloc(sizeof(float) * 8 * k * 16), *h1 = (float *)malloc(sizeof(float) * k * 1024);
    const float *xi = x + i * 7 * 1024;
    oconv(&L[0], xi, t32, sl);
    oconv(&L[1], t32, c1 + 2 * k * 1024, sl);             /* s1 -> concat slot */
    opool(c1 + 2 * k * 1024, k, 32, p1);
    oconv(&L[2], p1, t16, sl);
    oconv(&L[3], t16, c2 + 4 * k * 256, sl);              /* s2 */
    opool(c2 + 4 * k * 256, 2 * k, 16, p2);
    oconv(&L[4], p2, t8, sl);
    oconv(&L[5], t8, c3 + 8 * k * 64, sl);                /* s3 */
    opool(c3 + 8 * k * 64, 4 * k, 8, p3);
    oconv(&L[6], p3, b0, sl);
    oconv(&L[7], b0, b1, sl);
    oup(b1, 8 * k, 4, c3);
    oconv(&L[8], c3, t8, sl);
    free(b0);
    b0 = (float *)malloc(sizeof(float) * 4 * k * 64);
    oconv(&L[9], t8, b0, sl);
    oup(b0, 4 * k, 8, c2);
    oconv(&L[10], c2, t16, sl);
    float *d16 = (float *)malloc(sizeof(float) * 2 * k * 256);
    oconv(&L[11], t16, d16, sl);
    oup(d16, 2 * k, 16, c1);
    oconv(&L[12], c1, t32, sl);
    float *d32 = (float *)malloc(sizeof(float) * k * 1024);
    oconv(&L[13], t32, d32, sl);
    oconv(&L[14], d32, h1, sl);
    oconv(&L[15], h1, t32, sl);  /* k/4 @32 fits in t32 */
    oconv(&L[16], t32, y + i * 3 * 1024, sl);
    free(c1); free(t32); free(p1); free(c2); free(t16); free(p2); free(c3); free(t8); free(p3);
    free(b0); free(b1); free(h1); free(d16); free(d32);
  }
}
