/*
 * drc_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, scalar, fp64 restatement of the reference's rendering path
 * (/root/reference/pkg/src/drc, numpy) used as the CPU checker for libdrcb
 * and as the CPU baseline ("port") in bench.py. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. It is pinned against golden vectors produced by the
 * unmodified reference (tests/golden/make_golden.py; tests/test_oracle.py).
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef DRC_ORACLE_H
#define DRC_ORACLE_H
#include <stdint.h>

typedef struct OrSceneDesc {
  int32_t n_spheres, n_quads, n_tris, n_materials, n_point_lights;
  const double *sph_center, *sph_radius;
  const int32_t *sph_mat;
  const double *quad_corner, *quad_eu, *quad_ev;
  const int32_t *quad_mat;
  const double *tri_v0, *tri_v1, *tri_v2;
  const int32_t *tri_mat;
  const int32_t *mat_kind;
  const double *mat_albedo, *mat_exponent, *mat_ior, *mat_emission;
  const double *point_pos, *point_intensity;
  double global_up[3], rotated_up[3], environment[3];
} OrSceneDesc;

typedef struct OrCamera {
  double position[3], forward[3], right[3], up[3];
  double tan_half;
  int32_t width, height;
} OrCamera;

typedef struct OrCfg {
  int32_t direct_spp, max_path_depth, mis_samples, rr_start, sampler_kind, tile;
  uint64_t seed;
} OrCfg;

typedef struct OrScene OrScene;
typedef struct OrNet OrNet;

OrScene *or_scene_create(const OrSceneDesc *d);
void or_scene_destroy(OrScene *s);

void or_set_threads(int n);

/* geometry.py:217-329 */
void or_intersect(const OrScene *s, const double *O, const double *D, int64_t n,
                  const double *tmin, const double *tmax, int record, uint8_t *hit,
                  double *t, int64_t *prim, int32_t *mat, double *pos, double *nrm);
/* integrators.py:427-518; out arrays (n,..) */
void or_primary_chain(const OrScene *s, const double *O, const double *D, int64_t n,
                      uint8_t *found, uint8_t *escaped, double *pos, double *nrm,
                      int32_t *mat, double *thr, double *dir, double *t_total);
/* integrators.py:305-424; sampler = (cfg.sampler_kind, cfg.seed, cfg.direct_spp) */
int64_t or_li_direct(const OrScene *s, const OrCfg *cfg, const double *O, const double *D,
                     const uint64_t *pix, const uint64_t *smp, int64_t n, int include_bg,
                     double *L);
/* integrators.py:175-302 */
int64_t or_trace_radiance(const OrScene *s, const OrCfg *cfg, const double *O,
                          const double *D, const uint64_t *pix, const uint64_t *smp,
                          int64_t n, int max_depth, int skip_first, int rr_start, double *L);
/* cache.py:157-176 + 393-423 for one camera: geo buffers + direct image.
 * Only pixels [p0, p1) (flat index) are computed (bounded CPU samples). */
int64_t or_gbuffer_direct(const OrScene *s, const OrCamera *cam, const OrCfg *cfg, int64_t p0,
                          int64_t p1, uint8_t *found, uint8_t *escaped, double *pos,
                          double *nrm, int32_t *mat, double *thr, double *dir,
                          double *t_total, double *direct);
/* hemimap.py:229-281: stacks (n,7,32,32) f32, s_r, s_d, frames (n,9) */
int64_t or_render_stacks(const OrScene *s, const OrCfg *cfg, const double *pos,
                         const double *nrm, const uint64_t *keys, int64_t n, float *stacks,
                         double *s_r, double *s_d, double *frames);
/* integrators.py:564-614 */
void or_shade(const OrScene *s, const OrCfg *cfg, const float *pred, const double *s_r,
              const double *frames, const double *wo, const int32_t *mat,
              const uint64_t *keys, int64_t n, double *L);
/* cache.py:283-345 + 463 */
void or_interp_composite(int32_t W, int32_t H, const uint8_t *found, const uint8_t *escaped,
                         const double *nrm, const double *thr, const double *env,
                         const int32_t *epx, const int32_t *epy, const double *en,
                         const double *erad, int64_t m, int32_t r, const double *direct,
                         double *image);

/* network: cnn.py. Weights given in DRCW byte form. */
OrNet *or_net_create(const uint8_t *drcw, int64_t len);
void or_net_destroy(OrNet *net);
/* cnn.py:193-215, x (n,7,32,32) -> y (n,3,32,32) */
void or_net_forward(const OrNet *net, const float *x, float *y, int64_t n);

#endif
