/*
 * drcb.h — C ABI of libdrcb.so, the B200 (sm_100a) implementation of the
 * deep-radiance-cache hot path of arXiv 1910.02480.
 *
 * Every entry point replaces one Python surface of the reference
 * (/root/reference/pkg); the reference interface is cited beside each one.
 * Conventions
 *   - plain C types only; no torch, no C++ across the ABI;
 *   - all array arguments are DEVICE pointers owned by the caller unless
 *     the comment says "host";
 *   - every call is asynchronous on the `stream` argument (a cudaStream_t
 *     passed as void*; NULL = legacy default stream);
 *   - return 0 on success or a DRCB_E* status; drcb_last_error() returns a
 *     thread-local message. Status codes mirror drc/errors.py:4-31.
 *   - `precision` selects the arithmetic of the ray/path kernels: 64 = the
 *     fp64 parity build (matches the reference's float64 numpy), 32 = fp32.
 */
#ifndef DRCB_H
#define DRCB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (drc/errors.py:4-31 -> 1..4; CUDA/NCCL failures 10/11) */
#define DRCB_OK 0
#define DRCB_ECONFIG 1      /* ConfigError      */
#define DRCB_ECONTRACT 2    /* ContractError    */
#define DRCB_EFORMAT 3      /* FormatError      */
#define DRCB_EVALIDATION 4  /* SceneValidationError */
#define DRCB_ECUDA 10
#define DRCB_ENCCL 11

/* material kinds (drc/bsdf.py:24) */
#define DRCB_DIFFUSE 0
#define DRCB_GLOSSY 1
#define DRCB_MIRROR 2
#define DRCB_TRANSMISSION 3

typedef struct DrcbScene DrcbScene;
typedef struct DrcbNet DrcbNet;
typedef struct DrcbTrainer DrcbTrainer;

/* Scene geometry + materials + lights, all HOST pointers, copied at create.
 * Prim ids are global over [spheres | quads | triangles] in shape order
 * (drc/geometry.py:48-119). */
typedef struct DrcbSceneDesc {
  int32_t n_spheres, n_quads, n_tris, n_materials, n_point_lights;
  const double *sph_center;  /* (n_spheres,3) */
  const double *sph_radius;  /* (n_spheres,)  */
  const int32_t *sph_mat;
  const double *quad_corner, *quad_eu, *quad_ev; /* (n_quads,3) each */
  const int32_t *quad_mat;
  const double *tri_v0, *tri_v1, *tri_v2;        /* (n_tris,3) each  */
  const int32_t *tri_mat;
  const int32_t *mat_kind;      /* (n_materials,) DRCB_DIFFUSE..       */
  const double *mat_albedo;     /* (n_materials,3)                      */
  const double *mat_exponent;   /* Phong exponent 2/r^2-2, 0 otherwise  */
  const double *mat_ior;        /* 1 unless transmission                */
  const double *mat_emission;   /* (n_materials,3)                      */
  const double *point_pos, *point_intensity;    /* (n_point_lights,3)  */
  double global_up[3];
  double rotated_up[3];         /* bsdf._rotated_up(global_up), host-computed */
  double environment[3];
} DrcbSceneDesc;

/* Pinhole camera (drc/scene.py:70-93); the basis is precomputed on the
 * host exactly as Camera.basis() does. */
typedef struct DrcbCamera {
  double position[3], forward[3], right[3], up[3];
  double tan_half;   /* tan(radians(fov)/2) */
  int32_t width, height;
} DrcbCamera;

/* RenderConfig subset used on the device (drc/integrators.py:41-72). */
typedef struct DrcbRenderCfg {
  int32_t direct_spp;
  int32_t max_path_depth;
  int32_t mis_samples;
  int32_t rr_start;
  int32_t sampler_kind;   /* 0 independent, 1 stratified (drc/sampler.py:46-78) */
  int32_t precision;      /* 32 or 64 */
  int32_t tile;           /* RenderConfig.tile: only fixes the direct-pass
                             summation grouping (cache.py:399-413) */
  int32_t include_background; /* direct pass: add env seen by camera chains
                                 (render(mode="direct") = 1; render_drc = 0) */
  int32_t map_spp;        /* sampler spp of map paths (render_drc: 1; dataset
                             reference mode: ref_spp, dataset.py:92) */
  int32_t reserved;
  uint64_t seed;
} DrcbRenderCfg;

/* Primary-chain G-buffer, one row per pixel (drc/integrators.py:427-518).
 * Real-typed fields use `precision`. */
typedef struct DrcbGBuffer {
  uint8_t *found, *escaped;
  void *position, *normal, *throughput, *direction, *t_total; /* (n,3)/(n,) */
  int32_t *mat;
} DrcbGBuffer;

/* ---- scene ------------------------------------------------------------ */
/* Geometry(scene) + BVH (drc/geometry.py:48-185, 335-460). */
int drcb_scene_create(const DrcbSceneDesc *desc, DrcbScene **out);
void drcb_scene_destroy(DrcbScene *scene);
/* host out[0..7]: n_prims, n_nodes, n_leaves, max_depth, n_lights, bytes */
int drcb_scene_stats(const DrcbScene *scene, int64_t *out8);

/* ---- stage kernels ---------------------------------------------------- */
/* intersect_batch / occluded_batch (drc/geometry.py:217-329).
 * O, D: (n,3) Real; tmin/tmax: (n,) Real or NULL (T_EPS / +inf).
 * record=0 fills hit/t/prim only.
 * precision DRCB_PREC_MIXED: the fp32 build's traversal of fp64 rays (every
 * buffer fp64), candidates whose fp32 decision lies within its rounding bound
 * re-tested in fp64 against the fp64 ray — the G-buffer's primary casts. */
#define DRCB_PREC_MIXED 3264
int drcb_intersect(const DrcbScene *scene, int32_t precision, const void *O,
                   const void *D, int64_t n, const void *tmin, const void *tmax,
                   int32_t record, uint8_t *hit, void *t, int64_t *prim,
                   int32_t *mat, void *pos, void *nrm, void *stream);

/* primary_chain_batch (drc/integrators.py:427-518). */
int drcb_primary_chain(const DrcbScene *scene, int32_t precision,
                       const void *O, const void *D, int64_t n,
                       const DrcbGBuffer *out, void *stream);

/* li_direct_batch (drc/integrators.py:305-424). keys: (n,) uint64.
 * nonfinite: device int64 counter (may be NULL). */
int drcb_li_direct(const DrcbScene *scene, const DrcbRenderCfg *cfg,
                   const void *O, const void *D, const uint64_t *pix,
                   const uint64_t *smp, int64_t n, int32_t include_background,
                   void *L, int64_t *nonfinite, void *stream);

/* trace_radiance_batch (drc/integrators.py:175-302). */
int drcb_trace_radiance(const DrcbScene *scene, const DrcbRenderCfg *cfg,
                        const void *O, const void *D, const uint64_t *pix,
                        const uint64_t *smp, int64_t n, int32_t max_depth,
                        int32_t skip_first_emission, int32_t rr_start,
                        void *L, int64_t *nonfinite, void *stream);

/* DrcState geometry buffers + the direct pass, fused
 * (drc/cache.py:157-176 + 393-423): unjittered centre chains into `gb`,
 * direct_spp jittered li_direct samples averaged into direct (H*W,3) Real. */
int drcb_gbuffer_direct(const DrcbScene *scene, const DrcbCamera *cam,
                        const DrcbRenderCfg *cfg, const DrcbGBuffer *gb,
                        void *direct, int64_t *nonfinite, void *stream);

/* render_input_stacks_batch (drc/hemimap.py:229-281) for n cache points.
 * pos/nrm: (n,3) Real front-facing hit data; keys (n,) uint64.
 * Outputs: stacks (n,7,32,32) float32 NCHW (InputStack.as_tensor order),
 * s_r, s_d: (n,) Real; frames (n,9) Real (t,b,n of build_frame). */
int drcb_render_stacks(const DrcbScene *scene, const DrcbRenderCfg *cfg,
                       const void *pos, const void *nrm, const uint64_t *keys,
                       int64_t n, float *stacks, void *s_r, void *s_d,
                       void *frames, int64_t *nonfinite, void *stream);

/* shade_indirect (drc/integrators.py:564-614) over n points.
 * pred: (n,3,32,32) float32 network output (normalised); frames (n,9);
 * wo (n,3) = -direction; mat (n,) int32; out L (n,3) Real. */
int drcb_shade(const DrcbScene *scene, const DrcbRenderCfg *cfg,
               const float *pred, const void *s_r, const void *frames,
               const void *wo, const int32_t *mat, const uint64_t *keys,
               int64_t n, void *L, void *stream);

/* _interpolate_layer + composite (drc/cache.py:283-345, 463).
 * Entries: e_px,e_py (m,) int32, e_normal,e_rad (m,3) Real.
 * image (H*W,3) Real = direct + layer (direct may be NULL -> layer only). */
int drcb_interp_composite(const DrcbScene *scene, int32_t precision,
                          int32_t width, int32_t height, const DrcbGBuffer *gb,
                          const int32_t *e_px, const int32_t *e_py,
                          const void *e_normal, const void *e_rad, int64_t m,
                          int32_t r, const void *direct, void *image,
                          void *stream);

/* Whole frame (drc/cache.py:377-470): gbuffer+direct, then the planned
 * cache points (host arrays px,py,keys in budget order, n_points), stacks,
 * network, shade, compaction, interpolation with final pass spacing r,
 * composite. image: (H*W,3) Real device. telemetry (host, 10 x int64, or
 * NULL): entries, fallback_pixels(=0), nonfinite, n_points, then stage times
 * in microseconds from CUDA events on `stream`: gbuffer+direct, maps (paths
 * + stacks), network, shade+interp, and the split of the last one: shade +
 * entry compaction, interpolation + composite. */
int drcb_render_drc(const DrcbScene *scene, const DrcbNet *net,
                    const DrcbCamera *cam, const DrcbRenderCfg *cfg,
                    const int32_t *px_host, const int32_t *py_host,
                    const uint64_t *keys_host, int64_t n_points, int32_t r_final,
                    int32_t net_mode, void *image, int64_t *telemetry_host,
                    void *stream);

/* The frame's entry pool (DrcState.entries, drc/cache.py:183-201): device
 * buffers with room for n_points entries; the first telemetry[0] are valid,
 * in the reference's append order. Real arrays use cfg->precision. */
typedef struct DrcbEntries {
  int32_t *px, *py;
  void *position, *normal, *radiance, *throughput; /* (n,3) each */
} DrcbEntries;

/* drcb_render_drc that also copies the entry pool out (the `--cache-out`
 * DRCC dump of cli.py:130-132 and DrcState.entries()). */
int drcb_render_drc_entries(const DrcbScene *scene, const DrcbNet *net,
                            const DrcbCamera *cam, const DrcbRenderCfg *cfg,
                            const int32_t *px_host, const int32_t *py_host,
                            const uint64_t *keys_host, int64_t n_points, int32_t r_final,
                            int32_t net_mode, void *image, int64_t *telemetry_host,
                            const DrcbEntries *entries, void *stream);

/* ---- progressive frames: the control plane of render_drc
 * (drc/cache.py:426-469). begin renders the G-buffer and direct pass and
 * reserves an entry pool for max_points cache points; add_points evaluates
 * a batch of cache points (host arrays in budget order: stacks, network,
 * shade) and appends the live ones to the pool in order; composite writes
 * image = direct + the interpolation of the entries so far at pass spacing
 * r (a pass end, a snapshot, or the interrupted frame); info synchronises
 * and returns {entries, nonfinite, points evaluated, max_points}. All
 * asynchronous on `stream` except info. */
typedef struct DrcbFrame DrcbFrame;
int drcb_frame_begin(const DrcbScene *scene, const DrcbNet *net, const DrcbCamera *cam,
                     const DrcbRenderCfg *cfg, int32_t net_mode, int64_t max_points,
                     DrcbFrame **out, void *stream);
int drcb_frame_add_points(DrcbFrame *frame, const int32_t *px_host, const int32_t *py_host,
                          const uint64_t *keys_host, int64_t n, void *stream);
int drcb_frame_composite(DrcbFrame *frame, int32_t r, void *image, void *stream);
int drcb_frame_info(DrcbFrame *frame, int64_t *out4, void *stream);
int drcb_frame_entries(DrcbFrame *frame, const DrcbEntries *out, void *stream);
int drcb_frame_end(DrcbFrame *frame, void *stream);

/* render(mode="pt") (drc/integrators.py:678-722): spp = cfg->direct_spp
 * jittered paths per pixel (max_path_depth, rr_start), image (H*W,3) Real. */
int drcb_render_pt(const DrcbScene *scene, const DrcbCamera *cam, const DrcbRenderCfg *cfg,
                   void *image, int64_t *nonfinite, void *stream);

/* _reference_map (drc/dataset.py:107-127): ground-truth radiance map of one
 * cache point (pos/nrm (3,) Real device, front-facing), ref_spp paths per
 * texel with the cfg sampler; out (32*32,3) Real, texel order v*32+u. */
int drcb_reference_map(const DrcbScene *scene, const DrcbRenderCfg *cfg, const void *pos,
                       const void *nrm, uint64_t key, int32_t ref_spp, void *out,
                       int64_t *nonfinite, void *stream);

/* ---- network ---------------------------------------------------------- */
/* DRCW container parse + validation (drc/cnn.py:221-281): host bytes. */
int drcb_net_create(const void *drcw, size_t len, DrcbNet **out);
void drcb_net_destroy(DrcbNet *net);
/* host out: k, n_params, version, slope bits */
int drcb_net_info(const DrcbNet *net, int64_t *out4);
/* forward (drc/cnn.py:193-215; trainer model.py:80-88 eval mode):
 * x (n,7,32,32) f32 -> y (n,3,32,32) f32.
 * mode: 0 fp32 SIMT (exact), 1 tf32 tcgen05, 2 bf16 tcgen05, 3 fp16 tcgen05
 * (16-bit operands with a 10-bit mantissa at the bf16 tensor rate; fp32
 * accumulation and epilogue in every tensor-core mode). */
#define DRCB_NET_FP32 0
#define DRCB_NET_TF32 1
#define DRCB_NET_BF16 2
#define DRCB_NET_FP16 3
int drcb_net_forward(const DrcbNet *net, const float *x, float *y, int64_t n,
                     int32_t mode, void *stream);

/* single tensor-core conv layer with an identity epilogue, HOST arrays
 * (unit-test harness for the implicit-GEMM kernel): x (n,hw,hw,cin) NHWC,
 * w (cout,cin,3,3) conv form, y (n,hw,hw,cout). */
int drcb_debug_conv(int32_t mode, int32_t cin, int32_t cout, int32_t hw, int64_t n,
                    const float *x, const float *w, float *y);

/* weight gradient of one 3x3 layer on the tensor cores (the training step's
 * wgrad), HOST arrays (unit-test harness): x (n,hw,hw,cin) NHWC, dz
 * (n,hw,hw,cout) NHWC, both rounded to bf16; dw (cout,cin,3,3) fp32 with
 * dw[co][ci][ky][kx] = sum_p dz[p][co] * x[p + (ky-1, kx-1)][ci]. */
int drcb_debug_wgrad(int32_t cin, int32_t cout, int32_t hw, int64_t n, const float *x,
                     const float *dz, float *dw);

/* traversal counters for roofline accounting: buf = device u64[12]
 * {inner nodes visited, primitives tested, casts, max nodes, max prims,
 * prims-tested histogram [5], sum of converged lanes at cast entry, any-hit
 * casts}, accumulated by every cast until disarmed with NULL (adds a few
 * atomics per cast when armed). */
int drcb_trav_stats(unsigned long long *buf);

/* number of kernels this library has launched so far (process-wide) */
int64_t drcb_kernel_launches(void);

/* Profiling hook: streams an L2-resident buffer `iters` times through L2 ->
 * SM loads on `stream` (time it with events): the measured L2 read peak the
 * ray-casting stages are reported against. `sink`: one device word. */
int drcb_l2_read_probe(const void *buf, int64_t bytes, int32_t iters,
                       unsigned long long *sink, void *stream);

/* ---- trainer input pipeline (trainer/src/drc_trainer/data.py:77-121) -- */
/* numpy cos/sin of 2*pi*shift/32 for shift = 0, 8, 16, 24 (host-computed so
 * the float64 normal re-expression matches _rotate_normals_xy bit for bit) */
typedef struct DrcbAugmentTrig {
  double cos_a[4], sin_a[4];
} DrcbAugmentTrig;

/* Gather n examples from a resident base set (x_base (N,7,32,32), y_base
 * (N,3,32,32) fp32 device) by base[i] and apply variant[i] (NULL = 0):
 * shift = 8*(v>>1) columns (np.roll by -shift), flip = v&1, normals
 * re-expressed (transform_example, data.py:86-100); ablate bit 0 = normals,
 * bit 1 = distance (ablate, data.py:106-117). augment() order is
 * v = 2*shift_index + flip (data.py:103-104). */
int drcb_augment_gather(const float *x_base, const float *y_base, const int64_t *base,
                        const int32_t *variant, int64_t n, const DrcbAugmentTrig *trig,
                        int32_t ablate, float *x_out, float *y_out, void *stream);

/* ---- training step (trainer/src/drc_trainer/train.py:97-103) ---------- */
/* MapAutoencoder in train mode (batch-statistics BN, momentum 0.1), L1 loss,
 * Adam(lr, betas, eps) with fp32 master weights, from DRCW bytes (host). */
int drcb_trainer_create(const void *drcw, size_t len, float lr, float beta1, float beta2,
                        float eps, DrcbTrainer **out);
void drcb_trainer_destroy(DrcbTrainer *t);
/* host out: k, n_params, n_running, steps taken */
int drcb_trainer_info(const DrcbTrainer *t, int64_t *out4);
/* device pointers of the flat fp32 parameter / gradient / running-stat
 * buffers, torch named_parameters() order (for all-reduce and inspection) */
int drcb_trainer_buffers(const DrcbTrainer *t, void **params, void **grads, void **running);
/* forward + loss + backward into the gradient buffer; x (n,7,32,32),
 * y (n,3,32,32) device fp32; apply_adam=1 also takes the optimiser step.
 * loss_host (optional) receives the mean L1 loss (synchronises). */
/* conv engine: 0 = fp32 CUDA cores (the parity engine, default), 2 = bf16
 * tensor cores (forward + dgrad on the tcgen05 implicit-GEMM conv kernels,
 * weight gradient as one bf16 GEMM over all pixels; fp32 master weights,
 * batch norm, activations and Adam). Env DRCB_TRAIN_CHECK=1 makes every bf16
 * step compare each layer's dgrad/wgrad with the fp32 kernels (fails > 2e-2). */
int drcb_trainer_set_mode(DrcbTrainer *t, int32_t mode);
int drcb_trainer_step(DrcbTrainer *t, const float *x, const float *y, int64_t n,
                      double *loss_host, int32_t apply_adam, void *stream);
/* Adam on the gradient buffer scaled by grad_scale (1/world after an
 * all-reduce sum across data-parallel ranks). */
int drcb_trainer_apply(DrcbTrainer *t, float grad_scale, void *stream);
/* Data-parallel communicator (NULL = single process). With a communicator
 * the step uses SyncBN (batch statistics all-reduced over NVLink/NVSwitch)
 * and all-reduces the gradient buffer; Adam averages by 1/world. */
int drcb_trainer_set_comm(DrcbTrainer *t, void *nccl_comm, int32_t world);
/* test hook (tensor-core trainer): the bf16 pre-BN conv output Z of one of
 * the 16 3x3 layers from the last step, device NHWC (batch rounded up to 8,
 * hw, hw, cout rounded up to 64) -> dst (device); layer 16: the head's input
 * activation (head.deconv2's BN + LeakyReLU output, 32x32 x 64 channels). */
int drcb_trainer_debug_z(DrcbTrainer *t, int32_t layer, void *dst, void *stream);

/* The batch L1 loss of the last bf16 (mode 2) step, read on `stream`
 * (synchronises). drcb_trainer_step is graph-capture safe in mode 2 after one
 * eager step at the same batch size (no allocation, no host sync when
 * loss_host is NULL; the Adam step counter lives on the device), so a
 * captured step can be replayed and its loss read here. */
int drcb_trainer_last_loss(DrcbTrainer *t, double *loss, void *stream);

/* reduction hook replacing NCCL for the trainer's SyncBN statistics and
 * gradient all-reduce: fn(user, device buffer, count, is_double, stream)
 * leaves the sum over the `world` ranks in buf. */
typedef int (*DrcbReduceFn)(void *user, void *buf, int64_t count, int32_t is_double, void *stream);
int drcb_trainer_set_reducer(DrcbTrainer *t, DrcbReduceFn fn, void *user, int32_t world);

/* loopback communicator: `world` ranks as host threads of one process
 * (half-batch trainers on one GPU), reduced in rank order; per-rank ctx for
 * drcb_loopback_reduce (a DrcbReduceFn). */
int drcb_loopback_create(int32_t world, void **out);
int drcb_loopback_rank(void *lb, int32_t rank, void **ctx);
int drcb_loopback_reduce(void *ctx, void *buf, int64_t count, int32_t is_double, void *stream);
void drcb_loopback_destroy(void *lb, void **ranks, int32_t n);
/* synchronous byte copy between host / device addresses on `stream` (the
 * host-staged reduction hooks, e.g. a gloo all-reduce). */
int drcb_copy_sync(void *dst, const void *src, int64_t bytes, void *stream);

/* ---- NCCL plumbing (libnccl.so.2 opened at first use) ------------------ */
int drcb_nccl_unique_id(void *out128);
int drcb_nccl_comm_create(const void *id128, int32_t world, int32_t rank, void **comm);
int drcb_nccl_comm_destroy(void *comm);
int drcb_allreduce_sum_f32(void *comm, float *buf, int64_t n, void *stream);

/* DRCW bytes of the current weights + running stats into host buf (cap
 * bytes); returns the size (buf = NULL to query). */
int64_t drcb_trainer_export(const DrcbTrainer *t, void *buf, int64_t cap);

const char *drcb_last_error(void);
int drcb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DRCB_H */
