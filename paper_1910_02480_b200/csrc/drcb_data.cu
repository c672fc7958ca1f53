// drcb_data.cu — the trainer's input pipeline on the device
// (trainer/src/drc_trainer/data.py:86-121): gather a batch of examples from
// the resident base set, apply one augmentation variant per item (azimuthal
// circular column shift by {0, 8, 16, 24} and optional horizontal flip, with
// the frame-local normals re-expressed) and the ablation mask.
#include "drcb_internal.h"

namespace drcb {
namespace {

constexpr int RES = 32;
constexpr int PIX = RES * RES;

// One thread per (item, pixel). Variant v: shift = 8 * (v >> 1), flip = v & 1.
// transform_example (data.py:86-100): inp = roll(inp, -shift, axis=-1) then
// [..., ::-1] when flipped, so output column c reads input column
// (c' + shift) mod 32 with c' = flipped ? 31 - c : c. The normal pair is
// rotated in float64 exactly as _rotate_normals_xy (data.py:77-83):
// (x ca + y sa, -x sa + y ca), cast to float32, y negated under the flip.
// cs = host-computed numpy cos/sin of 2*pi*shift/32 for the four shifts.
__global__ void k_augment(const float* __restrict__ xb, const float* __restrict__ yb,
                          const int64_t* __restrict__ base, const int32_t* __restrict__ variant,
                          int64_t n, DrcbAugmentTrig cs, int32_t ablate, float* __restrict__ xo,
                          float* __restrict__ yo) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * PIX) return;
  const int64_t i = t / PIX;
  const int pix = int(t % PIX), r = pix / RES, c = pix % RES;
  const int v = variant ? variant[i] : 0;
  const int s = v >> 1;
  const bool flip = v & 1;
  const int src_c = ((flip ? RES - 1 - c : c) + 8 * s) & (RES - 1);
  const int64_t b = base[i];
  const float* xi = xb + b * 7 * PIX + r * RES + src_c;
  const float* yi = yb + b * 3 * PIX + r * RES + src_c;
  float* xout = xo + i * 7 * PIX + pix;
  float* yout = yo + i * 3 * PIX + pix;
  for (int ch = 0; ch < 3; ++ch) {
    xout[ch * PIX] = __ldg(xi + ch * PIX);
    yout[ch * PIX] = __ldg(yi + ch * PIX);
  }
  // ablate (data.py:106-117) zeroes the channels before the transform; the
  // rotation and flip keep exact zeros zero (up to the sign of -0.0)
  const bool no_n = ablate & 1, no_d = ablate & 2;
  const double x = no_n ? 0.0 : double(__ldg(xi + 3 * PIX));
  const double y = no_n ? 0.0 : double(__ldg(xi + 4 * PIX));
  const double ca = cs.cos_a[s], sa = cs.sin_a[s];
  const float nx = __double2float_rn(__dadd_rn(__dmul_rn(x, ca), __dmul_rn(y, sa)));
  const float ny = __double2float_rn(__dadd_rn(__dmul_rn(-x, sa), __dmul_rn(y, ca)));
  xout[3 * PIX] = nx;
  xout[4 * PIX] = flip ? -ny : ny;
  xout[5 * PIX] = no_n ? 0.f : __ldg(xi + 5 * PIX);
  xout[6 * PIX] = no_d ? 0.f : __ldg(xi + 6 * PIX);
}

}  // namespace
}  // namespace drcb

using namespace drcb;

extern "C" int drcb_augment_gather(const float* x_base, const float* y_base, const int64_t* base,
                                   const int32_t* variant, int64_t n, const DrcbAugmentTrig* trig,
                                   int32_t ablate, float* x_out, float* y_out, void* stream) {
  if (n <= 0) return 0;
  if (!x_base || !y_base || !base || !trig || !x_out || !y_out)
    return fail(DRCB_ECONTRACT, "drcb_augment_gather: null argument");
  if (ablate & ~3) return fail(DRCB_ECONFIG, "drcb_augment_gather: unknown ablation bits");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tot = n * PIX;
  k_augment<<<unsigned((tot + 255) / 256), 256, 0, st>>>(x_base, y_base, base, variant, n, *trig,
                                                          ablate, x_out, y_out);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_augment");
}
