// drcb_train.cu — the autoencoder's training step on the B200
// (trainer/src/drc_trainer/train.py:97-103): MapAutoencoder forward with
// train-mode batch norm (model.py:20-88), L1 loss, backward through every
// layer (LeakyReLU, batch norm, conv/deconv dgrad + wgrad, max-pool,
// bilinear upsample, channel concat), Adam with fp32 master weights, and an
// optional NCCL all-reduce of gradients + batch-norm statistics (SyncBN) for
// data-parallel training. fp32 CUDA-core engine (the parity engine).
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "drcb_train.h"

namespace drcb {

int conv_f32(const ConvLayer& L, const float* in, int cin_tot, int cin_off, float* out,
             int cout_tot, int cout_off, int64_t n, float slope, cudaStream_t st);
int maxpool_f32(const float* in, int c_tot, int c_off, int c, int hw_out, float* out, int64_t n,
                cudaStream_t st);
int upsample_f32(const float* in, int c, int hw_in, float* out, int c_tot, int64_t n,
                 cudaStream_t st);

namespace train {

__global__ void k_fill(float* p, int64_t n, float v) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// conv-form weights for the forward (deconv: swap channel axes + flip,
// cnn.py:124-131) and for dgrad (transpose + flip of the conv form)
__global__ void k_wforms(const float* __restrict__ w, int cin, int cout, int ks, int deconv,
                         float* __restrict__ wf, float* __restrict__ wt) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t n = int64_t(cin) * cout * ks * ks;
  if (i >= n) return;
  int kx = int(i % ks), ky = int((i / ks) % ks);
  int64_t r = i / (ks * ks);
  int ci = int(r % cin), co = int(r / cin);
  // conv form wf[co][ci][ky][kx]
  float v;
  if (deconv)
    v = w[((int64_t(ci) * cout + co) * ks + (ks - 1 - ky)) * ks + (ks - 1 - kx)];
  else
    v = w[((int64_t(co) * cin + ci) * ks + ky) * ks + kx];
  wf[i] = v;
  // dgrad form wt[ci][co][ky][kx] = wf[co][ci][ks-1-ky][ks-1-kx]
  wt[((int64_t(ci) * cout + co) * ks + (ks - 1 - ky)) * ks + (ks - 1 - kx)] = v;
}

// Deterministic reductions: every block writes its partial sums to its own
// slot (part[(slot * gridDim.x + block) ...]); k_reduce_partials adds a
// slot's partials in block order. No floating-point atomics anywhere, so a
// step is bit-reproducible run to run (the reference's determinism, SURVEY
// §8(b)).
__global__ void k_reduce_partials(const double* __restrict__ part, int nparts, int nslots,
                                  double* __restrict__ out) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  double a = 0.0;
  for (int b = 0; b < nparts; ++b) a += part[int64_t(s) * nparts + b];
  out[s] = a;
}

// per-channel sum / sum of squares (double accumulation) of an NCHW slice:
// partial slots (2c, 2c+1) of block blockIdx.x
__global__ void k_chan_stats(const float* __restrict__ x, int c_tot, int c_off, int hw2, int64_t n,
                             double* part) {
  int c = blockIdx.y;
  int64_t total = n * hw2;
  double s = 0, ss = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t m = i / hw2;
    int p = int(i % hw2);
    double v = x[(m * c_tot + c_off + c) * hw2 + p];
    s += v;
    ss += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  __shared__ double red[2][32];
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    red[0][w] = s;
    red[1][w] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) {
      s += red[0][k];
      ss += red[1][k];
    }
    part[int64_t(2 * c) * gridDim.x + blockIdx.x] = s;
    part[int64_t(2 * c + 1) * gridDim.x + blockIdx.x] = ss;
  }
}

// batch statistics -> mean / invstd, running-stat update (momentum 0.1,
// unbiased variance for the running estimate; torch BatchNorm2d defaults)
__global__ void k_bn_finalize(const double* acc, int c, double count, float* mean, float* invstd,
                              float* rm, float* rv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c) return;
  double mu = acc[2 * i] / count;
  double var = acc[2 * i + 1] / count - mu * mu;
  if (var < 0) var = 0;
  mean[i] = float(mu);
  invstd[i] = float(1.0 / sqrt(var + double(EPS)));
  rm[i] = (1.f - MOMENTUM) * rm[i] + MOMENTUM * float(mu);
  rv[i] = (1.f - MOMENTUM) * rv[i] + MOMENTUM * float(var * count / (count - 1.0));
}

// a = LeakyReLU(gamma * (z - mean) * invstd + beta) into an output slice
__global__ void k_bn_act(const float* __restrict__ z, int c, int hw2, int64_t n,
                         const float* __restrict__ mean, const float* __restrict__ invstd,
                         const float* __restrict__ gamma, const float* __restrict__ beta,
                         float slope, float* __restrict__ out, int c_tot, int c_off) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * c * hw2) return;
  int p = int(i % hw2);
  int64_t r = i / hw2;
  int ch = int(r % c);
  int64_t m = r / c;
  float y = gamma[ch] * ((z[i] - mean[ch]) * invstd[ch]) + beta[ch];
  out[(m * c_tot + c_off + ch) * hw2 + p] = y > 0.f ? y : slope * y;
}

// L1 loss (mean |pred - target|) and its gradient through the final ReLU
__global__ void k_l1(const float* __restrict__ pred, const float* __restrict__ tgt, int64_t n,
                     double* part, float* __restrict__ dpre) {
  double s = 0;
  float inv = 1.f / float(n);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float d = pred[i] - tgt[i];
    s += fabs(double(d));
    float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    dpre[i] = pred[i] > 0.f ? sg * inv : 0.f;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) s += red[k];
    part[blockIdx.x] = s;
  }
}

// LeakyReLU + BN backward, pass 1: per-channel sums of dyb and dyb * xhat
__global__ void k_bn_bwd_stats(const float* __restrict__ z, const float* __restrict__ da,
                               int da_tot, int da_off, int c, int hw2, int64_t n,
                               const float* __restrict__ mean, const float* __restrict__ invstd,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               float slope, double* part) {
  int ch = blockIdx.y;
  int64_t total = n * hw2;
  double s = 0, sx = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t m = i / hw2;
    int p = int(i % hw2);
    float xh = (z[(m * c + ch) * hw2 + p] - mean[ch]) * invstd[ch];
    float y = gamma[ch] * xh + beta[ch];
    float g = da[(m * da_tot + da_off + ch) * hw2 + p];
    float dyb = y > 0.f ? g : slope * g;
    s += dyb;
    sx += double(dyb) * xh;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
  }
  __shared__ double red[2][32];
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    red[0][w] = s;
    red[1][w] = sx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) {
      s += red[0][k];
      sx += red[1][k];
    }
    part[int64_t(2 * ch) * gridDim.x + blockIdx.x] = s;
    part[int64_t(2 * ch + 1) * gridDim.x + blockIdx.x] = sx;
  }
}

// pass 2: dz = gamma * invstd * (dyb - mean(dyb) - xhat * mean(dyb * xhat))
__global__ void k_bn_bwd_apply(const float* __restrict__ z, const float* __restrict__ da, int da_tot,
                               int da_off, int c, int hw2, int64_t n,
                               const float* __restrict__ mean, const float* __restrict__ invstd,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               float slope, const double* acc, double count, float* __restrict__ dz) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * c * hw2) return;
  int p = int(i % hw2);
  int64_t r = i / hw2;
  int ch = int(r % c);
  int64_t m = r / c;
  float xh = (z[i] - mean[ch]) * invstd[ch];
  float y = gamma[ch] * xh + beta[ch];
  float g = da[(m * da_tot + da_off + ch) * hw2 + p];
  float dyb = y > 0.f ? g : slope * g;
  float md = float(acc[2 * ch] / count), mdx = float(acc[2 * ch + 1] / count);
  dz[i] = gamma[ch] * invstd[ch] * (dyb - md - xh * mdx);
}

__global__ void k_bn_param_grads(const double* acc, int c, float* dgamma, float* dbeta) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c) return;
  dbeta[i] = float(acc[2 * i]);
  dgamma[i] = float(acc[2 * i + 1]);
}

// weight gradient of a stride-1 conv: dW[co][ci][ky][kx] =
//   sum_{n,y,x} dz[n,co,y,x] * in[n,ci,y+ky-r,x+kx-r]; one block per (co, ci)
template <int KS>
__global__ void __launch_bounds__(256) k_wgrad(const float* __restrict__ dz, int cout,
                                               const float* __restrict__ in, int cin_tot,
                                               int cin_off, int cin, int hw, int64_t n,
                                               float* __restrict__ dw) {
  const int co = blockIdx.x / cin, ci = blockIdx.x % cin;
  const int hw2 = hw * hw;
  const int R = KS / 2;
  float acc[KS * KS];
#pragma unroll
  for (int t = 0; t < KS * KS; ++t) acc[t] = 0.f;
  for (int64_t i = threadIdx.x; i < n * hw2; i += blockDim.x) {
    int64_t m = i / hw2;
    int p = int(i % hw2);
    int y = p / hw, x = p % hw;
    float g = dz[(m * cout + co) * hw2 + p];
    const float* ib = in + (m * cin_tot + cin_off + ci) * hw2;
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      int yy = y + ky - R;
#pragma unroll
      for (int kx = 0; kx < KS; ++kx) {
        int xx = x + kx - R;
        float v = (yy >= 0 && yy < hw && xx >= 0 && xx < hw) ? __ldg(ib + yy * hw + xx) : 0.f;
        acc[ky * KS + kx] += g * v;
      }
    }
  }
  __shared__ float red[KS * KS][8];
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
#pragma unroll
  for (int t = 0; t < KS * KS; ++t) {
    float v = acc[t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[t][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < KS * KS) {
    float s = 0.f;
    for (int k = 0; k < int(blockDim.x / 32); ++k) s += red[threadIdx.x][k];
    dw[(int64_t(co) * cin + ci) * KS * KS + threadIdx.x] = s;
  }
}

// conv-form weight gradient -> parameter layout (deconv: back-transpose)
__global__ void k_wgrad_to_param(const float* __restrict__ dwf, int cin, int cout, int ks,
                                 int deconv, float* __restrict__ g) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t n = int64_t(cin) * cout * ks * ks;
  if (i >= n) return;
  int kx = int(i % ks), ky = int((i / ks) % ks);
  int64_t r = i / (ks * ks);
  int ci = int(r % cin), co = int(r / cin);
  float v = dwf[i];
  if (deconv)
    g[((int64_t(ci) * cout + co) * ks + (ks - 1 - ky)) * ks + (ks - 1 - kx)] = v;
  else
    g[i] = v;
}

// per-channel sum of an NCHW tensor into float (conv bias gradient)
__global__ void k_chan_sum(const float* __restrict__ x, int c, int hw2, int64_t n, float* out) {
  int ch = blockIdx.x;
  double s = 0;
  for (int64_t i = threadIdx.x; i < n * hw2; i += blockDim.x) {
    int64_t m = i / hw2;
    int p = int(i % hw2);
    s += x[(m * c + ch) * hw2 + p];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) s += red[k];
    out[ch] = float(s);
  }
}

// max-pool backward (first maximum of the 2x2 window in scan order gets the
// gradient, torch's tie rule) + the skip-connection gradient slice
__global__ void k_pool_bwd_add(const float* __restrict__ a, int a_tot, int a_off, int c,
                               int hw_out, int64_t n, const float* __restrict__ dp,
                               const float* __restrict__ dskip, int ds_tot, int ds_off,
                               float* __restrict__ da) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * c * hw_out * hw_out) return;
  int x = int(i % hw_out);
  int64_t r = i / hw_out;
  int y = int(r % hw_out);
  r /= hw_out;
  int ch = int(r % c);
  int64_t m = r / c;
  int hi = 2 * hw_out;
  const float* ab = a + ((m * a_tot + a_off + ch) * hi + 2 * y) * hi + 2 * x;
  float v[4] = {ab[0], ab[1], ab[hi], ab[hi + 1]};
  int best = 0;
  for (int k = 1; k < 4; ++k)
    if (v[k] > v[best] || isnan(v[k])) best = k;
  float g = dp[i];
  const float* sb = dskip + ((m * ds_tot + ds_off + ch) * hi + 2 * y) * hi + 2 * x;
  float* ob = da + ((m * c + ch) * hi + 2 * y) * hi + 2 * x;
  int offs[4] = {0, 1, hi, hi + 1};
  for (int k = 0; k < 4; ++k) ob[offs[k]] = sb[offs[k]] + (k == best ? g : 0.f);
}

// bilinear-2x backward (adjoint of upsample_bilinear2x2): gather form
__device__ __forceinline__ float up_weight(int o, int i, int n) {
  // weight of low-res index i in output o (align_corners=False)
  int i0, i1;
  float fr;
  const int h = o >> 1;
  if (o & 1) {
    i0 = h;
    i1 = min(h + 1, n - 1);
    fr = 0.25f;
  } else if (o == 0) {
    i0 = 0;
    i1 = min(1, n - 1);
    fr = 0.f;
  } else {
    i0 = h - 1;
    i1 = h;
    fr = 0.75f;
  }
  return (i0 == i ? 1.f - fr : 0.f) + (i1 == i ? fr : 0.f);
}

__global__ void k_up_bwd(const float* __restrict__ dhigh, int c_tot, int c, int hw_in, int64_t n,
                         float* __restrict__ dlow) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * c * hw_in * hw_in) return;
  int x = int(i % hw_in);
  int64_t r = i / hw_in;
  int y = int(r % hw_in);
  r /= hw_in;
  int ch = int(r % c);
  int64_t m = r / c;
  int ho = 2 * hw_in;
  const float* b = dhigh + (m * c_tot + ch) * ho * ho;
  float s = 0.f;
  for (int oy = max(0, 2 * y - 2); oy <= min(ho - 1, 2 * y + 3); ++oy) {
    float wy = up_weight(oy, y, hw_in);
    if (wy == 0.f) continue;
    for (int ox = max(0, 2 * x - 2); ox <= min(ho - 1, 2 * x + 3); ++ox) {
      float wx = up_weight(ox, x, hw_in);
      if (wx != 0.f) s += wy * wx * b[oy * ho + ox];
    }
  }
  dlow[i] = s;
}

// torch.optim.Adam (amsgrad=False, weight_decay=0): m, v, bias corrections,
// p -= lr/bc1 * m / (sqrt(v)/sqrt(bc2) + eps)
// The step counter and the bias corrections live on the device (double, as
// torch computes them on the host) so that a captured step graph replays
// with the right step number: coef = {lr / bc1, sqrt(bc2)}.
__global__ void k_adam_coef(int64_t* step, float lr, float b1, float b2, float* coef) {
  const int64_t s = *step + 1;
  *step = s;
  const double bc1 = 1.0 - pow(double(b1), double(s));
  const double bc2 = 1.0 - pow(double(b2), double(s));
  coef[0] = float(double(lr) / bc1);
  coef[1] = float(sqrt(bc2));
}

__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, const float* __restrict__ coef, float b1,
                       float b2, float eps, float gscale) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float step_size = coef[0], bc2_sqrt = coef[1];
  float gi = g[i] * gscale;
  float mi = m[i] + (1.f - b1) * (gi - m[i]);  // exp_avg.lerp_(grad, 1 - beta1)
  float vi = b2 * v[i] + (1.f - b2) * (gi * gi);
  m[i] = mi;
  v[i] = vi;
  float denom = sqrtf(vi) / bc2_sqrt + eps;
  p[i] = p[i] - step_size * (mi / denom);
}

inline unsigned nb(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// 1x1 conv weight gradient (head.conv_out): dW[co][ci] = sum_p dz x, grid
// (chunks, cout * cin), double accumulation, partial slot blockIdx.y
__global__ void k_wgrad1_part(const float* __restrict__ dz, int cout, const float* __restrict__ in,
                              int cin, int hw2, int64_t n, double* part) {
  const int co = blockIdx.y / cin, ci = blockIdx.y % cin;
  double s = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * hw2;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / hw2;
    const int p = int(i % hw2);
    s += double(dz[(m * cout + co) * hw2 + p]) * in[(m * cin + ci) * hw2 + p];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) s += red[k];
    part[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = s;
  }
}

// per-channel sum of an NCHW tensor (conv bias gradient), grid (chunks, c)
__global__ void k_chan_sum_part(const float* __restrict__ x, int c, int hw2, int64_t n, double* part) {
  const int ch = blockIdx.y;
  double s = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * hw2;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / hw2;
    s += x[(m * c + ch) * hw2 + int(i % hw2)];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x / 32); ++k) s += red[k];
    part[int64_t(ch) * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void k_acc_to_float(const double* acc, int c, float* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < c) out[i] = float(acc[i]);
}

}  // namespace train
}  // namespace drcb


namespace drcb {
namespace train {

struct Spec {
  const char* name;
  const char* bn;
  int cin, cout, hw, ks;
  bool deconv;
};

std::vector<Spec> specs(int k) {
  return {{"enc1.conv1", "enc1.bn1", 7, k, 32, 3, false},
          {"enc1.conv2", "enc1.bn2", k, k, 32, 3, false},
          {"enc2.conv1", "enc2.bn1", k, 2 * k, 16, 3, false},
          {"enc2.conv2", "enc2.bn2", 2 * k, 2 * k, 16, 3, false},
          {"enc3.conv1", "enc3.bn1", 2 * k, 4 * k, 8, 3, false},
          {"enc3.conv2", "enc3.bn2", 4 * k, 4 * k, 8, 3, false},
          {"bott.conv1", "bott.bn1", 4 * k, 8 * k, 4, 3, false},
          {"bott.conv2", "bott.bn2", 8 * k, 8 * k, 4, 3, false},
          {"dec3.deconv1", "dec3.bn1", 12 * k, 4 * k, 8, 3, true},
          {"dec3.deconv2", "dec3.bn2", 4 * k, 4 * k, 8, 3, true},
          {"dec2.deconv1", "dec2.bn1", 6 * k, 2 * k, 16, 3, true},
          {"dec2.deconv2", "dec2.bn2", 2 * k, 2 * k, 16, 3, true},
          {"dec1.deconv1", "dec1.bn1", 3 * k, k, 32, 3, true},
          {"dec1.deconv2", "dec1.bn2", k, k, 32, 3, true},
          {"head.deconv1", "head.bn1", k, k / 2, 32, 3, true},
          {"head.deconv2", "head.bn2", k / 2, k / 4, 32, 3, true},
          {"head.conv_out", "", k / 4, 3, 32, 1, false}};
}

// an NCHW activation view: buffer, total channels, channel offset
struct View {
  float* p;
  int ctot, coff;
};

struct Work {
  std::vector<float*> z;    // pre-BN outputs per layer
  std::vector<float*> mean, invstd;
  // forward activations
  float *a0, *c1, *p1, *a2, *c2, *p2, *a4, *c3, *p3, *a6, *a7, *a8, *a9, *a10, *a11, *a12, *a13,
      *a14, *a15, *pred;
  // gradients
  float *d0, *da1, *dp1, *d2, *da3, *dp2, *d4, *da5, *dp3, *d6, *d7, *d8, *d9, *d10, *d11, *d12,
      *d13, *d14, *d15, *dc1, *dc2, *dc3, *dpre, *dz, *dwf;
  double* acc;   // reduced sums (2 x channels)
  double* part;  // per-block partial sums (see k_reduce_partials)
  double* loss;
  void* base = nullptr;
};

constexpr int GX = 64;  // partial blocks of the per-channel reductions

}  // namespace train
}  // namespace drcb

using namespace drcb;
using namespace drcb::train;

namespace {

int alloc_work(DrcbTrainer* T, int64_t n, Work& W, cudaStream_t st) {
  const int k = T->k;
  std::vector<std::pair<float**, size_t>> req;
  size_t per = 0;
  auto add = [&](float** p, size_t floats_per_map) { req.push_back({p, floats_per_map}); };
  W.z.assign(16, nullptr);
  for (int l = 0; l < 16; ++l) add(&W.z[l], size_t(T->L[l].cout) * T->L[l].hw * T->L[l].hw);
  add(&W.a0, k * 1024); add(&W.c1, 3 * k * 1024); add(&W.p1, k * 256); add(&W.a2, 2 * k * 256);
  add(&W.c2, 6 * k * 256); add(&W.p2, 2 * k * 64); add(&W.a4, 4 * k * 64); add(&W.c3, 12 * k * 64);
  add(&W.p3, 4 * k * 16); add(&W.a6, 8 * k * 16); add(&W.a7, 8 * k * 16); add(&W.a8, 4 * k * 64);
  add(&W.a9, 4 * k * 64); add(&W.a10, 2 * k * 256); add(&W.a11, 2 * k * 256); add(&W.a12, k * 1024);
  add(&W.a13, k * 1024); add(&W.a14, k / 2 * 1024); add(&W.a15, k / 4 * 1024); add(&W.pred, 3 * 1024);
  add(&W.d0, k * 1024); add(&W.da1, k * 1024); add(&W.dp1, k * 256); add(&W.d2, 2 * k * 256);
  add(&W.da3, 2 * k * 256); add(&W.dp2, 2 * k * 64); add(&W.d4, 4 * k * 64); add(&W.da5, 4 * k * 64);
  add(&W.dp3, 4 * k * 16); add(&W.d6, 8 * k * 16); add(&W.d7, 8 * k * 16); add(&W.d8, 4 * k * 64);
  add(&W.d9, 4 * k * 64); add(&W.d10, 2 * k * 256); add(&W.d11, 2 * k * 256); add(&W.d12, k * 1024);
  add(&W.d13, k * 1024); add(&W.d14, k / 2 * 1024); add(&W.d15, k / 4 * 1024);
  add(&W.dc1, 3 * k * 1024); add(&W.dc2, 6 * k * 256); add(&W.dc3, 12 * k * 64);
  add(&W.dpre, 3 * 1024); add(&W.dz, size_t(k) * 1024 * 3);
  for (auto& r : req) per += (r.second + 63) / 64 * 64;
  int64_t maxw = 0;
  for (const auto& l : T->L) maxw = std::max(maxw, l.nw);
  size_t bytes = per * n * 4 + size_t(maxw) * 4 + (16 * 2 * 1024 + 4096) * 8 + 1024 * 1024 +
                 size_t(GX) * 2 * 1024 * 8 + 1024 * 8;
  DRCB_CUDA(cudaMallocAsync(&W.base, bytes, st));
  float* cur = static_cast<float*>(W.base);
  for (auto& r : req) {
    *r.first = cur;
    cur += (r.second + 63) / 64 * 64 * n;
  }
  W.dwf = cur;
  cur += (maxw + 63) / 64 * 64;
  W.mean.assign(16, nullptr);
  W.invstd.assign(16, nullptr);
  for (int l = 0; l < 16; ++l) {
    W.mean[l] = cur;
    cur += 1024;
    W.invstd[l] = cur;
    cur += 1024;
  }
  uintptr_t a = (reinterpret_cast<uintptr_t>(cur) + 7) & ~uintptr_t(7);
  W.acc = reinterpret_cast<double*>(a);
  W.loss = W.acc + 2 * 1024;
  W.part = W.loss + 8;

  return 0;
}

void conv_layer_view(const DrcbTrainer* T, int l, const float* wf, ConvLayer& L) {
  const TL& t = T->L[l];
  L.cin = t.cin;
  L.cout = t.cout;
  L.hw = t.hw;
  L.ksize = t.ks;
  L.act = false;
  L.mode = 0;  // bias only: batch norm runs in its own kernels
  L.d_w = const_cast<float*>(wf);
  L.d_bias = T->params + t.b;
  L.d_scale = nullptr;
  L.d_shift = nullptr;
}

#define TCHECK(name)                                        \
  do {                                                      \
    count_launch();                                         \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return cuda_fail(_e, name);      \
  } while (0)

}  // namespace

extern "C" int drcb_trainer_create(const void* drcw, size_t len, float lr, float beta1,
                                   float beta2, float eps, DrcbTrainer** out) {
  if (!drcw || !out) return fail(DRCB_ECONTRACT, "drcb_trainer_create: null argument");
  DrcbNet* net = nullptr;
  int rc = drcb_net_create(drcw, len, &net);  // validates the container
  if (rc) return rc;
  DrcbTrainer* T = new DrcbTrainer();
  const NetImpl& N = net->impl;
  T->k = N.k;
  T->slope = N.slope;
  T->slope_bits = N.slope_bits;
  T->lr = lr;
  T->b1 = beta1;
  T->b2 = beta2;
  T->eps = eps;
  std::vector<float> hp, hr;
  for (const Spec& s : specs(N.k)) {
    TL t;
    t.name = s.name;
    t.bn = s.bn;
    t.cin = s.cin;
    t.cout = s.cout;
    t.hw = s.hw;
    t.ks = s.ks;
    t.deconv = s.deconv;
    t.has_bn = s.bn[0] != 0;
    const auto& w = N.tensors.at(t.name + ".weight");
    const auto& b = N.tensors.at(t.name + ".bias");
    t.nw = int64_t(w.size());
    t.w = int64_t(hp.size());
    hp.insert(hp.end(), w.begin(), w.end());
    t.b = int64_t(hp.size());
    hp.insert(hp.end(), b.begin(), b.end());
    t.g = t.be = t.rm = t.rv = -1;
    if (t.has_bn) {
      const auto& g = N.tensors.at(t.bn + ".gamma");
      const auto& be = N.tensors.at(t.bn + ".beta");
      t.g = int64_t(hp.size());
      hp.insert(hp.end(), g.begin(), g.end());
      t.be = int64_t(hp.size());
      hp.insert(hp.end(), be.begin(), be.end());
      const auto& rm = N.tensors.at(t.bn + ".running_mean");
      const auto& rv = N.tensors.at(t.bn + ".running_var");
      t.rm = int64_t(hr.size());
      hr.insert(hr.end(), rm.begin(), rm.end());
      t.rv = int64_t(hr.size());
      hr.insert(hr.end(), rv.begin(), rv.end());
    }
    T->L.push_back(t);
  }
  drcb_net_destroy(net);
  T->n_params = int64_t(hp.size());
  T->n_running = int64_t(hr.size());
  int64_t wtot = 0;
  for (const auto& t : T->L) {
    T->wf_off.push_back(wtot);
    wtot += t.nw;
  }
  size_t pbytes = size_t(T->n_params) * 4;
  void* p = nullptr;
  const size_t sbytes = (pbytes * 4 + size_t(T->n_running) * 4 + size_t(wtot) * 8 + 15) & ~size_t(15);
  if (cudaMalloc(&p, sbytes + 16) != cudaSuccess) {
    delete T;
    return fail(DRCB_ECUDA, "cudaMalloc trainer state");
  }
  T->allocs.push_back(p);
  float* f = static_cast<float*>(p);
  T->params = f;
  T->grads = f + T->n_params;
  T->m = f + 2 * T->n_params;
  T->v = f + 3 * T->n_params;
  T->running = f + 4 * T->n_params;
  T->wf = T->running + T->n_running;
  T->wt = T->wf + wtot;
  T->d_step = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(p) + sbytes);
  T->d_coef = reinterpret_cast<float*>(T->d_step + 1);
  cudaMemset(T->d_step, 0, 16);
  cudaMemcpy(T->params, hp.data(), pbytes, cudaMemcpyHostToDevice);
  cudaMemset(T->grads, 0, pbytes * 3);
  cudaMemcpy(T->running, hr.data(), size_t(T->n_running) * 4, cudaMemcpyHostToDevice);
  *out = T;
  return 0;
}

// Select the conv engine: 0 = fp32 CUDA cores (the parity engine, default),
// 2 = the NHWC bf16 tensor-core engine (drcb_train_tc.cu: forward, dgrad and
// wgrad on tcgen05, fp32 master weights, batch statistics and Adam).
extern "C" int drcb_trainer_set_mode(DrcbTrainer* T, int32_t mode) {
  if (!T) return fail(DRCB_ECONTRACT, "drcb_trainer_set_mode: null trainer");
  if (mode != 0 && mode != 2) return fail(DRCB_ECONFIG, "trainer mode must be 0 (fp32) or 2 (bf16)");
  if (mode == 2 && T->k != 64)
    return fail(DRCB_ECONFIG, "the tensor-core trainer is built for k = 64 (use mode 0 for other k)");
  T->mode = mode;
  return 0;
}

extern "C" void drcb_trainer_destroy(DrcbTrainer* T) {
  if (!T) return;
  if (T->tc) tc_engine_destroy(T->tc);
  if (T->comm_stream) {
    for (cudaEvent_t e : T->comm_ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : T->sync_ev)
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(T->comm_stream);
  }
  for (void* p : T->allocs) cudaFree(p);
  delete T;
}

extern "C" int drcb_trainer_info(const DrcbTrainer* T, int64_t* out4) {
  if (!T || !out4) return fail(DRCB_ECONTRACT, "drcb_trainer_info: null argument");
  out4[0] = T->k;
  out4[1] = T->n_params;
  out4[2] = T->n_running;
  int64_t step = 0;  // the device counter (graph replays advance it too)
  if (cudaMemcpy(&step, T->d_step, sizeof(step), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(DRCB_ECUDA, "drcb_trainer_info: step counter");
  out4[3] = step;
  return 0;
}

// device pointers of the flat parameter and gradient buffers (fp32, torch
// parameter order) — for external all-reduce or inspection
extern "C" int drcb_trainer_buffers(const DrcbTrainer* T, void** params, void** grads,
                                    void** running) {
  if (!T) return fail(DRCB_ECONTRACT, "drcb_trainer_buffers: null trainer");
  if (params) *params = T->params;
  if (grads) *grads = T->grads;
  if (running) *running = T->running;
  return 0;
}

namespace {

int bn_forward(DrcbTrainer* T, int l, Work& W, int64_t n, const View& out, cudaStream_t st) {
  const TL& t = T->L[l];
  const int hw2 = t.hw * t.hw;
  k_chan_stats<<<dim3(GX, t.cout), 256, 0, st>>>(W.z[l], t.cout, 0, hw2, n, W.part);
  TCHECK("k_chan_stats");
  k_reduce_partials<<<nb(2 * t.cout), 256, 0, st>>>(W.part, GX, 2 * t.cout, W.acc);
  TCHECK("k_reduce_partials");
  // SyncBN: batch statistics over all data-parallel ranks (NVLink all-reduce)
  int rc = trainer_allreduce(T, W.acc, size_t(2) * t.cout, 1, st);
  if (rc) return rc;
  k_bn_finalize<<<nb(t.cout), 256, 0, st>>>(W.acc, t.cout, double(n) * hw2 * T->world, W.mean[l],
                                               W.invstd[l], T->running + t.rm, T->running + t.rv);
  TCHECK("k_bn_finalize");
  k_bn_act<<<nb(n * t.cout * hw2), 256, 0, st>>>(W.z[l], t.cout, hw2, n, W.mean[l], W.invstd[l],
                                                  T->params + t.g, T->params + t.be, T->slope,
                                                  out.p, out.ctot, out.coff);
  TCHECK("k_bn_act");
  return 0;
}

// conv/deconv + train BN + LeakyReLU layer l: in -> out slice
int layer_forward(DrcbTrainer* T, int l, Work& W, int64_t n, const View& in, const View& out,
                  cudaStream_t st) {
  ConvLayer L;
  conv_layer_view(T, l, T->wf + T->wf_off[l], L);
  int rc = conv_f32(L, in.p, in.ctot, in.coff, W.z[l], T->L[l].cout, 0, n, T->slope, st);
  if (rc) return rc;
  return bn_forward(T, l, W, n, out, st);
}

// backward of layer l: dout slice -> dz, param grads, din (full buffer of
// the layer input, written; NULL to skip dgrad)
int layer_backward(DrcbTrainer* T, int l, Work& W, int64_t n, const View& in, const View& dout,
                   float* din, int din_ctot, cudaStream_t st) {
  const TL& t = T->L[l];
  const int hw2 = t.hw * t.hw;
  k_bn_bwd_stats<<<dim3(GX, t.cout), 256, 0, st>>>(W.z[l], dout.p, dout.ctot, dout.coff, t.cout, hw2,
                                                  n, W.mean[l], W.invstd[l], T->params + t.g,
                                                  T->params + t.be, T->slope, W.part);
  TCHECK("k_bn_bwd_stats");
  k_reduce_partials<<<nb(2 * t.cout), 256, 0, st>>>(W.part, GX, 2 * t.cout, W.acc);
  TCHECK("k_reduce_partials");
  // local gamma/beta gradients first (they join the gradient all-reduce)
  k_bn_param_grads<<<nb(t.cout), 256, 0, st>>>(W.acc, t.cout, T->grads + t.g, T->grads + t.be);
  TCHECK("k_bn_param_grads");
  // SyncBN backward: global means of dyb and dyb * xhat
  {
    int rc = trainer_allreduce(T, W.acc, size_t(2) * t.cout, 1, st);
    if (rc) return rc;
  }
  k_bn_bwd_apply<<<nb(n * t.cout * hw2), 256, 0, st>>>(W.z[l], dout.p, dout.ctot, dout.coff,
                                                        t.cout, hw2, n, W.mean[l], W.invstd[l],
                                                        T->params + t.g, T->params + t.be,
                                                        T->slope, W.acc, double(n) * hw2 * T->world,
                                                        W.dz);
  TCHECK("k_bn_bwd_apply");
  k_chan_sum_part<<<dim3(GX, t.cout), 256, 0, st>>>(W.dz, t.cout, hw2, n, W.part);
  TCHECK("k_chan_sum_part");
  k_reduce_partials<<<nb(t.cout), 256, 0, st>>>(W.part, GX, t.cout, W.acc);
  TCHECK("k_reduce_partials");
  k_acc_to_float<<<nb(t.cout), 256, 0, st>>>(W.acc, t.cout, T->grads + t.b);
  TCHECK("k_acc_to_float");
  k_wgrad<3><<<t.cout * t.cin, 256, 0, st>>>(W.dz, t.cout, in.p, in.ctot, in.coff, t.cin, t.hw, n,
                                              W.dwf);
  TCHECK("k_wgrad");
  k_wgrad_to_param<<<nb(t.nw), 256, 0, st>>>(W.dwf, t.cin, t.cout, 3, t.deconv, T->grads + t.w);
  TCHECK("k_wgrad_to_param");
  if (din) {
    ConvLayer D;
    D.cin = t.cout;
    D.cout = t.cin;
    D.hw = t.hw;
    D.ksize = 3;
    D.act = false;
    D.mode = 0;
    D.d_w = T->wt + T->wf_off[l];
    D.d_bias = nullptr;
    int rc = conv_f32(D, W.dz, t.cout, 0, din, din_ctot, 0, n, T->slope, st);
    if (rc) return rc;
  }
  return 0;
}

}  // namespace

extern "C" int drcb_trainer_apply(DrcbTrainer* T, float grad_scale, void* stream);

namespace drcb {
namespace train {
int trainer_allreduce(DrcbTrainer* T, void* buf, size_t count, int is_double, cudaStream_t st) {
  if (T->reduce_fn) {
    int rc = T->reduce_fn(T->reduce_user, buf, int64_t(count), is_double, st);
    return rc ? fail(DRCB_ENCCL, "reduction hook failed") : 0;
  }
  return allreduce_sum(T->comm, buf, count, is_double, st);
}

void layer_param_range(const DrcbTrainer* T, int l, int64_t& off, int64_t& count) {
  const TL& t = T->L[l];
  off = t.w;
  count = (t.has_bn ? t.be + t.cout : t.b + t.cout) - t.w;
}

// conv-form (forward) and transposed-flipped (dgrad) fp32 weights of every
// layer from the master parameters
int weight_forms(DrcbTrainer* T, cudaStream_t st) {
  for (int l = 0; l < NL; ++l) {
    const TL& t = T->L[l];
    k_wforms<<<nb(t.nw), 256, 0, st>>>(T->params + t.w, t.cin, t.cout, t.ks, t.deconv,
                                        T->wf + T->wf_off[l], T->wt + T->wf_off[l]);
    TCHECK("k_wforms");
  }
  return 0;
}
}  // namespace train
}  // namespace drcb

// One optimisation step (train.py:97-103) on n examples: x (n,7,32,32),
// y (n,3,32,32) device fp32. loss_host (optional) receives the batch L1 loss
// (synchronises). apply_adam = 0 leaves parameters untouched (grads only).
extern "C" int drcb_trainer_step(DrcbTrainer* T, const float* x, const float* y, int64_t n,
                                 double* loss_host, int32_t apply_adam, void* stream) {
  if (!T || !x || !y) return fail(DRCB_ECONTRACT, "drcb_trainer_step: null argument");
  if (n < 1) return fail(DRCB_ECONFIG, "training step needs n >= 1 examples");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  keep_pool_memory();
  const int64_t nout = n * 3 * 1024;
  int rc = 0;
  if (T->mode == 2) {
    // the NHWC tensor-core engine: forward, loss and backward into T->grads
    // (it packs its bf16 operands straight from the master parameters)
    double* loss_dev = nullptr;
    rc = tc_step(T, x, y, n, &loss_dev, st);
    // NCCL: the gradients were all-reduced layer by layer inside the step
    // (bucketed, overlapping the backward); a reduction hook gets one call
    if (!rc && (T->reduce_fn || !T->comm)) rc = trainer_allreduce(T, T->grads, size_t(T->n_params), 0, st);
    if (!rc && apply_adam) rc = drcb_trainer_apply(T, 1.0f / float(T->world), stream);
    if (rc) return rc;
    if (loss_host) {
      double loss = 0;
      DRCB_CUDA(cudaMemcpyAsync(&loss, loss_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
      DRCB_CUDA(cudaStreamSynchronize(st));
      *loss_host = loss / double(nout);
    }
    return 0;
  }
  rc = weight_forms(T, st);
  if (rc) return rc;
  const int k = T->k;
  Work W;
  rc = alloc_work(T, n, W, st);
  if (rc) return rc;
  float* xin = const_cast<float*>(x);
  // ---- forward (model.py:80-88)
  rc |= layer_forward(T, 0, W, n, {xin, 7, 0}, {W.a0, k, 0}, st);
  rc |= layer_forward(T, 1, W, n, {W.a0, k, 0}, {W.c1, 3 * k, 2 * k}, st);
  rc |= maxpool_f32(W.c1, 3 * k, 2 * k, k, 16, W.p1, n, st);
  rc |= layer_forward(T, 2, W, n, {W.p1, k, 0}, {W.a2, 2 * k, 0}, st);
  rc |= layer_forward(T, 3, W, n, {W.a2, 2 * k, 0}, {W.c2, 6 * k, 4 * k}, st);
  rc |= maxpool_f32(W.c2, 6 * k, 4 * k, 2 * k, 8, W.p2, n, st);
  rc |= layer_forward(T, 4, W, n, {W.p2, 2 * k, 0}, {W.a4, 4 * k, 0}, st);
  rc |= layer_forward(T, 5, W, n, {W.a4, 4 * k, 0}, {W.c3, 12 * k, 8 * k}, st);
  rc |= maxpool_f32(W.c3, 12 * k, 8 * k, 4 * k, 4, W.p3, n, st);
  rc |= layer_forward(T, 6, W, n, {W.p3, 4 * k, 0}, {W.a6, 8 * k, 0}, st);
  rc |= layer_forward(T, 7, W, n, {W.a6, 8 * k, 0}, {W.a7, 8 * k, 0}, st);
  rc |= upsample_f32(W.a7, 8 * k, 4, W.c3, 12 * k, n, st);
  rc |= layer_forward(T, 8, W, n, {W.c3, 12 * k, 0}, {W.a8, 4 * k, 0}, st);
  rc |= layer_forward(T, 9, W, n, {W.a8, 4 * k, 0}, {W.a9, 4 * k, 0}, st);
  rc |= upsample_f32(W.a9, 4 * k, 8, W.c2, 6 * k, n, st);
  rc |= layer_forward(T, 10, W, n, {W.c2, 6 * k, 0}, {W.a10, 2 * k, 0}, st);
  rc |= layer_forward(T, 11, W, n, {W.a10, 2 * k, 0}, {W.a11, 2 * k, 0}, st);
  rc |= upsample_f32(W.a11, 2 * k, 16, W.c1, 3 * k, n, st);
  rc |= layer_forward(T, 12, W, n, {W.c1, 3 * k, 0}, {W.a12, k, 0}, st);
  rc |= layer_forward(T, 13, W, n, {W.a12, k, 0}, {W.a13, k, 0}, st);
  rc |= layer_forward(T, 14, W, n, {W.a13, k, 0}, {W.a14, k / 2, 0}, st);
  rc |= layer_forward(T, 15, W, n, {W.a14, k / 2, 0}, {W.a15, k / 4, 0}, st);
  {
    ConvLayer L;  // head.conv_out (1x1) + bias + ReLU (model.py:48-51)
    conv_layer_view(T, 16, T->wf + T->wf_off[16], L);
    L.mode = 2;
    rc |= conv_f32(L, W.a15, k / 4, 0, W.pred, 3, 0, n, T->slope, st);
  }
  if (rc) {
    cudaFreeAsync(W.base, st);
    return rc;
  }
  // ---- L1 loss (train.py:88) + gradient through the final ReLU
  k_l1<<<1024, 256, 0, st>>>(W.pred, y, nout, W.part, W.dpre);
  TCHECK("k_l1");
  k_reduce_partials<<<1, 32, 0, st>>>(W.part, 1024, 1, W.loss);
  TCHECK("k_l1");
  // ---- backward
  {
    const TL& t = T->L[16];
    // conv_out: dW, db, d(a15)
    k_chan_sum_part<<<dim3(GX, 3), 256, 0, st>>>(W.dpre, 3, 1024, n, W.part);
    TCHECK("k_chan_sum_part");
    k_reduce_partials<<<1, 32, 0, st>>>(W.part, GX, 3, W.acc);
    k_acc_to_float<<<1, 32, 0, st>>>(W.acc, 3, T->grads + t.b);
    TCHECK("k_acc_to_float");
    k_wgrad1_part<<<dim3(GX, 3 * t.cin), 256, 0, st>>>(W.dpre, 3, W.a15, t.cin, 1024, n, W.part);
    TCHECK("k_wgrad1_part");
    k_reduce_partials<<<nb(3 * t.cin), 256, 0, st>>>(W.part, GX, 3 * t.cin, W.acc + 3);
    k_acc_to_float<<<nb(3 * t.cin), 256, 0, st>>>(W.acc + 3, 3 * t.cin, W.dwf);
    TCHECK("k_acc_to_float");
    k_wgrad_to_param<<<nb(t.nw), 256, 0, st>>>(W.dwf, t.cin, 3, 1, 0, T->grads + t.w);
    TCHECK("k_wgrad_to_param");
    ConvLayer D;
    D.cin = 3;
    D.cout = t.cin;
    D.hw = 32;
    D.ksize = 1;
    D.act = false;
    D.mode = 0;
    D.d_w = T->wt + T->wf_off[16];
    D.d_bias = nullptr;
    rc |= conv_f32(D, W.dpre, 3, 0, W.d15, k / 4, 0, n, T->slope, st);
  }
  rc |= layer_backward(T, 15, W, n, {W.a14, k / 2, 0}, {W.d15, k / 4, 0}, W.d14, k / 2, st);
  rc |= layer_backward(T, 14, W, n, {W.a13, k, 0}, {W.d14, k / 2, 0}, W.d13, k, st);
  rc |= layer_backward(T, 13, W, n, {W.a12, k, 0}, {W.d13, k, 0}, W.d12, k, st);
  rc |= layer_backward(T, 12, W, n, {W.c1, 3 * k, 0}, {W.d12, k, 0}, W.dc1, 3 * k, st);
  k_up_bwd<<<nb(n * 2 * k * 256), 256, 0, st>>>(W.dc1, 3 * k, 2 * k, 16, n, W.d11);
  TCHECK("k_up_bwd");
  rc |= layer_backward(T, 11, W, n, {W.a10, 2 * k, 0}, {W.d11, 2 * k, 0}, W.d10, 2 * k, st);
  rc |= layer_backward(T, 10, W, n, {W.c2, 6 * k, 0}, {W.d10, 2 * k, 0}, W.dc2, 6 * k, st);
  k_up_bwd<<<nb(n * 4 * k * 64), 256, 0, st>>>(W.dc2, 6 * k, 4 * k, 8, n, W.d9);
  TCHECK("k_up_bwd");
  rc |= layer_backward(T, 9, W, n, {W.a8, 4 * k, 0}, {W.d9, 4 * k, 0}, W.d8, 4 * k, st);
  rc |= layer_backward(T, 8, W, n, {W.c3, 12 * k, 0}, {W.d8, 4 * k, 0}, W.dc3, 12 * k, st);
  k_up_bwd<<<nb(n * 8 * k * 16), 256, 0, st>>>(W.dc3, 12 * k, 8 * k, 4, n, W.d7);
  TCHECK("k_up_bwd");
  rc |= layer_backward(T, 7, W, n, {W.a6, 8 * k, 0}, {W.d7, 8 * k, 0}, W.d6, 8 * k, st);
  rc |= layer_backward(T, 6, W, n, {W.p3, 4 * k, 0}, {W.d6, 8 * k, 0}, W.dp3, 4 * k, st);
  k_pool_bwd_add<<<nb(n * 4 * k * 16), 256, 0, st>>>(W.c3, 12 * k, 8 * k, 4 * k, 4, n, W.dp3, W.dc3,
                                                      12 * k, 8 * k, W.da5);
  TCHECK("k_pool_bwd_add");
  rc |= layer_backward(T, 5, W, n, {W.a4, 4 * k, 0}, {W.da5, 4 * k, 0}, W.d4, 4 * k, st);
  rc |= layer_backward(T, 4, W, n, {W.p2, 2 * k, 0}, {W.d4, 4 * k, 0}, W.dp2, 2 * k, st);
  k_pool_bwd_add<<<nb(n * 2 * k * 64), 256, 0, st>>>(W.c2, 6 * k, 4 * k, 2 * k, 8, n, W.dp2, W.dc2,
                                                      6 * k, 4 * k, W.da3);
  TCHECK("k_pool_bwd_add");
  rc |= layer_backward(T, 3, W, n, {W.a2, 2 * k, 0}, {W.da3, 2 * k, 0}, W.d2, 2 * k, st);
  rc |= layer_backward(T, 2, W, n, {W.p1, k, 0}, {W.d2, 2 * k, 0}, W.dp1, k, st);
  k_pool_bwd_add<<<nb(n * k * 256), 256, 0, st>>>(W.c1, 3 * k, 2 * k, k, 16, n, W.dp1, W.dc1, 3 * k,
                                                   2 * k, W.da1);
  TCHECK("k_pool_bwd_add");
  rc |= layer_backward(T, 1, W, n, {W.a0, k, 0}, {W.da1, k, 0}, W.d0, k, st);
  rc |= layer_backward(T, 0, W, n, {xin, 7, 0}, {W.d0, k, 0}, nullptr, 0, st);
  if (rc) {
    cudaFreeAsync(W.base, st);
    return rc;
  }
  // ---- data-parallel gradient average happens between here and Adam
  // (drcb_trainer_apply after an external all-reduce, or apply_adam below)
  // gradient all-reduce over the data-parallel ranks (sum); the per-rank
  // loss is a local mean, so the average is sum / world
  rc = trainer_allreduce(T, T->grads, size_t(T->n_params), 0, st);
  if (rc) {
    cudaFreeAsync(W.base, st);
    return rc;
  }
  if (apply_adam) {
    rc = drcb_trainer_apply(T, 1.0f / float(T->world), stream);
    if (rc) {
      cudaFreeAsync(W.base, st);
      return rc;
    }
  }
  double loss = 0;
  if (loss_host) {
    DRCB_CUDA(cudaMemcpyAsync(&loss, W.loss, sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  DRCB_CUDA(cudaFreeAsync(W.base, st));
  if (loss_host) {
    DRCB_CUDA(cudaStreamSynchronize(st));
    *loss_host = loss / double(nout);
  }
  return 0;
}

// Adam on the (externally all-reduced) gradient buffer; grad_scale
// multiplies the gradients first (1/world for an all-reduce sum)
extern "C" int drcb_trainer_apply(DrcbTrainer* T, float grad_scale, void* stream) {
  if (!T) return fail(DRCB_ECONTRACT, "drcb_trainer_apply: null trainer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_adam_coef<<<1, 1, 0, st>>>(T->d_step, T->lr, T->b1, T->b2, T->d_coef);
  TCHECK("k_adam_coef");
  k_adam<<<nb(T->n_params), 256, 0, st>>>(T->params, T->grads, T->m, T->v, T->n_params, T->d_coef,
                                           T->b1, T->b2, T->eps, grad_scale);
  TCHECK("k_adam");
  return 0;
}

// data-parallel communicator (ncclComm_t from drcb_nccl_comm_create; NULL =
// single process): SyncBN statistics and the gradient all-reduce use it
extern "C" int drcb_trainer_set_comm(DrcbTrainer* T, void* comm, int32_t world) {
  if (!T || world < 1) return fail(DRCB_ECONTRACT, "drcb_trainer_set_comm: bad arguments");
  T->comm = comm;
  T->reduce_fn = nullptr;
  T->reduce_user = nullptr;
  T->world = comm ? world : 1;
  return 0;
}

// a reduction hook in place of NCCL: fn(user, device buffer, count, is_double,
// stream) must leave the sum over the `world` ranks in the buffer (the
// SyncBN statistics and the gradients of the data-parallel step go through it)
extern "C" int drcb_trainer_set_reducer(DrcbTrainer* T, DrcbReduceFn fn, void* user, int32_t world) {
  if (!T || world < 1) return fail(DRCB_ECONTRACT, "drcb_trainer_set_reducer: bad arguments");
  T->comm = nullptr;
  T->reduce_fn = fn;
  T->reduce_user = user;
  T->world = fn ? world : 1;
  return 0;
}

// DRCW export of the current parameters + running statistics (host bytes);
// returns the size (call with buf = NULL to query)
extern "C" int64_t drcb_trainer_export(const DrcbTrainer* T, void* buf, int64_t cap) {
  if (!T) return -1;
  std::vector<float> hp(T->n_params), hr(T->n_running);
  cudaMemcpy(hp.data(), T->params, hp.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hr.data(), T->running, hr.size() * 4, cudaMemcpyDeviceToHost);
  std::map<std::string, std::pair<std::vector<uint32_t>, std::vector<float>>> ts;
  for (const auto& t : T->L) {
    std::vector<uint32_t> wd = t.deconv ? std::vector<uint32_t>{uint32_t(t.cin), uint32_t(t.cout), 3, 3}
                                        : std::vector<uint32_t>{uint32_t(t.cout), uint32_t(t.cin),
                                                                uint32_t(t.ks), uint32_t(t.ks)};
    ts[t.name + ".weight"] = {wd, std::vector<float>(hp.begin() + t.w, hp.begin() + t.w + t.nw)};
    ts[t.name + ".bias"] = {{uint32_t(t.cout)}, std::vector<float>(hp.begin() + t.b, hp.begin() + t.b + t.cout)};
    if (t.has_bn) {
      ts[t.bn + ".gamma"] = {{uint32_t(t.cout)}, std::vector<float>(hp.begin() + t.g, hp.begin() + t.g + t.cout)};
      ts[t.bn + ".beta"] = {{uint32_t(t.cout)}, std::vector<float>(hp.begin() + t.be, hp.begin() + t.be + t.cout)};
      ts[t.bn + ".running_mean"] = {{uint32_t(t.cout)}, std::vector<float>(hr.begin() + t.rm, hr.begin() + t.rm + t.cout)};
      ts[t.bn + ".running_var"] = {{uint32_t(t.cout)}, std::vector<float>(hr.begin() + t.rv, hr.begin() + t.rv + t.cout)};
    }
  }
  std::vector<uint8_t> out;
  auto put = [&](const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    out.insert(out.end(), b, b + n);
  };
  put("DRCW", 4);
  uint32_t ver = 1, cnt = uint32_t(ts.size());
  put(&ver, 4);
  put(&T->slope_bits, 4);
  put(&cnt, 4);
  for (const auto& kv : ts) {  // std::map: sorted by name, as the reference writes
    uint16_t nl = uint16_t(kv.first.size());
    put(&nl, 2);
    put(kv.first.data(), nl);
    uint8_t rank = uint8_t(kv.second.first.size());
    put(&rank, 1);
    put(kv.second.first.data(), 4 * rank);
    put(kv.second.second.data(), 4 * kv.second.second.size());
  }
  if (buf && cap >= int64_t(out.size())) std::memcpy(buf, out.data(), out.size());
  return int64_t(out.size());
}
