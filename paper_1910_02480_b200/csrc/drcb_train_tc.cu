// drcb_train_tc.cu — the autoencoder's training step on the tensor cores,
// NHWC bf16 end to end (trainer/src/drc_trainer/train.py:97-103 with
// MapAutoencoder in train mode, model.py:20-88; BASELINE config 5: bf16
// compute, fp32 master weights).
//
// Per 3x3 layer, forward: conv (tcgen05 implicit GEMM, epilogue = bias) ->
// Z (bf16) -> batch statistics (deterministic per-block partials) -> BN +
// LeakyReLU (+ the fused 2x2 max-pool of the encoder skips) straight into
// the next layer's input buffer or the decoder's concat slice. Backward:
// BN/LeakyReLU backward (two passes: per-channel sums, then dZ), dgrad
// (tcgen05 transposed conv into the input-gradient buffer / concat slices),
// wgrad (tcgen05 with MN-major operands read from the same NHWC tensors,
// drcb_wgrad.cu), pool / upsample backward as NHWC gathers, the 1x1 head +
// L1 loss fused in one kernel. Activations never leave NHWC bf16; every
// buffer is allocated once per batch capacity (no per-step allocations); no
// floating-point atomics (the step is bit-reproducible). The fp32 master
// weights, gradients, running statistics and Adam live in drcb_train.cu.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "drcb_train.h"

namespace drcb {

int tc_conv_bf16(int cin, int cout, int hw, int64_t nmaps, const void* in, int cin_pad, void* out,
                 int out_ctot, int out_coff, const void* wpacked, int cout_pad, const float* ep_a,
                 const float* ep_b, float slope, cudaStream_t st, int in_pitch);
int tc_conv_in8_bf16(int64_t nmaps, const void* in, void* out, int out_ctot, const void* w8,
                     const float* ep_a, const float* ep_b, float slope, cudaStream_t st);
int wgrad_bf16(const void* x, int cin, int cin_pad, const void* dz, int cout, int cout_pad, int hw,
               int64_t nmaps, float* dwf, int deconv, void* ws, size_t* ws_bytes, cudaStream_t st,
               int x_pitch, int dz_pitch);

namespace train {

using bf16 = __nv_bfloat16;

inline int pad64(int c) { return (c + 63) / 64 * 64; }
// 8-channel groups a per-channel pass covers per 64-channel tile: 8, or the
// real channels of a layer with fewer than 64 (head.deconv1 / deconv2)
inline int chan_groups(int cout) { return cout <= 16 ? 2 : (cout <= 32 ? 4 : 8); }
// elements between pixels of a layer's Z / activation / gradient tensors:
// 64-channel multiples, except the head's 32- and 16-channel layers, which
// are stored at that width (a quarter / half of the bytes of every pass over
// them; the tensor-core kernels load them into 64-channel boxes through the
// TMA zero fill and store them through box clipping)
inline int zpitch(int cout) { return cout < 64 ? 8 * chan_groups(cout) : pad64(cout); }
inline unsigned nbk(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

#define TC_CHECK(name)                                      \
  do {                                                      \
    count_launch();                                         \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return cuda_fail(_e, name);      \
  } while (0)

// ---------------------------------------------------------------------------
// 16-B vectors of 8 bf16 channels
__device__ __forceinline__ void ld8(const bf16* p, float (&f)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
// the same through the streaming cache policy (evict-first), for the passes
// that read a tensor for the last time in a while (the BN applies: Z and dA
// are dead after the backward's apply, which leaves L2 to the dZ it writes
// for the dgrad and wgrad; the statistics passes keep the default policy,
// their tensors are re-read by the apply right after). DRCB_BN_NOSTREAM:
// plain loads (A/B)
__device__ __forceinline__ void ld8s(const bf16* p, float (&f)[8]) {
#ifdef DRCB_BN_NOSTREAM
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
#else
  const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
#endif
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ void st8(bf16* p, const float (&f)[8]) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&b);
  }
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void round8(float (&f)[8]) {  // the stored (bf16) values
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = __bfloat162float(__float2bfloat16_rn(f[j]));
}

// ---------------------------------------------------------------------------
// input (n,7,32,32) fp32 NCHW -> X0 (np,32,32,8) bf16 NHWC: channels 0..6,
// zeros in channel 7 and in the maps beyond n (stored 8 channels wide: the
// convs load it into 64-channel boxes through the TMA zero fill)
__global__ void k_x_in(const float* __restrict__ x, int64_t n, int64_t np, bf16* __restrict__ out) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= np * 1024) return;
  const int64_t m = i / 1024;
  const int p = int(i % 1024);
  float f[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) f[c] = (c < 7 && m < n) ? __ldg(x + (m * 7 + c) * 1024 + p) : 0.f;
  st8(out + i * 8, f);
}

// Every layer's step operands straight from the fp32 master parameters, in
// one launch: the forward form wpf[co][tap][ci] (a deconv's weight flipped
// and transposed, model.py:33-34), the dgrad form wpt[ci][tap][co] =
// wf[co][ci][8 - tap], both bf16 and zero-padded to 64 channels, and the
// padded conv bias. One thread per (layer, form, output row, input channel)
// moves the 9 taps; the fastest index is the packed layout's contiguous one
// so the 2-byte stores coalesce (the 36-byte tap runs are read whole).
struct PrepLayer {
  const float *w, *b;
  bf16 *wpf, *wpt;
  float* ep_b;
  int cin, cout, cinp, coutp, deconv;
};
struct PrepArgs {
  PrepLayer L[16];
  int64_t start[17];  // thread-segment starts; segment = wpf rows, wpt rows, bias
};

__global__ void k_prep_weights(const __grid_constant__ PrepArgs a) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.start[16]) return;
  int l = 0;
  while (i >= a.start[l + 1]) ++l;
  const PrepLayer& t = a.L[l];
  int64_t j = i - a.start[l];
  const int64_t nf = int64_t(t.coutp) * t.cinp;
  if (j < 2 * nf) {
    const bool fwd = j < nf;
    if (!fwd) j -= nf;
    // forward rows: (co, ci) ci fastest; dgrad rows: (ci, co) co fastest
    const int inner = fwd ? t.cinp : t.coutp;
    const int r = int(j / inner), c = int(j % inner);
    const int co = fwd ? r : c, ci = fwd ? c : r;
    float v[9];
    if (co < t.cout && ci < t.cin) {
      // wf[co][ci][tap]: conv w[co][ci][tap], deconv w[ci][co][8 - tap]
      const float* src = t.deconv ? t.w + (int64_t(ci) * t.cout + co) * 9
                                  : t.w + (int64_t(co) * t.cin + ci) * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) v[k] = src[t.deconv ? 8 - k : k];
    } else {
#pragma unroll
      for (int k = 0; k < 9; ++k) v[k] = 0.f;
    }
    if (fwd) {
      bf16* dst = t.wpf + int64_t(co) * 9 * t.cinp + ci;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[int64_t(k) * t.cinp] = __float2bfloat16_rn(v[k]);
    } else {
      bf16* dst = t.wpt + int64_t(ci) * 9 * t.coutp + co;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[int64_t(k) * t.coutp] = __float2bfloat16_rn(v[8 - k]);
    }
    return;
  }
  j -= 2 * nf;
  t.ep_b[j] = j < t.cout ? t.b[j] : 0.f;
}

// enc1.conv1's weights in the in8 kernel's layout: w8[co][tap * 8 + ci]
// (bf16, zeros for ci >= cin and K >= 72), from the conv-form fp32 w[co][ci][tap]
__global__ void k_prep_in8(const float* __restrict__ w, int cin, int cout, bf16* __restrict__ w8) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 64 * 128) return;
  const int co = i / 128, kk = i % 128, t = kk / 8, ci = kk % 8;
  const float v = (co < cout && t < 9 && ci < cin) ? w[(int64_t(co) * cin + ci) * 9 + t] : 0.f;
  w8[i] = __float2bfloat16_rn(v);
}

// padded epilogue vector: v[c] (or fill when v == NULL) for c < n, 0 beyond
__global__ void k_pad_vec(const float* __restrict__ v, int n, int np, float fill, float* out) {
  pdl_wait();
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < np) out[c] = c < n ? (v ? v[c] : fill) : 0.f;
}

// Per-channel reductions over the first npx pixels of an NHWC tensor (pixel
// pitch cpad): blocks (bx, channel tile of 64) sweep the tensor together in
// chunks of 4 * PL pixels, chunk k to block k % gx (grid-stride: the grid
// moves through memory as one front, low to high, or high to low with `rev`,
// so a pass can start where the previous kernel's writes ended while they
// are still in L2); thread = (8-ch group, one of PL = 256/CG pixel lanes);
// the lanes' sums are combined in lane order in double. CG = 8 groups cover
// a 64-channel tile; a layer with fewer real channels (head.deconv1 /
// deconv2: 32 / 16) runs CG = 4 / 2 and never touches the padding (a quarter
// / half of the bytes). Partial slot (q*cpad + c) of block bx at
// part[(q*cpad + c)*gx + bx], q = 0..NQ-1.
template <int NQ, int CG, class F>
__device__ __forceinline__ void chan_reduce(int64_t npx, int rev, int cpad, double* part, F f) {
  constexpr int PL = 256 / CG, CT = 8 * CG, CH = 4 * PL;
  const int cg = threadIdx.x % CG, pl = threadIdx.x / CG;
  const int c0 = blockIdx.y * 64 + cg * 8;
  f.init(c0);  // this thread's 8 channels are fixed: per-channel constants once
  float acc[NQ][8];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[q][j] = 0.f;
  // four pixels per lane in flight (the loads of one chunk are issued before
  // their arithmetic: enough bytes in flight per SM for HBM rate)
  const int64_t nch = (npx + CH - 1) / CH;
  for (int64_t k = blockIdx.x; k < nch; k += gridDim.x) {
    const int64_t kc = rev ? nch - 1 - k : k;
    const int64_t q0 = kc * CH + pl;
    if ((kc + 1) * CH <= npx) {
      f.template go<4, PL>(q0, c0, acc);
    } else {
      for (int64_t p = q0; p < npx; p += PL) f.template go<1, PL>(p, c0, acc);
    }
  }
  __shared__ float red[NQ][PL][CT + 1];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) red[q][pl][cg * 8 + j] = acc[q][j];
  __syncthreads();
  if (threadIdx.x < CT * NQ) {
    const int q = threadIdx.x / CT, c = threadIdx.x % CT;
    double s = 0.0;
    for (int l = 0; l < PL; ++l) s += double(red[q][l][c]);
    part[(int64_t(q) * cpad + blockIdx.y * 64 + c) * gridDim.x + blockIdx.x] = s;
  }
}

// one warp per slot: lane l adds parts l, l+32, ... in order, then a fixed
// butterfly combines the lanes (deterministic)
// Optional fp32 copies of two slot ranges (gradients that are these sums):
// f0[i] = out[i] and f1[i] = out[cpad + i] for i < c.
__global__ void k_reduce_parts(const double* __restrict__ part, int nparts, int nslots,
                               double* __restrict__ out, int c = 0, int cpad = 0,
                               float* __restrict__ f0 = nullptr, float* __restrict__ f1 = nullptr) {
  pdl_wait();
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (s >= nslots) return;
  double a = 0.0;
  {
    // (four loads in flight ahead of the in-order adds: same sums, same bits)
    const double* q = part + int64_t(s) * nparts;
    int b = lane;
    for (; b + 96 < nparts; b += 128) {
      const double v0 = q[b], v1 = q[b + 32], v2 = q[b + 64], v3 = q[b + 96];
      a += v0;
      a += v1;
      a += v2;
      a += v3;
    }
    for (; b < nparts; b += 32) a += q[b];
  }
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) {
    out[s] = a;
    if (f0 && s < c) f0[s] = float(a);
    if (f1 && s >= cpad && s < cpad + c) f1[s - cpad] = float(a);
  }
}
inline unsigned nb_slots(int nslots) { return unsigned((int64_t(nslots) * 32 + 255) / 256); }

// forward batch statistics: sum z, sum z^2 per channel
struct StatsF {
  const bf16* z;
  int pitch;
  __device__ __forceinline__ void init(int) {}
  template <int U, int PS>
  __device__ __forceinline__ void go(int64_t p, int c0, float (&acc)[2][8]) const {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) ld8(z + (p + PS * u) * pitch + c0, v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[0][j] += v[u][j];
        acc[1][j] = fmaf(v[u][j], v[u][j], acc[1][j]);
      }
  }
};
template <int CG>
__global__ void __launch_bounds__(256) k_bn_stats(const bf16* __restrict__ z, int pitch, int cpad,
                                                  int64_t npx, double* part) {
  pdl_wait();
  chan_reduce<2, CG>(npx, 0, cpad, part, StatsF{z, pitch});
}

// BN finalize (torch BatchNorm2d train mode: biased variance normalises,
// unbiased variance updates the running estimate, momentum 0.1):
// y = z * s + t with s = gamma * invstd, t = beta - mean * s
struct BnFin {  // forward: batch mean / invstd -> scale, shift, running stats
  int c, cpad;
  double count;
  const float *gamma, *beta;
  float *rm, *rv, *bnv;
  __device__ void operator()(int i, double s0, double s1) const {
    if (i >= c) return;
    double mu = s0 / count;
    double var = s1 / count - mu * mu;
    if (var < 0) var = 0;
    const float invstd = float(1.0 / sqrt(var + double(EPS)));
    const float s = gamma[i] * invstd;
    bnv[i] = s;                               // scale
    bnv[cpad + i] = beta[i] - float(mu) * s;  // shift
    bnv[2 * cpad + i] = float(mu);            // mean
    bnv[3 * cpad + i] = invstd;               // invstd
    rm[i] = (1.f - MOMENTUM) * rm[i] + MOMENTUM * float(mu);
    rv[i] = (1.f - MOMENTUM) * rv[i] + MOMENTUM * float(var * count / (count - 1.0));
  }
};

// backward: means of dyb and dyb * xhat over the (global) batch, and
// gamma * invstd; with `dbeta` set (one rank: the sums are already the
// batch's) also the beta / gamma gradients
struct BnbCoef {
  int c, cpad;
  double count;
  const float* gamma;
  float* bnv;
  float *dbeta, *dgamma;
  __device__ void operator()(int i, double s0, double s1) const {
    const bool real = i < c;
    if (real && dbeta) {
      dbeta[i] = float(s0);
      dgamma[i] = float(s1);
    }
    bnv[4 * cpad + i] = real ? float(s0 / count) : 0.f;              // m1
    bnv[5 * cpad + i] = real ? float(s1 / count) : 0.f;              // m2
    bnv[6 * cpad + i] = real ? gamma[i] * bnv[3 * cpad + i] : 0.f;  // gamma * invstd
  }
};

// finalise from all-reduced sums (sum slot i, square/product slot cpad + i)
template <class F>
__global__ void k_fin(const double* sums, int n, F f) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f(i, sums[i], sums[f.cpad + i]);
}

// one rank (nothing to all-reduce): the partial reduction and the
// finalisation in one launch, a warp per channel, partials summed in block
// order exactly as k_reduce_parts does
template <class F>
__global__ void k_reduce_fin(const double* __restrict__ part, int nparts, int n, F f) {
  pdl_wait();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (i >= n) return;
  double a = 0.0, b = 0.0;
  {
    // (four loads per sum in flight ahead of the in-order adds: same bits)
    const double* qa = part + int64_t(i) * nparts;
    const double* qb = part + int64_t(f.cpad + i) * nparts;
    int k = lane;
    for (; k + 96 < nparts; k += 128) {
      const double a0 = qa[k], a1 = qa[k + 32], a2 = qa[k + 64], a3 = qa[k + 96];
      const double b0 = qb[k], b1 = qb[k + 32], b2 = qb[k + 64], b3 = qb[k + 96];
      a += a0;
      a += a1;
      a += a2;
      a += a3;
      b += b0;
      b += b1;
      b += b2;
      b += b3;
    }
    for (; k < nparts; k += 32) {
      a += qa[k];
      b += qb[k];
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) f(i, a, b);
}

// Elementwise NHWC kernels: one thread per (pixel, 8-channel group); every
// extent is a power of two (lg* = log2) except the concat buffers' channel
// totals, which only multiply: 32-bit shift / mask indexing (no 64-bit
// division in the address math).
__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

// a = LeakyReLU(z * s + t) into out[.., c_off + c] (all np maps). Walked
// from the last pixel down: the stats pass that precedes it ended on the
// high pixels (still in L2), and the next layer's conv starts on the low
// ones this leaves in L2 (measured with the bnb_apply direction below:
// ~0.25 ms of a B = 4,096 step).
// (the first `groups` 8-channel groups of each pixel: the padding of a
// layer with fewer than 64 channels keeps its zeros)
__global__ void __launch_bounds__(256) k_bn_apply(const bf16* __restrict__ z, int zp, int cpad, int npx,
                                                  const float* __restrict__ bnv, float slope,
                                                  bf16* __restrict__ out, int c_tot, int c_off,
                                                  int groups) {
  pdl_wait();
  const int lg = ilog2(groups);
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (npx << lg)) return;
  i = (npx << lg) - 1 - i;  // high to low (see k_bn_apply's comment above)
  const int p = i >> lg, c0 = (i & ((1 << lg) - 1)) * 8;
  float v[8];
  ld8s(z + int64_t(p) * zp + c0, v);  // (Z's last reader until the backward)
  const float4 s0 = __ldg(reinterpret_cast<const float4*>(bnv + c0));
  const float4 s1 = __ldg(reinterpret_cast<const float4*>(bnv + c0 + 4));
  const float4 t0 = __ldg(reinterpret_cast<const float4*>(bnv + cpad + c0));
  const float4 t1 = __ldg(reinterpret_cast<const float4*>(bnv + cpad + c0 + 4));
  const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  const float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float y = fmaf(v[j], sv[j], tv[j]);
    v[j] = y >= 0.f ? y : slope * y;
  }
  st8(out + int64_t(p) * c_tot + c_off + c0, v);
}

// the same with the encoder's fused 2x2 max-pool (cnn.py:152-156) of the
// stored values into pool (hw/2 maps, cpad channels)
__global__ void __launch_bounds__(256) k_bn_apply_pool(const bf16* __restrict__ z, int cpad, int hw, int np,
                                                       const float* __restrict__ bnv, float slope,
                                                       bf16* __restrict__ out, int c_tot, int c_off,
                                                       bf16* __restrict__ pool) {
  pdl_wait();
  const int lg = ilog2(cpad / 8), lho = ilog2(hw / 2), hw_ = hw;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (np << (2 * lho + lg))) return;
  i = (np << (2 * lho + lg)) - 1 - i;  // high to low, as k_bn_apply
  const int c0 = (i & ((1 << lg) - 1)) * 8;
  const int pp = i >> lg;
  const int px = pp & ((1 << lho) - 1), py = (pp >> lho) & ((1 << lho) - 1), m = pp >> (2 * lho);
  float sv[8], tv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sv[j] = __ldg(bnv + c0 + j);
    tv[j] = __ldg(bnv + cpad + c0 + j);
  }
  float mx[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t p = (int64_t(m) * hw_ + 2 * py + (k >> 1)) * hw_ + 2 * px + (k & 1);
    float v[8];
    ld8(z + p * cpad + c0, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float y = fmaf(v[j], sv[j], tv[j]);
      v[j] = y >= 0.f ? y : slope * y;
    }
    round8(v);
#pragma unroll
    for (int j = 0; j < 8; ++j) mx[j] = k == 0 ? v[j] : fmaxf(mx[j], v[j]);
    st8(out + p * c_tot + c_off + c0, v);
  }
  st8(pool + int64_t(pp) * cpad + c0, mx);
}

// bilinear 2x upsample (align_corners=False, cnn.py:159-174): output index o
// reads low-res i0 = (o-1)/2, i1 = i0 + 1 (clamped) with weight 0.25 / 0.75
// (the closed form of src = max((o + 0.5)/2 - 0.5, 0))
__device__ __forceinline__ void up_src(int o, int n, int& i0, int& i1, float& fr) {
  if (o == 0) {
    i0 = 0;
    i1 = min(1, n - 1);
    fr = 0.f;
  } else if (o & 1) {
    i0 = o >> 1;
    i1 = min(i0 + 1, n - 1);
    fr = 0.25f;
  } else {
    i0 = (o >> 1) - 1;
    i1 = o >> 1;
    fr = 0.75f;
  }
}
// 16-B vector of 8 bf16 kept raw (4 registers) and widened on use
__device__ __forceinline__ uint4 ldraw(const bf16* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void widen(uint4 u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

// packed fp32 pairs (FFMA2 / FMUL2 on sm_100a: per lane the same correctly
// rounded fma / mul as the scalar instruction, half the issue slots)
__device__ __forceinline__ void widen2(uint4 u, float2 (&f)[4]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) f[j] = make_float2(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xffff0000u));
}
__device__ __forceinline__ uint4 narrow2(const float2 (&f)[4]) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 b = __floats2bfloat162_rn(f[j].x, f[j].y);
    w[j] = *reinterpret_cast<uint32_t*>(&b);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// a * (1 - f) + b * f as fma(a, 1 - f, b * f), the contraction the scalar
// kernels compile to
__device__ __forceinline__ float2 mix2(float2 a, float2 b, float f) {
  return __ffma2_rn(a, make_float2(1.f - f, 1.f - f), __fmul2_rn(b, make_float2(f, f)));
}

// one thread = the 2x2 output block of low-res pixel (i, j), 8 channels:
// rows i-1 .. i+1 x columns j-1 .. j+1 (clamped), nine 16-B loads for four
// outputs, the row and column mixes in packed fp32 pairs. Per output the same
// sources, weights and fma order as the reference-order scalar form (up_src:
// rows first, then columns), so the same bits. The two-output scalar kernel
// was issue-bound (80 % issue-active, 3.5 TB/s for the 16 -> 32 upsample);
// this one is bit-identical and 7 % faster (639 -> 596 us for the three
// upsamples at B = 4,096), now latency-bound at 64 registers (37 % warps
// active; 48 or 40 registers spill and are slower, 72 is slower too).
__global__ void __launch_bounds__(256) k_up_fwd(const bf16* __restrict__ in, int c, int hw_in, int np,
                                                bf16* __restrict__ out, int c_tot) {
  pdl_wait();
  const int lg = ilog2(c / 8), lhi = ilog2(hw_in), ho = 2 * hw_in;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (np << (2 * lhi + lg))) return;
  const int c0 = (t & ((1 << lg) - 1)) * 8;
  const int rest = t >> lg;
  const int j = rest & (hw_in - 1), i = (rest >> lhi) & (hw_in - 1), m = rest >> (2 * lhi);
  const bf16* b = in + int64_t(m) * hw_in * hw_in * c + c0;
  const int cl = max(j - 1, 0), cr = min(j + 1, hw_in - 1);
  const int rt = max(i - 1, 0), rb = min(i + 1, hw_in - 1);
  // output row 2i mixes rows (i-1, i) at 0.75 (rows (0, min(1, n-1)) at 0 for
  // i = 0); row 2i+1 mixes rows (i, min(i+1, n-1)) at 0.25 (up_src)
  const int a0 = i == 0 ? i : rt, a1 = i == 0 ? rb : i;
  const float fa = i == 0 ? 0.f : 0.75f;
  float2 ra[3][4], rbm[3][4];  // row-mixed columns (l, m, r) of output rows 2i, 2i+1
  {
    const int cols[3] = {cl, j, cr};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float2 x0[4], x1[4], x2[4];
      widen2(ldraw(b + (a0 * hw_in + cols[q]) * c), x0);
      widen2(ldraw(b + (a1 * hw_in + cols[q]) * c), x1);
      widen2(ldraw(b + (rb * hw_in + cols[q]) * c), x2);
      if (i != 0) {  // row i (= a1) then serves output row 2i+1 as its first row
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          ra[q][e] = mix2(x0[e], x1[e], fa);
          rbm[q][e] = mix2(x1[e], x2[e], 0.25f);
        }
      } else {  // i = 0: rows (0, min(1, n-1)) for both output rows
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          ra[q][e] = mix2(x0[e], x1[e], 0.f);
          rbm[q][e] = mix2(x0[e], x1[e], 0.25f);
        }
      }
    }
  }
  // columns: output 2j mixes (j-1, j) at 0.75 or, on the left border, (0,
  // min(1, n-1)) at 0; output 2j+1 mixes (j, min(j+1, n-1)) at 0.25
  const bool left = j == 0;
  const float fe = left ? 0.f : 0.75f;
  bf16* o = out + (int64_t(m) * ho * ho + int64_t(2 * i) * ho + 2 * j) * c_tot + c0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const float2(&v)[3][4] = r ? rbm : ra;
    float2 ve[4], vo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 e0 = left ? v[1][e] : v[0][e], e1 = left ? v[2][e] : v[1][e];
      ve[e] = mix2(e0, e1, fe);
      vo[e] = mix2(v[1][e], v[2][e], 0.25f);
    }
    bf16* orow = o + int64_t(r) * ho * c_tot;
    *reinterpret_cast<uint4*>(orow) = narrow2(ve);
    *reinterpret_cast<uint4*>(orow + c_tot) = narrow2(vo);
  }
}

// adjoint of the upsample: low index i receives from outputs 2i-1 .. 2i+2
// with weights (0.25, 0.75, 0.75, 0.25), folded at the map borders (output 0
// and 2n-1 give both of their taps to the border sample)
__device__ __forceinline__ void up_adj(int i, int n, int (&o)[4], float (&w)[4]) {
  o[0] = 2 * i - 1; o[1] = 2 * i; o[2] = 2 * i + 1; o[3] = 2 * i + 2;
  w[0] = 0.25f; w[1] = 0.75f; w[2] = 0.75f; w[3] = 0.25f;
  if (i == 0) {         // output 0 reads (0, 1) with weights (1, 0)
    w[0] = 0.f;
    w[1] = 1.f;
  }
  if (i == n - 1) {     // output 2n-1 reads (n-1, n-1): 0.75 + 0.25
    w[2] = 1.f;
    w[3] = 0.f;
  }
  if (n == 1) {         // a 1-pixel map: both outputs copy it
    w[1] = 1.f;
    w[2] = 1.f;
  }
}
// one thread = a column strip of the low-res gradient: output (y, x) for
// every y of one map, 8 channels, from high-res rows 2y - 1 .. 2y + 2 and
// columns 2x - 1 .. 2x + 2 (up_adj weights, folded at the borders). The
// adjoint is separable: each high-res row is first reduced over its four
// columns, h(o) = sum_b wx[b] d[o][ox[b]], once (two new rows per output: the
// last two of one y are the first two of the next), then the output is
// sum_a wy[a] h(2y - 1 + a); both in packed fp32 pairs. (The double sum with
// the products wy[a] wx[b] in one chain widened and multiplied every tap of
// every row twice and was issue-bound: 346 us for the 16 -> 32 adjoint at
// B = 4,096, 3.8 TB/s.)
__global__ void __launch_bounds__(256) k_up_bwd(const bf16* __restrict__ dhigh, int c_tot, int c, int hw_in,
                                                int np, bf16* __restrict__ dlow) {
  pdl_wait();
  const int lg = ilog2(c / 8), lhi = ilog2(hw_in), ho = 2 * hw_in;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (np << (lhi + lg))) return;
  const int c0 = (i & ((1 << lg) - 1)) * 8;
  const int rest = i >> lg;
  const int x = rest & (hw_in - 1), m = rest >> lhi;
  int ox[4];
  float wx[4];
  up_adj(x, hw_in, ox, wx);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (ox[b] < 0 || ox[b] >= ho) wx[b] = 0.f;
    ox[b] = min(max(ox[b], 0), ho - 1);
  }
  const bf16* base = dhigh + int64_t(m) * ho * ho * c_tot + c0;
  auto row = [&](int o, uint4 (&v)[4]) {
    const int oc = min(max(o, 0), ho - 1);
#pragma unroll
    for (int b = 0; b < 4; ++b) v[b] = ldraw(base + int64_t(oc * ho + ox[b]) * c_tot);
  };
  auto colsum = [&](const uint4 (&v)[4], float2 (&h)[4]) {
    float2 d[4];
    widen2(v[0], d);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __fmul2_rn(d[e], make_float2(wx[0], wx[0]));
#pragma unroll
    for (int b = 1; b < 4; ++b) {
      widen2(v[b], d);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __ffma2_rn(d[e], make_float2(wx[b], wx[b]), h[e]);
    }
  };
  float2 h0[4], h1[4], h2[4], h3[4];  // column sums of high-res rows 2y - 1 .. 2y + 2 (clamped)
  uint4 n2[4], n3[4];                 // raw rows 2y + 3, 2y + 4 (prefetched)
  row(-1, n2);
  row(0, n3);
  colsum(n2, h0);
  colsum(n3, h1);
  row(1, n2);
  row(2, n3);
  colsum(n2, h2);
  colsum(n3, h3);
  bf16* ob = dlow + (int64_t(m) * hw_in * hw_in + x) * c + c0;
  for (int y = 0; y < hw_in; ++y) {
    if (y > 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        h0[e] = h2[e];
        h1[e] = h3[e];
      }
      colsum(n2, h2);
      colsum(n3, h3);
    }
    if (y + 1 < hw_in) {  // the next y's new rows, in flight during this y's sums
      row(2 * y + 3, n2);
      row(2 * y + 4, n3);
    }
    int oy[4];
    float wy[4];
    up_adj(y, hw_in, oy, wy);
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (oy[a] < 0 || oy[a] >= ho) wy[a] = 0.f;
    float2 s[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s[e] = __fmul2_rn(h0[e], make_float2(wy[0], wy[0]));
      s[e] = __ffma2_rn(h1[e], make_float2(wy[1], wy[1]), s[e]);
      s[e] = __ffma2_rn(h2[e], make_float2(wy[2], wy[2]), s[e]);
      s[e] = __ffma2_rn(h3[e], make_float2(wy[3], wy[3]), s[e]);
    }
    *reinterpret_cast<uint4*>(ob + int64_t(y) * hw_in * c) = narrow2(s);
  }
}

// max-pool backward + the skip-connection gradient: ds = dskip + dp at the
// window's first maximum in scan order (torch's tie rule)
__global__ void __launch_bounds__(256) k_pool_bwd(const bf16* __restrict__ a, int a_tot, int a_off, int c,
                                                  int hw_out, int np, const bf16* __restrict__ dp,
                                                  const bf16* __restrict__ dskip, int ds_tot, int ds_off,
                                                  bf16* __restrict__ ds) {
  pdl_wait();
  const int lg = ilog2(c / 8), lho = ilog2(hw_out), hi = 2 * hw_out;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (np << (2 * lho + lg))) return;
  const int c0 = (i & ((1 << lg) - 1)) * 8;
  const int pp = i >> lg;
  const int px = pp & (hw_out - 1), py = (pp >> lho) & (hw_out - 1), m = pp >> (2 * lho);
  float v[4][8], dpv[8];
  int64_t q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    q[k] = (int64_t(m) * hi + 2 * py + (k >> 1)) * hi + 2 * px + (k & 1);
    ld8(a + q[k] * a_tot + a_off + c0, v[k]);
  }
  ld8(dp + int64_t(pp) * c + c0, dpv);
  int best[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    best[j] = 0;
#pragma unroll
    for (int k = 1; k < 4; ++k)
      if (v[k][j] > v[best[j]][j]) best[j] = k;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float d[8];
    ld8(dskip + q[k] * ds_tot + ds_off + c0, d);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (best[j] == k) d[j] += dpv[j];
    st8(ds + q[k] * c + c0, d);
  }
}

// LeakyReLU + BN backward, pass 1: per-channel sums of dyb and dyb * xhat
struct BnbStatsF {
  const bf16 *z, *da;
  const float* bnv;
  int cpad, pitch;  // bnv vector stride; elements between pixels
  float slope;
  float s[8], t[8], mu[8], is[8];
  __device__ __forceinline__ void init(int c0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j] = __ldg(bnv + c0 + j);
      t[j] = __ldg(bnv + cpad + c0 + j);
      mu[j] = __ldg(bnv + 2 * cpad + c0 + j);
      is[j] = __ldg(bnv + 3 * cpad + c0 + j);
    }
  }
  template <int U, int PS>
  __device__ __forceinline__ void go(int64_t p, int c0, float (&acc)[2][8]) const {
    float zv[U][8], dv[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ld8(z + (p + PS * u) * pitch + c0, zv[u]);
      ld8(da + (p + PS * u) * pitch + c0, dv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float y = fmaf(zv[u][j], s[j], t[j]);
        const float dyb = y > 0.f ? dv[u][j] : slope * dv[u][j];
        const float xh = (zv[u][j] - mu[j]) * is[j];
        acc[0][j] += dyb;
        acc[1][j] = fmaf(dyb, xh, acc[1][j]);
      }
  }
};
template <int CG>
__global__ void __launch_bounds__(256) k_bnb_stats(const bf16* __restrict__ z, const bf16* __restrict__ da,
                                                   int pitch, int cpad, int64_t npx,
                                                   const float* __restrict__ bnv, float slope,
                                                   double* part) {
  pdl_wait();
  chan_reduce<2, CG>(npx, 0, cpad, part, BnbStatsF{z, da, bnv, cpad, pitch, slope});
}


// pass 2: dz = gamma * invstd * (dyb - m1 - xhat * m2) (zero beyond n maps
// and in padded channels), plus per-block partial sums of dz (bias gradient)
// dz = coef * (dyb - m1 - xhat * m2) = coef * dyb + (k0 + k1 * z) with
// k1 = -coef * m2 * invstd, k0 = -coef * (m1 - m2 * mean * invstd): three
// FMAs per element from constants held in registers
struct BnbApplyF {
  const bf16 *z, *da;
  const float* bnv;
  bf16* dz;
  int64_t npx;      // real pixels (maps beyond n get dz = 0)
  int cpad, pitch;  // bnv vector stride; elements between pixels
  float slope;
  float s[8], t[8], cf[8], k0[8], k1[8];
  __device__ __forceinline__ void init(int c0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      s[j] = __ldg(bnv + c);
      t[j] = __ldg(bnv + cpad + c);
      const float mu = __ldg(bnv + 2 * cpad + c), is = __ldg(bnv + 3 * cpad + c);
      const float m1 = __ldg(bnv + 4 * cpad + c), m2 = __ldg(bnv + 5 * cpad + c);
      cf[j] = __ldg(bnv + 6 * cpad + c);
      k1[j] = -cf[j] * m2 * is;
      k0[j] = -cf[j] * (m1 - m2 * mu * is);
    }
  }
  template <int U, int PS>
  __device__ __forceinline__ void go(int64_t p, int c0, float (&acc)[1][8]) const {
    float zv[U][8], dv[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ld8s(z + (p + PS * u) * pitch + c0, zv[u]);
      ld8s(da + (p + PS * u) * pitch + c0, dv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float o[8];
      const bool real = p + PS * u < npx;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float y = fmaf(zv[u][j], s[j], t[j]);
        const float dyb = y > 0.f ? dv[u][j] : slope * dv[u][j];
        const float g = real ? fmaf(cf[j], dyb, fmaf(k1[j], zv[u][j], k0[j])) : 0.f;
        o[j] = g;
        acc[0][j] += g;
      }
      st8(dz + (p + PS * u) * pitch + c0, o);
    }
  }
};
template <int CG>
__global__ void __launch_bounds__(256) k_bnb_apply(const bf16* __restrict__ z, const bf16* __restrict__ da,
                                                   int pitch, int cpad, int64_t npx_all, int64_t npx,
                                                   const float* __restrict__ bnv,
                                                   float slope, bf16* __restrict__ dz, double* part) {
  pdl_wait();
  // high to low: starts on the stats pass's last (L2-resident) pixels and
  // ends on the low ones the dgrad reads first
  chan_reduce<1, CG>(npx_all, 1, cpad, part, BnbApplyF{z, da, bnv, dz, npx, cpad, pitch, slope});
}

// head: conv_out (1x1, 16 -> 3) + ReLU, L1 loss against y (n,3,32,32) fp32,
// d(pred) = sign / n_out through the ReLU, d(a15) = W^T d(pred) and the
// partials of loss (slot 0), d bias (1..3) and d W (4..51) per block
constexpr int HEAD_SLOTS = 52;
__global__ void __launch_bounds__(256) k_head(const bf16* __restrict__ a15, const float* __restrict__ w,
                                              const float* __restrict__ b, const float* __restrict__ y,
                                              int64_t n, int64_t np, double inv_n, bf16* __restrict__ da15,
                                              double* part, int pitch) {
  pdl_wait();
  float wl[48], bl[3];
#pragma unroll
  for (int i = 0; i < 48; ++i) wl[i] = w[i];
#pragma unroll
  for (int o = 0; o < 3; ++o) bl[o] = b[o];
  double acc[HEAD_SLOTS];
#pragma unroll
  for (int s = 0; s < HEAD_SLOTS; ++s) acc[s] = 0.0;
  const float ginv = float(inv_n);
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < np * 1024;
       p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = p / 1024;
    const int px = int(p % 1024);
    float a[16];
    {
      float t[8];
      ld8(a15 + p * pitch, t);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = t[j];
      ld8(a15 + p * pitch + 8, t);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[8 + j] = t[j];
    }
    float gpre[3] = {0.f, 0.f, 0.f};
    if (m < n) {
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        float s = bl[o];
#pragma unroll
        for (int c = 0; c < 16; ++c) s = fmaf(wl[o * 16 + c], a[c], s);
        const float pred = fmaxf(s, 0.f);
        const float d = pred - y[(m * 3 + o) * 1024 + px];
        acc[0] += fabs(double(d));
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        gpre[o] = pred > 0.f ? sg * ginv : 0.f;
        acc[1 + o] += gpre[o];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[4 + o * 16 + c] += double(gpre[o]) * a[c];
      }
    }
    float da[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        da[j] = wl[h * 8 + j] * gpre[0] + wl[16 + h * 8 + j] * gpre[1] + wl[32 + h * 8 + j] * gpre[2];
      st8(da15 + p * pitch + 8 * h, da);
    }
  }
  // block reduction of the 52 slots in a fixed order
  __shared__ double red[8][HEAD_SLOTS];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
  for (int s = 0; s < HEAD_SLOTS; ++s) {
    double v = acc[s];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][s] = v;
  }
  __syncthreads();
  if (threadIdx.x < HEAD_SLOTS) {
    double v = 0.0;
    for (int k = 0; k < int(blockDim.x / 32); ++k) v += red[k][threadIdx.x];
    part[int64_t(threadIdx.x) * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void k_head_out(const double* sums, float* gw, float* gb, double* loss) {
  pdl_wait();
  const int i = threadIdx.x;
  if (i == 0) *loss = sums[0];
  if (i < 3) gb[i] = float(sums[1 + i]);
  if (i < 48) gw[i] = float(sums[4 + i]);
}

// ---------------------------------------------------------------------------
struct Buf {
  bf16* p = nullptr;
  int c = 0, hw = 0;
};

enum BufId {
  X0, A0, C1, P1, A2, C2, P2, A4, C3, P3, A6, A7, A8, A9, A10, A11, A12, A13, A14, A15,
  DZ, DA15, DA14, DA13, DA12, DC1, DA11, DA10, DC2, DA9, DA8, DC3, DA7, DA6, DP3, DS3, DA4, DP2,
  DS2, DA2, DP1, DS1, DA0, NBUF
};

struct LayerPlan {
  int in;           // input buffer
  int out, off;     // BN output buffer and channel offset
  int pool;         // fused-pool destination or -1
  int up;           // upsample destination (concat buffer) after the layer, or -1
  int dA;           // gradient of the layer output (BN backward input)
  int din;          // dgrad destination or -1 (enc1.conv1)
};

struct TcEngine {
  int64_t cap = 0;  // maps the buffers hold (a multiple of 8)
  Buf B[NBUF];
  bf16* Z[16] = {};
  bf16 *wpf[16] = {}, *wpt[16] = {};
  bf16* w8 = nullptr;  // enc1.conv1 in the in8 kernel's layout
  float *ep_one_f[16] = {}, *ep_b[16] = {}, *ep_one_t[16] = {}, *ep_zero[16] = {};
  float* bnv[16] = {};  // per layer: s, t, mean, invstd, m1, m2, coef (7 x cout_pad)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  double *part = nullptr, *sums = nullptr, *loss = nullptr;
  int64_t last_n = 0;  // examples in the last step (the loss normaliser)
  std::vector<void*> allocs;
  ~TcEngine() {
    for (void* p : allocs) cudaFree(p);
  }
};

void tc_engine_destroy(TcEngine* e) { delete e; }

const LayerPlan PLAN[16] = {
    {X0, A0, 0, -1, -1, DA0, -1},      {A0, C1, 128, P1, -1, DS1, DA0},
    {P1, A2, 0, -1, -1, DA2, DP1},     {A2, C2, 256, P2, -1, DS2, DA2},
    {P2, A4, 0, -1, -1, DA4, DP2},     {A4, C3, 512, P3, -1, DS3, DA4},
    {P3, A6, 0, -1, -1, DA6, DP3},     {A6, A7, 0, -1, C3, DA7, DA6},
    {C3, A8, 0, -1, -1, DA8, DC3},     {A8, A9, 0, -1, C2, DA9, DA8},
    {C2, A10, 0, -1, -1, DA10, DC2},   {A10, A11, 0, -1, C1, DA11, DA10},
    {C1, A12, 0, -1, -1, DA12, DC1},   {A12, A13, 0, -1, -1, DA13, DA12},
    {A13, A14, 0, -1, -1, DA14, DA13}, {A14, A15, 0, -1, -1, DA15, DA14},
};

int engine_setup(DrcbTrainer* T, int64_t np, cudaStream_t st) {
  TcEngine* E = T->tc;
  if (E && E->cap >= np) return 0;
  if (E) {
    DRCB_CUDA(cudaStreamSynchronize(st));
    delete E;
  }
  E = T->tc = new TcEngine();
  E->cap = np;
  const int spec[NBUF][2] = {
      {8, 32}, {64, 32}, {192, 32}, {64, 16}, {128, 16}, {384, 16}, {128, 8}, {256, 8}, {768, 8},
      {256, 4}, {512, 4}, {512, 4}, {256, 8}, {256, 8}, {128, 16}, {128, 16}, {64, 32}, {64, 32},
      {32, 32}, {16, 32},  // A14, A15: the head's 32- / 16-channel layers stored at that width
      {64, 32},            // DZ: the largest cout_pad * hw^2 (64 * 1024)
      {16, 32}, {32, 32}, {64, 32}, {64, 32}, {192, 32}, {128, 16}, {128, 16}, {384, 16}, {256, 8},
      {256, 8}, {768, 8}, {512, 4}, {512, 4}, {256, 4}, {256, 8}, {256, 8}, {128, 8}, {128, 16},
      {128, 16}, {64, 16}, {64, 32}, {64, 32}};
  size_t total = 0;
  std::vector<size_t> off(NBUF + 16);
  for (int i = 0; i < NBUF; ++i) {
    off[i] = total;
    total += (size_t(np) * spec[i][1] * spec[i][1] * spec[i][0] * 2 + 1023) & ~size_t(1023);
  }
  for (int l = 0; l < 16; ++l) {
    const TL& t = T->L[l];
    off[NBUF + l] = total;
    total += (size_t(np) * t.hw * t.hw * zpitch(t.cout) * 2 + 1023) & ~size_t(1023);
  }
  void* base = nullptr;
  if (cudaMalloc(&base, total) != cudaSuccess) return fail(DRCB_ECUDA, "cudaMalloc tensor-core trainer activations");
  E->allocs.push_back(base);
  DRCB_CUDA(cudaMemsetAsync(base, 0, total, st));
  uint8_t* b = static_cast<uint8_t*>(base);
  for (int i = 0; i < NBUF; ++i) E->B[i] = Buf{reinterpret_cast<bf16*>(b + off[i]), spec[i][0], spec[i][1]};
  for (int l = 0; l < 16; ++l) E->Z[l] = reinterpret_cast<bf16*>(b + off[NBUF + l]);
  // weights, epilogue vectors, BN vectors
  size_t wb = 0;
  std::vector<size_t> wo;
  for (int l = 0; l < 16; ++l) {
    const TL& t = T->L[l];
    const size_t cinp = pad64(t.cin), coutp = pad64(t.cout);
    const size_t sz[7] = {coutp * 9 * cinp * 2, cinp * 9 * coutp * 2, coutp * 4, coutp * 4,
                          cinp * 4, cinp * 4, 7 * coutp * 4};
    for (size_t z : sz) {
      wo.push_back(wb);
      wb += (z + 255) & ~size_t(255);
    }
  }
  // wgrad split-K partials, reduction partials
  size_t wsb = 0;
  for (int l = 0; l < 16; ++l) {
    const TL& t = T->L[l];
    size_t q = 0;
    int rc = wgrad_bf16(nullptr, t.cin, pad64(E->B[PLAN[l].in].c), nullptr, t.cout, pad64(t.cout), t.hw,
                        np, nullptr, 0, nullptr, &q, st, 0, 0);
    if (rc) return rc;
    wsb = std::max(wsb, q);
  }
  const size_t w8_off = wb;
  wb += 64 * 128 * 2;
  const size_t ws_off = wb;
  wb += (wsb + 255) & ~size_t(255);
  const size_t part_off = wb;
  wb += size_t(2048) * 2 * 1024 * 8 + size_t(1024) * HEAD_SLOTS * 8;
  const size_t sums_off = wb;
  wb += 2 * 1024 * 8 + 64 * 8;
  void* wbase = nullptr;
  if (cudaMalloc(&wbase, wb) != cudaSuccess) return fail(DRCB_ECUDA, "cudaMalloc tensor-core trainer state");
  E->allocs.push_back(wbase);
  DRCB_CUDA(cudaMemsetAsync(wbase, 0, wb, st));
  uint8_t* w = static_cast<uint8_t*>(wbase);
  for (int l = 0; l < 16; ++l) {
    const TL& t = T->L[l];
    E->wpf[l] = reinterpret_cast<bf16*>(w + wo[7 * l]);
    E->wpt[l] = reinterpret_cast<bf16*>(w + wo[7 * l + 1]);
    E->ep_one_f[l] = reinterpret_cast<float*>(w + wo[7 * l + 2]);
    E->ep_b[l] = reinterpret_cast<float*>(w + wo[7 * l + 3]);
    E->ep_one_t[l] = reinterpret_cast<float*>(w + wo[7 * l + 4]);
    E->ep_zero[l] = reinterpret_cast<float*>(w + wo[7 * l + 5]);
    E->bnv[l] = reinterpret_cast<float*>(w + wo[7 * l + 6]);
    const int cinp = pad64(t.cin), coutp = pad64(t.cout);
    launch_pdl(k_pad_vec, nbk(coutp), 256, 0, st, nullptr, t.cout, coutp, 1.f, E->ep_one_f[l]);
    launch_pdl(k_pad_vec, nbk(cinp), 256, 0, st, nullptr, t.cin, cinp, 1.f, E->ep_one_t[l]);
  }
  E->w8 = reinterpret_cast<bf16*>(w + w8_off);
  E->ws = w + ws_off;
  E->ws_bytes = wsb;
  E->part = reinterpret_cast<double*>(w + part_off);
  E->sums = reinterpret_cast<double*>(w + sums_off);
  E->loss = E->sums + 2 * 1024;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "trainer engine setup");
}

// reduction geometry over npx pixels: pixels per block and blocks
// resident blocks per SM of a 256-thread reduction kernel on this device
inline int resident_blocks(const void* kern) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find({dev, kern});
  if (it != cache.end()) return it->second;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0) != cudaSuccess || b < 1) b = 1;
  cache[{dev, kern}] = b;
  return b;
}

// reduction grid over npx pixels (blocks per channel tile). With
// `kern` given, the grid is whole waves of that kernel's resident blocks
// (DRCB_RED_WAVES, default 1; 2 / 4 waves measured 0.1 / 0.4 ms slower per
// B = 4,096 step) instead of 8 blocks per SM: a partial last wave left SMs
// idle at the end of every pass.
inline int red_grid(int64_t npx, int ctiles, const void* kern = nullptr) {
  static const int waves = [] {
    const char* e = getenv("DRCB_RED_WAVES");
    return e ? atoi(e) : 1;
  }();
  const int per_sm = (kern && waves > 0) ? waves * resident_blocks(kern) : 8;
  const int64_t target = std::max<int64_t>(1, int64_t(sm_count()) * per_sm / ctiles);
  return int(std::min<int64_t>(target, std::max<int64_t>(1, (npx + 127) / 128)));
}

// N of a conv whose output has fewer than 64 real channels (head.deconv1 /
// deconv2 and their dgrads, 32x32): the row kernels compute N = channels
// rounded to 16 and zero-fill the rest of each 64-channel row (the padding
// the next layer's K reads), instead of multiplying zero weight rows
inline int narrow_n(int hw, int c, int c_pad) { return hw >= 16 && c < 64 ? (c + 15) / 16 * 16 : c_pad; }

// enc1.conv1 forward through the in8 kernel (DRCB_TRAIN_NO_IN8: the row
// kernel over a zero-filled 64-channel K block)
inline bool use_in8(const DrcbTrainer* T) {
  return T->L[0].cin <= 8 && T->L[0].cout == 64 && T->L[0].hw == 32 &&
         getenv("DRCB_TRAIN_NO_IN8") == nullptr;
}

// nothing to all-reduce: the SyncBN sums are already the batch's
inline bool one_rank(const DrcbTrainer* T) { return !T->reduce_fn && T->world == 1; }

// SyncBN sums. With the bucketed gradient all-reduce (NCCL, several ranks)
// every NCCL call of the step goes through comm_stream in host order: one
// communicator must see its collectives in the same order on every rank, and
// the device's order between two streams is not fixed. The compute stream
// forks into comm_stream and joins back (the BN statistics are on the
// critical path either way).
int syncbn_allreduce(DrcbTrainer* T, double* buf, size_t count, cudaStream_t st) {
  if (!T->comm_stream || !T->comm || T->reduce_fn || T->world <= 1)
    return trainer_allreduce(T, buf, count, 1, st);
  DRCB_CUDA(cudaEventRecord(T->sync_ev[0], st));
  DRCB_CUDA(cudaStreamWaitEvent(T->comm_stream, T->sync_ev[0], 0));
  int rc = allreduce_sum(T->comm, buf, count, 1, T->comm_stream);
  if (rc) return rc;
  DRCB_CUDA(cudaEventRecord(T->sync_ev[1], T->comm_stream));
  DRCB_CUDA(cudaStreamWaitEvent(st, T->sync_ev[1], 0));
  return 0;
}

int layer_fwd(DrcbTrainer* T, int l, int64_t n, int64_t np, cudaStream_t st) {
  TcEngine* E = T->tc;
  const TL& t = T->L[l];
  const LayerPlan& P = PLAN[l];
  const int coutp = pad64(t.cout), hw2 = t.hw * t.hw, zp = zpitch(t.cout);
  const Buf& in = E->B[P.in];
  // (K blocks of 64 channels; a narrow input is read at its own pitch;
  // enc1.conv1 through the in8 kernel: K = 72 instead of a 64-channel block
  // per tap of which 8 channels hold data)
  int rc = (l == 0 && use_in8(T))
               ? tc_conv_in8_bf16(np, in.p, E->Z[l], zp, E->w8, E->ep_one_f[l], E->ep_b[l], 1.0f, st)
               : tc_conv_bf16(t.cin, t.cout, t.hw, np, in.p, pad64(in.c), E->Z[l], zp, 0, E->wpf[l],
                              narrow_n(t.hw, t.cout, coutp), E->ep_one_f[l], E->ep_b[l], 1.0f, st,
                              in.c);
  if (rc) return rc;
  const int cg = chan_groups(t.cout);
  const int gx = red_grid(n * hw2, coutp / 64, reinterpret_cast<const void*>(k_bn_stats<8>));
  switch (cg) {
    case 2: launch_pdl(k_bn_stats<2>, dim3(gx, 1), 256, 0, st, E->Z[l], zp, coutp, n * hw2, E->part); break;
    case 4: launch_pdl(k_bn_stats<4>, dim3(gx, 1), 256, 0, st, E->Z[l], zp, coutp, n * hw2, E->part); break;
    default: launch_pdl(k_bn_stats<8>, dim3(gx, coutp / 64), 256, 0, st, E->Z[l], zp, coutp, n * hw2, E->part);
  }
  TC_CHECK("k_bn_stats");
  const BnFin fin{t.cout,           coutp,       double(n) * hw2 * T->world, T->params + t.g,
                  T->params + t.be, T->running + t.rm, T->running + t.rv,  E->bnv[l]};
  if (one_rank(T)) {
    launch_pdl(k_reduce_fin<BnFin>, nb_slots(t.cout), 256, 0, st, E->part, gx, t.cout, fin);
    TC_CHECK("k_reduce_fin");
  } else {
    launch_pdl(k_reduce_parts, nb_slots(2 * coutp), 256, 0, st, E->part, gx, 2 * coutp, E->sums, 0, 0,
               (float*)nullptr, (float*)nullptr);
    TC_CHECK("k_reduce_parts");
    rc = syncbn_allreduce(T, E->sums, size_t(2) * coutp, st);  // SyncBN
    if (rc) return rc;
    launch_pdl(k_fin<BnFin>, nbk(t.cout), 256, 0, st, E->sums, t.cout, fin);
    TC_CHECK("k_fin");
  }
  const Buf& out = E->B[P.out];
  if (P.pool >= 0) {
    const int64_t tot = np * (hw2 / 4) * (coutp / 8);
    launch_pdl(k_bn_apply_pool, nbk(tot), 256, 0, st, E->Z[l], coutp, t.hw, np, E->bnv[l], T->slope, out.p,
                                              out.c, P.off, E->B[P.pool].p);
    TC_CHECK("k_bn_apply_pool");
  } else {
    const int groups = cg < 8 ? cg : coutp / 8;
    const int64_t tot = np * hw2 * groups;
    launch_pdl(k_bn_apply, nbk(tot), 256, 0, st, E->Z[l], zp, coutp, int(np * hw2), E->bnv[l], T->slope, out.p,
                                         out.c, P.off, groups);
    TC_CHECK("k_bn_apply");
  }
  if (P.up >= 0) {
    const Buf& cat = E->B[P.up];
    const int64_t tot = np * hw2 * (coutp / 8);  // a 2x2 output block per thread
    launch_pdl(k_up_fwd, nbk(tot), 256, 0, st, out.p, coutp, t.hw, np, cat.p, cat.c);
    TC_CHECK("k_up_fwd");
  }
  return 0;
}

int layer_bwd(DrcbTrainer* T, int l, int64_t n, int64_t np, cudaStream_t st) {
  TcEngine* E = T->tc;
  const TL& t = T->L[l];
  const LayerPlan& P = PLAN[l];
  const int coutp = pad64(t.cout), hw2 = t.hw * t.hw, zp = zpitch(t.cout);
  const bf16* da = E->B[P.dA].p;
  const int cg = chan_groups(t.cout);
  const int gx = red_grid(n * hw2, coutp / 64, reinterpret_cast<const void*>(k_bnb_stats<8>));
  const dim3 gs(gx, cg < 8 ? 1 : coutp / 64);
  switch (cg) {
    case 2: launch_pdl(k_bnb_stats<2>, gs, 256, 0, st, E->Z[l], da, zp, coutp, n * hw2, E->bnv[l], T->slope, E->part); break;
    case 4: launch_pdl(k_bnb_stats<4>, gs, 256, 0, st, E->Z[l], da, zp, coutp, n * hw2, E->bnv[l], T->slope, E->part); break;
    default: launch_pdl(k_bnb_stats<8>, gs, 256, 0, st, E->Z[l], da, zp, coutp, n * hw2, E->bnv[l], T->slope, E->part);
  }
  TC_CHECK("k_bnb_stats");
  // (sums of dyb and dyb * xhat: the local beta and gamma gradients)
  BnbCoef coef{t.cout, coutp, double(n) * hw2 * T->world, T->params + t.g, E->bnv[l],
               T->grads + t.be, T->grads + t.g};
  int rc = 0;
  if (one_rank(T)) {
    launch_pdl(k_reduce_fin<BnbCoef>, nb_slots(coutp), 256, 0, st, E->part, gx, coutp, coef);
    TC_CHECK("k_reduce_fin");
  } else {
    launch_pdl(k_reduce_parts, nb_slots(2 * coutp), 256, 0, st, E->part, gx, 2 * coutp, E->sums, t.cout,
                                                        coutp, T->grads + t.be, T->grads + t.g);
    TC_CHECK("k_reduce_parts");
    rc = syncbn_allreduce(T, E->sums, size_t(2) * coutp, st);  // SyncBN backward
    if (rc) return rc;
    coef.dbeta = coef.dgamma = nullptr;  // (written above from the local sums)
    launch_pdl(k_fin<BnbCoef>, nbk(coutp), 256, 0, st, E->sums, coutp, coef);
    TC_CHECK("k_fin");
  }
  const int gx2 = red_grid(np * hw2, coutp / 64, reinterpret_cast<const void*>(k_bnb_apply<8>));
  bf16* dz = E->B[DZ].p;
  // (a narrow layer's dz is stored at its own width: its dgrad and wgrad
  // load it into 64-channel / narrow boxes through the TMA zero fill)
  const dim3 ga(gx2, cg < 8 ? 1 : coutp / 64);
  switch (cg) {
    case 2: launch_pdl(k_bnb_apply<2>, ga, 256, 0, st, E->Z[l], da, zp, coutp, np * hw2, n * hw2, E->bnv[l], T->slope, dz, E->part); break;
    case 4: launch_pdl(k_bnb_apply<4>, ga, 256, 0, st, E->Z[l], da, zp, coutp, np * hw2, n * hw2, E->bnv[l], T->slope, dz, E->part); break;
    default: launch_pdl(k_bnb_apply<8>, ga, 256, 0, st, E->Z[l], da, zp, coutp, np * hw2, n * hw2, E->bnv[l], T->slope, dz, E->part);
  }
  TC_CHECK("k_bnb_apply");
  launch_pdl(k_reduce_parts, nb_slots(t.cout), 256, 0, st, E->part, gx2, t.cout, E->sums, t.cout, 0,
             T->grads + t.b, (float*)nullptr);  // conv bias
  TC_CHECK("k_reduce_parts");
  // dgrad: the transposed conv of dz into the input-gradient buffer
  if (P.din >= 0) {
    const Buf& din = E->B[P.din];
    rc = tc_conv_bf16(t.cout, t.cin, t.hw, np, dz, coutp, din.p, din.c, 0, E->wpt[l],
                      narrow_n(t.hw, t.cin, din.c), E->ep_one_t[l], E->ep_zero[l], 1.0f, st, zp);
    if (rc) return rc;
  }
  // wgrad from the layer input and dz (both NHWC, straight from the buffers)
  const Buf& in = E->B[P.in];
  size_t wsb = E->ws_bytes;
  // (straight into the parameter layout of T->grads)
  return wgrad_bf16(in.p, t.cin, pad64(in.c), dz, t.cout, coutp, t.hw, np, T->grads + t.w,
                    t.deconv ? 1 : 0, E->ws, &wsb, st, in.c, zp);
}

int up_bwd(TcEngine* E, int dcat, int c, int hw_in, int dlow, int64_t np, cudaStream_t st) {
  const int64_t tot = np * hw_in * (c / 8);  // a column strip per thread
  launch_pdl(k_up_bwd, nbk(tot), 256, 0, st, E->B[dcat].p, E->B[dcat].c, c, hw_in, np, E->B[dlow].p);
  TC_CHECK("k_up_bwd");
  return 0;
}

int pool_bwd(TcEngine* E, int cat, int off, int c, int hw_out, int dp, int dcat, int ds, int64_t np,
             cudaStream_t st) {
  const int64_t tot = np * hw_out * hw_out * (c / 8);
  launch_pdl(k_pool_bwd, nbk(tot), 256, 0, st, E->B[cat].p, E->B[cat].c, off, c, hw_out, np, E->B[dp].p,
                                        E->B[dcat].p, E->B[dcat].c, off, E->B[ds].p);
  TC_CHECK("k_pool_bwd");
  return 0;
}

// One step's forward, L1 loss and backward (gradients of every parameter in
// T->grads, local to this rank); *loss_dev receives the device sum |pred - y|.
int tc_step(DrcbTrainer* T, const float* x, const float* y, int64_t n, double** loss_dev,
            cudaStream_t st) {
  if (T->k != 64) return fail(DRCB_ECONFIG, "the tensor-core trainer is built for k = 64");
  const int64_t np = (n + 7) / 8 * 8;
  int rc = engine_setup(T, np, st);
  if (rc) return rc;
  TcEngine* E = T->tc;
  E->last_n = n;
  // NCCL over several ranks: the side stream every collective of the step
  // goes through (bucketed gradients overlap the backward; SyncBN joins)
  if (T->comm && !T->reduce_fn && T->world > 1 && !T->comm_stream) {
    DRCB_CUDA(cudaStreamCreateWithFlags(&T->comm_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : T->comm_ev) DRCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (cudaEvent_t& e : T->sync_ev) DRCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // packed bf16 operands of this step's weights (forward and dgrad forms)
  {
    PrepArgs a;
    int64_t tot = 0;
    for (int l = 0; l < 16; ++l) {
      const TL& t = T->L[l];
      const int cinp = pad64(t.cin), coutp = pad64(t.cout);
      a.L[l] = PrepLayer{T->params + t.w, T->params + t.b, E->wpf[l], E->wpt[l], E->ep_b[l],
                         t.cin, t.cout, cinp, coutp, t.deconv ? 1 : 0};
      a.start[l] = tot;
      tot += 2 * int64_t(coutp) * cinp + coutp;
    }
    a.start[16] = tot;
    launch_pdl(k_prep_weights, nbk(tot), 256, 0, st, a);
    TC_CHECK("k_prep_weights");
    if (use_in8(T)) {
      const TL& t0 = T->L[0];
      launch_pdl(k_prep_in8, nbk(64 * 128), 256, 0, st, T->params + t0.w, t0.cin, t0.cout, E->w8);
      TC_CHECK("k_prep_in8");
    }
  }
  launch_pdl(k_x_in, nbk(np * 1024), 256, 0, st, x, n, np, E->B[X0].p);
  TC_CHECK("k_x_in");
  // ---- forward (model.py:80-88)
  for (int l = 0; l < 16 && !rc; ++l) rc = layer_fwd(T, l, n, np, st);
  if (rc) return rc;
  // ---- head.conv_out + ReLU + L1 loss (train.py:88) and its backward
  {
    const TL& t = T->L[16];
    const int gx = 1024;
    launch_pdl(k_head, gx, 256, 0, st, E->B[A15].p, T->params + t.w, T->params + t.b, y, n, np,
                               1.0 / double(n * 3 * 1024), E->B[DA15].p, E->part, E->B[A15].c);
    TC_CHECK("k_head");
    launch_pdl(k_reduce_parts, nb_slots(HEAD_SLOTS), 256, 0, st, E->part, gx, HEAD_SLOTS, E->sums, 0, 0,
               (float*)nullptr, (float*)nullptr);
    TC_CHECK("k_reduce_parts");
    launch_pdl(k_head_out, 1, 64, 0, st, E->sums, T->grads + t.w, T->grads + t.b, E->loss);
    TC_CHECK("k_head_out");
  }
  // ---- backward
  // NCCL (world > 1): each layer's gradients are all-reduced on a side stream
  // as soon as its backward is done (buckets = layers, in backward order),
  // overlapping the all-reduce with the remaining layers' backward
  const bool bucket = T->comm && !T->reduce_fn && T->world > 1;
  int nev = 0;
  auto reduce_layer = [&](int l) -> int {
    if (!bucket) return 0;
    int64_t off, cnt;
    layer_param_range(T, l, off, cnt);
    DRCB_CUDA(cudaEventRecord(T->comm_ev[nev], st));
    DRCB_CUDA(cudaStreamWaitEvent(T->comm_stream, T->comm_ev[nev], 0));
    ++nev;
    return allreduce_sum(T->comm, T->grads + off, size_t(cnt), 0, T->comm_stream);
  };
  rc = reduce_layer(16);  // the head (its gradients came with the loss)
  if (rc) return rc;
  const int order[] = {15, 14, 13, 12, -1, 11, 10, -2, 9, 8, -3, 7, 6, -4, 5, 4, -5, 3, 2, -6, 1, 0};
  for (int o : order) {
    if (o >= 0) {
      rc = layer_bwd(T, o, n, np, st);
      if (!rc) rc = reduce_layer(o);
    }
    else if (o == -1) rc = up_bwd(E, DC1, 128, 16, DA11, np, st);
    else if (o == -2) rc = up_bwd(E, DC2, 256, 8, DA9, np, st);
    else if (o == -3) rc = up_bwd(E, DC3, 512, 4, DA7, np, st);
    else if (o == -4) rc = pool_bwd(E, C3, 512, 256, 4, DP3, DC3, DS3, np, st);
    else if (o == -5) rc = pool_bwd(E, C2, 256, 128, 8, DP2, DC2, DS2, np, st);
    else rc = pool_bwd(E, C1, 128, 64, 16, DP1, DC1, DS1, np, st);
    if (rc) return rc;
  }
  if (bucket) {  // the step's stream waits for the last bucket
    DRCB_CUDA(cudaEventRecord(T->comm_ev[nev], T->comm_stream));
    DRCB_CUDA(cudaStreamWaitEvent(st, T->comm_ev[nev], 0));
  }
  *loss_dev = E->loss;
  return 0;
}

}  // namespace train
}  // namespace drcb

// The batch L1 loss of the last tensor-core step (device sum / n*3*1024),
// read on `stream` (synchronises): the loss of a replayed step graph.
extern "C" int drcb_trainer_last_loss(DrcbTrainer* T, double* loss, void* stream) {
  using namespace drcb;
  if (!T || !loss) return fail(DRCB_ECONTRACT, "drcb_trainer_last_loss: null argument");
  if (!T->tc || T->tc->last_n < 1)
    return fail(DRCB_ECONFIG, "drcb_trainer_last_loss: no tensor-core step has run");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double s = 0;
  DRCB_CUDA(cudaMemcpyAsync(&s, T->tc->loss, sizeof(double), cudaMemcpyDeviceToHost, st));
  DRCB_CUDA(cudaStreamSynchronize(st));
  *loss = s / double(T->tc->last_n * 3 * 1024);
  return 0;
}

// Test hook: the bf16 pre-BN conv output Z of layer `layer` (0..15) from the
// last tensor-core step, NHWC (capacity maps, hw, hw, pad64(cout)) -> dst.
extern "C" int drcb_trainer_debug_z(DrcbTrainer* T, int32_t layer, void* dst, void* stream) {
  using namespace drcb;
  using namespace drcb::train;
  if (!T || !dst || layer < 0 || layer > 16) return fail(DRCB_ECONTRACT, "drcb_trainer_debug_z: bad arguments");
  if (!T->tc) return fail(DRCB_ECONTRACT, "drcb_trainer_debug_z: no tensor-core step has run");
  // (the tensor unpacked into 64-channel padded rows, zeros in the padding)
  const bool head = layer == 16;
  const TL& t = T->L[head ? 15 : layer];
  const int cp = pad64(t.cout), zp = zpitch(t.cout);
  const size_t rows = size_t(T->tc->cap) * t.hw * t.hw;
  const void* src = head ? static_cast<const void*>(T->tc->B[A15].p) : T->tc->Z[layer];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (zp < cp) DRCB_CUDA(cudaMemsetAsync(dst, 0, rows * cp * 2, s));
  DRCB_CUDA(cudaMemcpy2DAsync(dst, size_t(cp) * 2, src, size_t(zp) * 2, size_t(zp) * 2, rows,
                              cudaMemcpyDeviceToDevice, s));
  return 0;
}
