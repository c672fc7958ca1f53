// drcb_wgrad.cu — the convolutions' weight gradient on the 5th-generation
// tensor cores (the training step's wgrad, trainer train.py:97-103 /
// MapAutoencoder model.py:20-88 backward).
//
// For a 3x3 layer with NHWC bf16 input X (Cin_pad channels) and NHWC bf16
// output gradient dZ (Cout_pad channels):
//
//   dW_tap[co][ci] = sum_p dZ[p][co] * X[p + (dy, dx)][ci]     (zero outside)
//
// is a GEMM whose reduction (K) runs over all pixels of the batch. Both
// operands are read straight from the NHWC activations as MN-major UMMA
// operands: a TMA box of 64 channels (128 B) x 128 pixels lands in SMEM in
// the 128B-swizzle layout with one pixel per 128-B row, which IS the
// canonical MN-major SW128 layout (64 MN elements per row, K down the rows).
// The tap shift (dy, dx) is the X box's coordinate offset; the TMA unit's
// out-of-bounds zero fill is the conv's zero padding (no im2col, no padded
// copies, no transposes).
//
// M tile (128 rows) = two (tap, 64-channel input block) blocks: the same tap
// over 128 input channels, or two taps of a 64-channel input. N tile = up to
// 256 output channels (dZ boxes). Each CTA owns `n_acc` accumulators (one
// M x N TMEM tile each, n_acc * N <= 512 columns) and a contiguous range of
// K chunks (split-K); per chunk it loads the dZ boxes once and every
// accumulator's X boxes, and issues 8 MMAs (K = 16 each) per accumulator.
// Split-K partials go to global memory and are summed in a fixed order by a
// second kernel: the result is deterministic.
//
//   warp 0: TMA producer     warp 1: MMA issuer (one thread)
//   warps 2-5: epilogue (tcgen05.ld -> fp32 partial tiles)
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "drcb_net.h"
#include "drcb_tc_ptx.cuh"

namespace drcb {
namespace tc {
int encode_act(CUtensorMap* m, const void* base, int kind, int c_tot, int hw, int64_t nmaps,
               int box_w, int box_h, int box_n, int c_dim = 0, int pitch = 0);
int encode_act_c(CUtensorMap* m, const void* base, int kind, int c_tot, int hw, int64_t nmaps,
                 int box_c, int box_w, int box_h, int box_n, int pitch = 0);
}  // namespace tc

namespace wg {
using namespace tc;

constexpr int THREADS = 192;
constexpr int BOX = 64 * 128 * 2;  // one 64-channel x 128-pixel bf16 box (16 KB)
constexpr int KPX = 128;           // pixels per K chunk

struct WgArgs {
  int hw;                 // map side
  int cb;                 // input channel blocks of 64 (Cin_pad / 64)
  int n_tile;             // N (output channels per tile, multiple of 64, <= 256)
  int nb_n;               // dZ boxes per stage (n_tile / 64)
  int n_acc;              // accumulators per CTA
  int npairs;             // M tiles: ceil(9 * cb / 2)
  int groups;             // ceil(npairs / n_acc)
  int units;              // n_tiles * groups
  int splits;             // K splits
  int chunks;             // K chunks of 128 pixels over the batch
  int rb, mb, cpm;        // box rows, box maps, chunks per map (hw >= 16)
  int dz_stages, x_stages;
  float* partial;         // [splits][units][n_acc][128][n_tile]
  // dx-in-N variant (hw >= 16)
  int xbox;               // bytes of the X box (rb + 2 rows)
  int zero_off;           // byte offset of the zero block from the SMEM base
};

__device__ __forceinline__ void chunk_origin(const WgArgs& a, int c, int& map0, int& row0) {
  if (a.hw >= 16) {
    map0 = c / a.cpm;
    row0 = (c % a.cpm) * a.rb;
  } else {
    map0 = c * a.mb;
    row0 = 0;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    k_wgrad(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapDZ,
            const __grid_constant__ WgArgs a) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int DZB = a.nb_n * BOX;  // one dZ stage
  uint8_t* dzring = smem;
  uint8_t* xring = smem + a.dz_stages * DZB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xring + a.x_stages * 2 * BOX);
  uint64_t* dzfull = bars;
  uint64_t* dzempty = bars + 4;
  uint64_t* xfull = bars + 8;
  uint64_t* xempty = bars + 16;
  uint64_t* tfull = bars + 24;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  const int unit = int(blockIdx.x) % a.units, split = int(blockIdx.x) / a.units;
  const int nt = unit / a.groups, g = unit % a.groups;
  const int c0 = int(int64_t(a.chunks) * split / a.splits);
  const int c1 = int(int64_t(a.chunks) * (split + 1) / a.splits);
  const int a0 = g * a.n_acc;
  const int nacc = min(a.n_acc, a.npairs - a0);
  const uint32_t cols = uint32_t(a.n_acc * a.n_tile);
  const uint32_t tcols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapX);
    prefetch_map(&mapDZ);
    for (int s = 0; s < a.dz_stages; ++s) {
      mbar_init(&dzfull[s], 1);
      mbar_init(&dzempty[s], 1);
    }
    for (int s = 0; s < a.x_stages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int ds = 0, xs = 0;
      uint32_t dp = 0, xp = 0;
      for (int c = c0; c < c1; ++c) {
        int map0, row0;
        chunk_origin(a, c, map0, row0);
        mbar_wait(&dzempty[ds], dp ^ 1);
        mbar_expect_tx(&dzfull[ds], uint32_t(DZB));
        for (int j = 0; j < a.nb_n; ++j)
          tma_load_4d(&mapDZ, &dzfull[ds], dzring + ds * DZB + j * BOX, nt * a.n_tile + 64 * j, 0, row0,
                      map0);
        if (++ds == a.dz_stages) {
          ds = 0;
          dp ^= 1;
        }
        for (int j = 0; j < nacc; ++j) {
          mbar_wait(&xempty[xs], xp ^ 1);
          mbar_expect_tx(&xfull[xs], uint32_t(2 * BOX));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int b = 2 * (a0 + j) + h;  // (tap, channel block)
            int cx = 0, x = 0, y = -4 * a.hw;  // an absent block: the box lies outside -> zeros
            if (b < 9 * a.cb) {
              const int tap = b / a.cb, cblk = b % a.cb;
              cx = 64 * cblk;
              x = tap % 3 - 1;
              y = row0 + tap / 3 - 1;
            }
            tma_load_4d(&mapX, &xfull[xs], xring + (xs * 2 + h) * BOX, cx, x, y, map0);
          }
          if (++xs == a.x_stages) {
            xs = 0;
            xp ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_mn(0, 128, a.n_tile);
      int ds = 0, xs = 0;
      uint32_t dp = 0, xp = 0;
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&dzfull[ds], dp);
        tc_fence_after();
        const uint32_t bz = smem_u32(dzring + ds * DZB);
        for (int j = 0; j < nacc; ++j) {
          mbar_wait(&xfull[xs], xp);
          tc_fence_after();
          const uint32_t ax = smem_u32(xring + xs * 2 * BOX);
#pragma unroll
          for (int k = 0; k < KPX / 16; ++k)
            tc_mma<0>(tmem_base + uint32_t(j * a.n_tile), mn128_desc(ax + k * 2048, BOX, 1024),
                      mn128_desc(bz + k * 2048, BOX, 1024), idesc, (c > c0 || k > 0) ? 1u : 0u);
          tc_commit(&xempty[xs]);
          if (++xs == a.x_stages) {
            xs = 0;
            xp ^= 1;
          }
        }
        tc_commit(&dzempty[ds]);
        if (++ds == a.dz_stages) {
          ds = 0;
          dp ^= 1;
        }
      }
      tc_commit(tfull);
    }
  } else {
    // epilogue: lane quarter q of the accumulators (rows 32q .. 32q+31)
    const int q = warp & 3, row = q * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    float* out = a.partial + (int64_t(split) * a.units + unit) * a.n_acc * 128 * a.n_tile;
    for (int j = 0; j < a.n_acc; ++j) {
      float* o = out + (int64_t(j) * 128 + row) * a.n_tile;
      for (int c = 0; c < a.n_tile; c += 16) {
        float v[16];
        if (j < nacc && c1 > c0) {
          uint32_t r[16];
          tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(j * a.n_tile + c), r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(o + c + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
  }
}

// dx-in-N variant (hw in {16, 32}: an image row is a whole number of
// 1024-B swizzle atoms). With the identity
//   dW_(dy,dx) = sum_q X[q + (dy, 0)] * dZ[q - (0, dx)]
// (exact: the terms it adds or drops have X or dZ out of the map = zero),
// a K chunk of rb image rows needs ONE X box of rb + 2 rows (the dy shift
// is a row offset inside it) and three dZ boxes shifted by dx = -1, 0, +1
// (TMA zero fill at the row ends). Two MMAs per K step cover the nine taps:
//   acc 0: M = [X(dy=-1) | X(dy=0)] (two 64-channel blocks, LBO = one row)
//          x N = [dZ(dx=-1) | dZ(0) | dZ(+1)] = 192 columns: six taps,
//   acc 1: M = [X(dy=+1) | zero block] x the same N: three taps.
// N = 192 per MMA (the small-N layers' 64-column MMAs ran at ~45 % of the
// tensor rate). A CTA owns one 64-channel input block x one 64-channel
// output block and a range of K chunks.
// NB = output channels per dZ box: 64 (128-B swizzled rows), or 32 / 16 for
// layers with fewer outputs (head.deconv1 / deconv2: N = 96 / 48 instead of
// multiplying 64-channel boxes that are mostly zero padding)
template <int NB>
__global__ void __launch_bounds__(THREADS, 1)
    k_wgrad_dxn(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapDZ,
                const __grid_constant__ WgArgs a) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int W = NB * 2;          // dZ row bytes (one pixel)
  constexpr int BOXZ = W * KPX;      // one dZ box
  const int STB = 3 * BOXZ + a.xbox;  // one stage: dZ boxes (dx = -1, 0, +1), then the X box
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.zero_off + BOX);
  uint64_t* full = bars;
  uint64_t* empty = bars + 4;
  uint64_t* tfull = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  const int unit = int(blockIdx.x) % a.units, split = int(blockIdx.x) / a.units;
  const int cob = unit / a.cb, cb = unit % a.cb;  // output / input channel blocks of 64
  const int c0 = int(int64_t(a.chunks) * split / a.splits);
  const int c1 = int(int64_t(a.chunks) * (split + 1) / a.splits);
  constexpr uint32_t NCOL = 3 * NB, TCOLS = 512;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapX);
    prefetch_map(&mapDZ);
    for (int s = 0; s < a.dz_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp >= 2) {  // the zero block (the M partner of the dy = +1 block)
    uint4* z = reinterpret_cast<uint4*>(smem + a.zero_off);
    for (int i = threadIdx.x - 64; i < BOX / 16; i += THREADS - 64) z[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int rowb = a.hw * 128;  // one image row of 64 channels
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int c = c0; c < c1; ++c) {
        const int map0 = c / a.cpm, row0 = (c % a.cpm) * a.rb;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], uint32_t(STB));
        uint8_t* st = smem + s * STB;
        for (int j = 0; j < 3; ++j)  // dZ[q - (0, dx)], dx = j - 1: box at x = 1 - j
          tma_load_4d(&mapDZ, &full[s], st + j * BOXZ, NB * cob, 1 - j, row0, map0);
        tma_load_4d(&mapX, &full[s], st + 3 * BOXZ, 64 * cb, 0, row0 - 1, map0);
        if (++s == a.dz_stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_mn(0, 128, NCOL);
      const uint32_t zero = smem_u32(smem + a.zero_off);
      int s = 0;
      uint32_t ph = 0;
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t bz = smem_u32(smem + s * STB);
        const uint32_t xs = bz + 3 * BOXZ;
        const uint32_t acc_flag = c > c0 ? 1u : 0u;
#pragma unroll
        for (int k = 0; k < KPX / 16; ++k) {
          const uint64_t bd = mn_desc(bz + k * 16 * W, BOXZ, 8 * W, W);
          // rows dy = -1, 0 of the X box: offsets 0, one row
          tc_mma<0>(tmem_base, mn128_desc(xs + k * 2048, rowb, 1024), bd, idesc, (acc_flag | k) ? 1u : 0u);
          // dy = +1 (offset two rows) and the zero block
          const uint32_t a1 = xs + 2 * rowb + k * 2048;
          tc_mma<0>(tmem_base + NCOL, mn128_desc(a1, zero - (xs + 2 * rowb), 1024), bd, idesc,
                    (acc_flag | k) ? 1u : 0u);
        }
        tc_commit(&empty[s]);
        if (++s == a.dz_stages) {
          s = 0;
          ph ^= 1;
        }
      }
      tc_commit(tfull);
    }
  } else {
    const int q = warp & 3, row = q * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    float* out = a.partial + (int64_t(split) * a.units + unit) * 2 * 128 * NCOL;
    for (int j = 0; j < 2; ++j) {
      float* o = out + (int64_t(j) * 128 + row) * NCOL;
      for (int c = 0; c < int(NCOL); c += 16) {
        float v[16];
        if (c1 > c0) {
          uint32_t r[16];
          tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(j * NCOL + c), r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(o + c + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TCOLS));
  }
}

// the split-K partials of one output element summed in split order (fixed:
// deterministic); eight loads in flight ahead of the adds (the reductions
// were latency-bound with one dependent load per split: 842 -> ~250 us per
// B = 4,096 step), the same additions in the same order
__device__ __forceinline__ float sum_splits(const float* __restrict__ p, int64_t stride, int splits) {
  float s = 0.f;
  int k = 0;
  for (; k + 8 <= splits; k += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + (k + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; k < splits; ++k) s += __ldcs(p + k * stride);
  return s;
}

// the output element (co, ci, tap): conv form dwf[co][ci][tap], or with
// `deconv` the ConvTranspose2d parameter layout w[ci][co][8 - tap] (the
// transposed, flipped conv form; model.py:33-34)
__device__ __forceinline__ int64_t wg_out(int co, int ci, int tap, int cin, int cout, int deconv) {
  return deconv ? (int64_t(ci) * cout + co) * 9 + (8 - tap) : (int64_t(co) * cin + ci) * 9 + tap;
}

// dx-in-N partials -> dwf: unit (output block, input block), acc j, row m
// (dy of the X block: acc 0 rows -1 / 0, acc 1 row +1), column n (dx, co)
__global__ void k_wgrad_reduce_dxn(const WgArgs a, int nb, int cin, int cout, int deconv,
                                   float* __restrict__ dwf) {
  pdl_wait();
  const int ncol = 3 * nb;
  const int64_t per = int64_t(2) * 128 * ncol;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= per * a.units) return;
  const int unit = int(e / per);
  int64_t r = e % per;
  const int n = int(r % ncol);
  r /= ncol;
  const int m = int(r % 128), j = int(r / 128);
  if (j == 1 && m >= 64) return;  // the zero block
  const int dy = j == 0 ? (m < 64 ? -1 : 0) : 1, dx = n / nb - 1;
  const int cob = unit / a.cb, cb = unit % a.cb;
  const int ci = 64 * cb + (m & 63), co = nb * cob + n % nb;
  if (ci >= cin || co >= cout) return;
  const int64_t stride = int64_t(a.units) * per;
  const float* p = a.partial + int64_t(unit) * per + (int64_t(j) * 128 + m) * ncol + n;
  dwf[wg_out(co, ci, (dy + 1) * 3 + (dx + 1), cin, cout, deconv)] = sum_splits(p, stride, a.splits);
}

// split-K partials -> conv-form fp32 weight gradient dwf[co][ci][tap], summed
// over the splits in order (deterministic). One thread per (n tile, M tile,
// row, column) accumulator element.
__global__ void k_wgrad_reduce(const WgArgs a, int cin, int cout, int deconv, float* __restrict__ dwf) {
  pdl_wait();
  const int64_t per_nt = int64_t(a.npairs) * 128 * a.n_tile;
  const int64_t total = per_nt * (int64_t(a.units) / a.groups);
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int nt = int(e / per_nt);
  int64_t r = e % per_nt;
  const int n = int(r % a.n_tile);
  r /= a.n_tile;
  const int m = int(r % 128);
  const int pair = int(r / 128);
  const int b = 2 * pair + (m >> 6);
  if (b >= 9 * a.cb) return;
  const int tap = b / a.cb, ci = 64 * (b % a.cb) + (m & 63), co = nt * a.n_tile + n;
  if (ci >= cin || co >= cout) return;
  const int unit = nt * a.groups + pair / a.n_acc, j = pair % a.n_acc;
  const int64_t stride = int64_t(a.units) * a.n_acc * 128 * a.n_tile;
  const float* p = a.partial + ((int64_t(unit) * a.n_acc + j) * 128 + m) * a.n_tile + n;
  dwf[wg_out(co, ci, tap, cin, cout, deconv)] = sum_splits(p, stride, a.splits);
}

}  // namespace wg

// Plan + launch the weight gradient of one 3x3 layer. x: NHWC bf16 (nmaps,
// hw, hw, cin_pad); dz: NHWC bf16 (nmaps, hw, hw, cout_pad); dwf: conv-form
// fp32 (cout, cin, 3, 3), or with `deconv` the transposed conv's parameter
// layout (cin, cout, 3, 3) flipped. `ws` / `ws_bytes`: scratch for the
// split-K partials (query with ws == nullptr: ws_bytes receives the size).
// x_pitch / dz_pitch (0 = cin_pad / cout_pad): elements between pixels of a
// tensor stored narrower than its 64-channel blocks (the missing channels
// load as zeros)
int wgrad_bf16(const void* x, int cin, int cin_pad, const void* dz, int cout, int cout_pad, int hw,
               int64_t nmaps, float* dwf, int deconv, void* ws, size_t* ws_bytes, cudaStream_t st,
               int x_pitch, int dz_pitch) {
  using namespace wg;
  if (cin_pad % 64 || cout_pad % 64 || (hw != 4 && hw != 8 && hw != 16 && hw != 32))
    return fail(DRCB_ECONFIG, "wgrad: channels must be padded to 64, hw in {4, 8, 16, 32}");
  WgArgs a;
  std::memset(&a, 0, sizeof(a));
  a.hw = hw;
  a.cb = cin_pad / 64;
  a.n_tile = cout_pad >= 256 ? 256 : cout_pad;
  while (cout_pad % a.n_tile) a.n_tile -= 64;
  a.nb_n = a.n_tile / 64;
  const bool taps_env = getenv("DRCB_WGRAD_TAPS") != nullptr;  // A/B: a box per tap
  const bool dxn = hw >= 16 && !taps_env;
  // dZ box width: the real output channels when there are fewer than 64
  static const bool no_narrow = getenv("DRCB_WGRAD_NO_NARROW") != nullptr;
  const int nb = (dxn && !no_narrow && cout <= 16) ? 16 : (dxn && !no_narrow && cout <= 32) ? 32 : 64;
  if (dxn) {
    a.units = ((cout + nb - 1) / nb) * a.cb;
  } else {
    a.npairs = (9 * a.cb + 1) / 2;
    a.n_acc = std::min(a.npairs, 512 / a.n_tile);
    a.groups = (a.npairs + a.n_acc - 1) / a.n_acc;
    a.units = (cout_pad / a.n_tile) * a.groups;
  }
  const int px_map = hw * hw;
  if (hw >= 16) {
    a.rb = KPX / hw;
    a.mb = 1;
    a.cpm = hw / a.rb;
    a.chunks = int(nmaps * a.cpm);
  } else {
    a.rb = hw;
    a.mb = KPX / px_map;
    a.cpm = 0;
    if (nmaps % a.mb) return fail(DRCB_ECONTRACT, "wgrad: batch must fill whole K chunks");
    a.chunks = int(nmaps / a.mb);
  }
  const int nsm = sm_count();
  // split-K over the pixel chunks: two CTAs per SM, but at least
  // `min_chunks` chunks per split (small batches: fewer, longer splits beat
  // a partial buffer the reduction then has to stream)
  static const int min_chunks = [] {
    const char* e = getenv("DRCB_WGRAD_MINCHUNKS");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  // Both kernels hold one CTA per SM (their SMEM plans): the grid runs in
  // waves of nsm CTAs, so the split count is chosen for the fewest waves per
  // unit of work, ceil(units * s / nsm) / s, over s up to two waves' worth
  // (the old rounding, ceil(2 nsm / units) splits, left a one-CTA third wave
  // for 297 = 2 x 148 + 1 CTAs: dec1.deconv1 with 3 units, dec3.deconv1 27)
  const int s_chunks = std::max(1, (a.chunks + min_chunks - 1) / min_chunks);
  static const bool old_splits = getenv("DRCB_WGRAD_OLD_SPLITS") != nullptr;
  if (old_splits) {
    a.splits = std::max(1, std::min(s_chunks, (2 * nsm + a.units - 1) / a.units));
  } else {
    const int s_max = std::max(1, std::min(s_chunks, (2 * nsm + a.units - 1) / a.units));
    int best = 1;
    double best_cost = 1e30;
    for (int sp = 1; sp <= s_max; ++sp) {
      const double cost = double((int64_t(a.units) * sp + nsm - 1) / nsm) / sp;
      if (cost < best_cost * (1.0 - 1e-9)) {
        best_cost = cost;
        best = sp;
      }
    }
    a.splits = best;
  }
  const size_t part = dxn ? size_t(a.splits) * a.units * 2 * 128 * (3 * nb) * 4
                          : size_t(a.splits) * a.units * a.n_acc * 128 * a.n_tile * 4;
  if (!ws) {
    *ws_bytes = part;
    return 0;
  }
  if (*ws_bytes < part) return fail(DRCB_ECONTRACT, "wgrad: scratch too small");
  a.partial = static_cast<float*>(ws);
  const int DZB = a.nb_n * BOX;
  static DeviceFlags attr_dxn[3];
  if (dxn) {
    a.xbox = (a.rb + 2) * hw * 128;
    const int stb = 3 * (nb * 2 * KPX) + a.xbox;
    a.dz_stages = std::min(4, (222 * 1024 - BOX) / stb);
    if (a.dz_stages < 2) return fail(DRCB_ECONFIG, "wgrad dx-in-N: SMEM plan");
    a.zero_off = a.dz_stages * stb;
    const size_t smem = 1024 + size_t(a.zero_off) + BOX + 256;
    CUtensorMap mX, mDZ;
    int rc = tc::encode_act(&mX, x, 0, cin_pad, hw, nmaps, hw, a.rb + 2, 1, 0, x_pitch);
    if (rc) return rc;
    rc = tc::encode_act_c(&mDZ, dz, 0, cout_pad, hw, nmaps, nb, hw, a.rb, 1, dz_pitch);
    if (rc) return rc;
    const unsigned grid = unsigned(a.units * a.splits);
    if (nb == 16) {
      smem_attr_once(attr_dxn[0], k_wgrad_dxn<16>, 227 * 1024);
      launch_pdl(k_wgrad_dxn<16>, grid, THREADS, smem, st, mX, mDZ, a);
    } else if (nb == 32) {
      smem_attr_once(attr_dxn[1], k_wgrad_dxn<32>, 227 * 1024);
      launch_pdl(k_wgrad_dxn<32>, grid, THREADS, smem, st, mX, mDZ, a);
    } else {
      smem_attr_once(attr_dxn[2], k_wgrad_dxn<64>, 227 * 1024);
      launch_pdl(k_wgrad_dxn<64>, grid, THREADS, smem, st, mX, mDZ, a);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_wgrad_dxn");
    const int64_t total = int64_t(2) * 128 * (3 * nb) * a.units;
    launch_pdl(k_wgrad_reduce_dxn, unsigned((total + 255) / 256), 256, 0, st, a, nb, cin, cout, deconv, dwf);
    count_launch();
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : cuda_fail(e, "k_wgrad_reduce_dxn");
  }
  a.dz_stages = 2;
  const int budget = 220 * 1024;
  a.x_stages = std::min(8, (budget - a.dz_stages * DZB) / (2 * BOX));
  if (a.x_stages < 2) return fail(DRCB_ECONFIG, "wgrad: SMEM plan");
  const size_t smem = 1024 + size_t(a.dz_stages) * DZB + size_t(a.x_stages) * 2 * BOX + 256;
  CUtensorMap mX, mDZ;
  const int bw = hw, bh = a.rb, bn = a.mb;
  int rc = tc::encode_act(&mX, x, 0, cin_pad, hw, nmaps, bw, bh, bn, 0, x_pitch);
  if (rc) return rc;
  rc = tc::encode_act(&mDZ, dz, 0, cout_pad, hw, nmaps, bw, bh, bn, 0, dz_pitch);
  if (rc) return rc;
  static DeviceFlags attr;
  smem_attr_once(attr, k_wgrad, 227 * 1024);
  launch_pdl(k_wgrad, a.units * a.splits, THREADS, smem, st, mX, mDZ, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_wgrad");
  const int64_t total = int64_t(a.npairs) * 128 * a.n_tile * (cout_pad / a.n_tile);
  launch_pdl(k_wgrad_reduce, unsigned((total + 255) / 256), 256, 0, st, a, cin, cout, deconv, dwf);
  count_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_wgrad_reduce");
}

}  // namespace drcb

// ---------------------------------------------------------------------------
// single-layer harness (tests only): host arrays, x (n,hw,hw,cin) NHWC,
// dz (n,hw,hw,cout) NHWC (rounded to bf16 here), dw (cout,cin,3,3) fp32
extern "C" int drcb_debug_wgrad(int32_t cin, int32_t cout, int32_t hw, int64_t n, const float* x,
                                const float* dz, float* dw) {
  using namespace drcb;
  const int cinp = (cin + 63) / 64 * 64, coutp = (cout + 63) / 64 * 64;
  const size_t px = size_t(n) * hw * hw;
  std::vector<__nv_bfloat16> hx(px * cinp, __float2bfloat16(0.f)), hz(px * coutp, __float2bfloat16(0.f));
  for (size_t i = 0; i < px; ++i) {
    for (int c = 0; c < cin; ++c) hx[i * cinp + c] = __float2bfloat16(x[i * cin + c]);
    for (int c = 0; c < cout; ++c) hz[i * coutp + c] = __float2bfloat16(dz[i * cout + c]);
  }
  void *dx = nullptr, *dd = nullptr, *ws = nullptr;
  float* dwf = nullptr;
  DRCB_CUDA(cudaMalloc(&dx, hx.size() * 2));
  DRCB_CUDA(cudaMalloc(&dd, hz.size() * 2));
  DRCB_CUDA(cudaMalloc(&dwf, size_t(cout) * cin * 9 * 4));
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, hz.data(), hz.size() * 2, cudaMemcpyHostToDevice);
  size_t wsb = 0;
  int rc = wgrad_bf16(dx, cin, cinp, dd, cout, coutp, hw, n, dwf, 0, nullptr, &wsb, 0, 0, 0);
  if (!rc) {
    if (cudaMalloc(&ws, wsb) != cudaSuccess) rc = fail(DRCB_ECUDA, "cudaMalloc wgrad scratch");
  }
  if (!rc) rc = wgrad_bf16(dx, cin, cinp, dd, cout, coutp, hw, n, dwf, 0, ws, &wsb, 0, 0, 0);
  if (!rc) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = cuda_fail(e, "drcb_debug_wgrad");
  }
  if (!rc) cudaMemcpy(dw, dwf, size_t(cout) * cin * 9 * 4, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dd);
  cudaFree(dwf);
  if (ws) cudaFree(ws);
  return rc;
}
