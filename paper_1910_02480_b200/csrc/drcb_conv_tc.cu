// drcb_conv_tc.cu — the U-Net on the 5th-generation tensor cores.
//
// Every 3x3 convolution / stride-1 transposed convolution of MapAutoencoder
// (cnn.py:193-215) runs as a persistent, warp-specialised implicit GEMM:
//
//   M = maps*H*W output pixels (tile 128), N = C_out (tile BN <= 256),
//   K = 9 taps x C_in (stage = one tap x 128 bytes of channels).
//
//   warp 0   TMA producer: the A tile of a tap is a 4-D TMA box of the NHWC
//            activation at (c0, x0+dx, y0+dy, n0); out-of-range rows/columns
//            are zero-filled by the TMA unit, which IS the conv's zero
//            padding (no im2col buffer). The B tile is a 2-D box of the
//            K-major packed weights. Both land 128B-swizzled.
//   warp 1   MMA issuer: one elected thread issues tcgen05.mma (kind::f16
//            bf16 or kind::tf32) into a double-buffered TMEM accumulator.
//   warps 2-5 epilogue: tcgen05.ld TMEM -> registers, fused bias + batch
//            norm (folded to y = acc*a + b) + LeakyReLU, store NHWC into the
//            destination channel slice (skips land inside the decoder's
//            concat buffers). The head's last deconv also fuses the 1x1
//            conv_out + ReLU and writes fp32 NCHW predictions.
//
// Max-pool and the bilinear 2x upsample run as small NHWC kernels.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <cstring>

#include "drcb_net.h"
#include "drcb_tc_ptx.cuh"

namespace drcb {

// The stream-ordered pool would release freed blocks to the OS at every
// synchronisation (release threshold 0), turning each frame's multi-GB
// activation workspace into a fresh cudaMalloc; keep them cached.
void keep_pool_memory() {
  static DeviceFlags done;
  const int dev = current_device();
  if (done.test(dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.set(dev);
}

namespace tc {

// src = max((o + 0.5)/2 - 0.5, 0) in closed form (no int<->float
// conversions on the XU pipe): o = 0 -> (0, 1, 0); o = 2i (i >= 1) ->
// (i-1, i, 0.75); o = 2i+1 -> (i, min(i+1, n-1), 0.25)
__device__ __forceinline__ void up_w(int o, int n, int& i0, int& i1, float& fr) {
  const int i = o >> 1;
  if (o & 1) {
    i0 = i;
    i1 = min(i + 1, n - 1);
    fr = 0.25f;
  } else if (o == 0) {
    i0 = 0;
    i1 = min(1, n - 1);
    fr = 0.f;
  } else {
    i0 = i - 1;
    i1 = i;
    fr = 0.75f;
  }
}

constexpr int BM = 128;
constexpr int NUM_THREADS = 192;  // 6 warps
constexpr int ROW_BYTES = 128;    // one swizzle row = one K stage per operand row

struct ConvArgs {
  int num_m_tiles, num_n_tiles, num_kb;   // kb = tap * cblocks + cb
  int cblocks;                            // C_in_pad / BK
  int hw;                                 // map side
  int rows_per_tile;                      // hw >= 12: 128 / hw, else hw
  int maps_per_tile;                      // 1 or 128 / hw^2
  int tiles_per_map;                      // hw*hw / 128 or 1
  int bn;                                 // N tile
  int cout;                               // real output channels written
  int cout_tot, cout_off;                 // destination buffer layout
  const float* ep_a;                      // per-channel scale
  const float* ep_b;                      // per-channel shift (bias folded)
  float slope;
  void* out;                              // NHWC bf16 / fp32
  int head;                               // 1: fuse head.conv_out + ReLU
  float* pred;                            // (maps,3,32,32) fp32 when head
  float hw_w[3 * 16];                     // conv_out weights (3, 16)
  float hw_b[3];
};

template <int KIND, int BN, int STAGES>
struct Smem {
  static constexpr int ELEM = elem_bytes(KIND);
  static constexpr int A_BYTES = BM * ROW_BYTES;
  static constexpr int B_BYTES = BN * ROW_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Epilogue of one 128 x BN accumulator tile held in TMEM: tcgen05.ld, folded
// BN + LeakyReLU, NHWC store into the destination slice; for the head layer
// the fused 1x1 conv_out + ReLU writes fp32 NCHW predictions.

// 16 accumulator columns [c0, c0+16) of this thread's pixel. DX: the tile
// holds three accumulators P_dx (dx = -1, 0, +1 at column offsets 0, BN, 2BN)
// computed from the UNSHIFTED input row; the conv output is
// P_-1(x-1) + P_0(x) + P_+1(x+1), the neighbours fetched from the adjacent
// lanes (a warp's 32 TMEM lanes are 32 consecutive pixels of one or two
// image rows) with zero beyond the row ends.
template <int BN, bool DX>
__device__ __forceinline__ void acc_chunk(uint32_t tbase, int c0, int x, int hw, float (&v)[16]) {
  uint32_t r[16];
  tmem_ld16(tbase + c0, r);
  if constexpr (!DX) {
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
  } else {
    uint32_t r0[16], r2[16];
    tmem_ld16(tbase + BN + c0, r0);
    tmem_ld16(tbase + 2 * BN + c0, r2);
    tmem_wait_ld();
    const bool has_l = x > 0, has_r = x < hw - 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float l = __shfl_up_sync(0xffffffffu, __uint_as_float(r[j]), 1);
      float rt = __shfl_down_sync(0xffffffffu, __uint_as_float(r2[j]), 1);
      float s = __uint_as_float(r0[j]);
      if (has_l) s += l;
      if (has_r) s += rt;
      v[j] = s;
    }
  }
}

// folded BN (scale a, shift b; 16-B aligned vectors) + LeakyReLU
__device__ __forceinline__ void bn_lrelu16(const float (&acc)[16], const float* a, const float* b,
                                           float slope, float (&v)[16]) {
#pragma unroll
  for (int j = 0; j < 16; j += 4) {
    const float4 av = __ldg(reinterpret_cast<const float4*>(a + j));
    const float4 bv = __ldg(reinterpret_cast<const float4*>(b + j));
    const float aa[4] = {av.x, av.y, av.z, av.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float x = acc[j + t] * aa[t] + bb[t];
      v[j + t] = x >= 0.f ? x : slope * x;
    }
  }
}
// the same with the folded vectors staged in SMEM (sa / sb: SMEM addresses
// of the chunk's first channel)
__device__ __forceinline__ void bn_lrelu16_s(const float (&acc)[16], uint32_t sa, uint32_t sb,
                                             float slope, float (&v)[16]) {
#pragma unroll
  for (int j = 0; j < 16; j += 4) {
    float aa[4], bb[4];
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(aa[0]), "=f"(aa[1]), "=f"(aa[2]), "=f"(aa[3])
                 : "r"(sa + 4 * j));
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(bb[0]), "=f"(bb[1]), "=f"(bb[2]), "=f"(bb[3])
                 : "r"(sb + 4 * j));
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float x = acc[j + t] * aa[t] + bb[t];
      v[j + t] = x >= 0.f ? x : slope * x;
    }
  }
}
// folded BN vectors of channels [0, EP_MAX) staged in SMEM: a at sep, b at
// sep + 4 * EP_MAX
constexpr int EP_MAX = 256;
__device__ __forceinline__ void stage_ep(const ConvArgs& p, int ncout, float* sep, int t0, int nthr) {
  for (int i = t0; i < ncout; i += nthr) {
    sep[i] = p.ep_a[i];
    sep[EP_MAX + i] = p.ep_b[i];
  }
}

// cbeg/cstep: the 16-column chunks this warp handles (several epilogue warps
// may share one TMEM lane quarter)
template <int KIND, int BN, bool DX = false>
__device__ __forceinline__ void epilogue_tile(const ConvArgs& p, uint32_t tbase, int64_t m, int nt,
                                              int cbeg = 0,
                                              int cstep = 16) {
  const int xpix = int(m & int64_t(p.hw - 1));  // hw is a power of two
  if (p.head) {
    if (cbeg != 0) return;
    // head.deconv2 (BN == 16 channels) + BN + LeakyReLU, then the fused
    // 1x1 conv_out + ReLU -> fp32 NCHW prediction (cnn.py:209-215)
    float acc[16];
    acc_chunk<BN, DX>(tbase, 0, xpix, p.hw, acc);
    float v[16];
    bn_lrelu16(acc, p.ep_a, p.ep_b, p.slope, v);
    int64_t n = m / 1024;
    int pix = int(m % 1024);
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      float s = p.hw_b[o];
#pragma unroll
      for (int j = 0; j < 16; ++j) s += p.hw_w[o * 16 + j] * v[j];
      p.pred[(n * 3 + o) * 1024 + pix] = fmaxf(s, 0.f);
    }
  } else {
#pragma unroll 1
    for (int c0 = cbeg; c0 < BN; c0 += cstep) {
      const int cg = nt * BN + c0;
      if (cg >= p.cout) break;
      float acc[16];
      acc_chunk<BN, DX>(tbase, c0, xpix, p.hw, acc);
      float v[16];
      bn_lrelu16(acc, p.ep_a + cg, p.ep_b + cg, p.slope, v);
      if constexpr (KIND != 1) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pk[j] = pack2<KIND>(v[2 * j], v[2 * j + 1]);
        uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.out) +
                                              m * p.cout_tot + p.cout_off + cg);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + m * p.cout_tot +
                                                p.cout_off + cg);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_float4(round_tf32(v[4 * j]), round_tf32(v[4 * j + 1]),
                               round_tf32(v[4 * j + 2]), round_tf32(v[4 * j + 3]));
      }
    }
  }
}

template <int KIND, int BN, int STAGES>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ ConvArgs p) {
  pdl_wait();
  using SM = Smem<KIND, BN, STAGES>;
  constexpr int UMMA_KSTEPS = ROW_BYTES / 32;  // 32 B of K per MMA for both kinds
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SM::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.num_m_tiles * p.num_n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mt = tile % p.num_m_tiles, nt = tile / p.num_m_tiles;
        int n0, y0;
        if (p.maps_per_tile == 1) {
          n0 = mt / p.tiles_per_map;
          y0 = (mt % p.tiles_per_map) * p.rows_per_tile;
        } else {
          n0 = mt * p.maps_per_tile;
          y0 = 0;
        }
        for (int kb = 0; kb < p.num_kb; ++kb) {
          int tap = kb / p.cblocks, cb = kb % p.cblocks;
          int dy = tap / 3 - 1, dx = tap % 3 - 1;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * SM::STAGE_BYTES;
          uint8_t* sB = sA + SM::A_BYTES;
          mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
          const int celems = ROW_BYTES / SM::ELEM;
          tma_load_4d(&mapA, &full[stage], sA, cb * celems, dx, y0 + dy, n0);
          tma_load_2d(&mapB, &full[stage], sB, kb * celems, nt * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint32_t a0 = smem_u32(smem + stage * SM::STAGE_BYTES);
          uint32_t b0 = a0 + SM::A_BYTES;
#pragma unroll
          for (int k = 0; k < UMMA_KSTEPS; ++k) {
            tc_mma<KIND>(tmem_d, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), idesc,
                         (kb | k) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    const int row = q * 32 + lane;  // pixel within the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt = tile % p.num_m_tiles, nt = tile / p.num_m_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t m = int64_t(mt) * BM + row;
      const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
      epilogue_tile<KIND, BN>(p, tbase, m, nt);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Epilogue into a SMEM staging tile for a TMA store: BN channels of 128
// pixels as BN/CEL sub-tiles of [128 px][128 B], each in the SWIZZLE_128B
// layout the output tensor map expects (16-B piece j of pixel r at
// r*128 + ((j ^ (r & 7)) << 4)): the global write is one coalesced bulk
// tensor store per sub-tile instead of 16-B scattered stores per thread.
template <int KIND, int BN, bool DX, int CSTEP>
__device__ __forceinline__ void epilogue_stage(const ConvArgs& p, uint32_t tbase, int64_t m, int nt,
                                               uint8_t* ost, int cbeg, uint32_t sep = 0) {
  constexpr int ELEM = elem_bytes(KIND);
  constexpr int CEL = ROW_BYTES / ELEM;
  const int xpix = int(m & int64_t(p.hw - 1));  // hw is a power of two
  const int r = int(m & (BM - 1));
  const uint32_t ost_s = smem_u32(ost);
  if constexpr (BN < CEL) {
    // channels [BN, CEL) of the stored row are the next layer's K padding
    if (cbeg == 0)
#pragma unroll
      for (int j = BN * ELEM / 16; j < 8; ++j) sts128(ost_s + r * ROW_BYTES + ((j ^ (r & 7)) << 4), 0u, 0u, 0u, 0u);
  }
  // unrolled so the next chunk's TMEM loads overlap this chunk's math
#pragma unroll
  for (int i = 0; i < (BN + CSTEP - 1) / CSTEP; ++i) {
    const int c0 = cbeg + i * CSTEP;
    if (c0 >= BN) break;
    const int cg = nt * BN + c0;
    float acc[16];
    acc_chunk<BN, DX>(tbase, c0, xpix, p.hw, acc);
    float v[16];
    if (sep)
      bn_lrelu16_s(acc, sep + 4 * cg, sep + 4 * (EP_MAX + cg), p.slope, v);
    else
      bn_lrelu16(acc, p.ep_a + cg, p.ep_b + cg, p.slope, v);
    const uint32_t sub = ost_s + (c0 / CEL) * (BM * ROW_BYTES) + r * ROW_BYTES;
    const int jb = (c0 % CEL) * ELEM / 16;
    if constexpr (KIND != 1) {
      uint32_t pk[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pk[j] = pack2<KIND>(v[2 * j], v[2 * j + 1]);
      sts128(sub + (((jb + 0) ^ (r & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
      sts128(sub + (((jb + 1) ^ (r & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        sts128(sub + (((jb + j) ^ (r & 7)) << 4), __float_as_uint(round_tf32(v[4 * j])),
               __float_as_uint(round_tf32(v[4 * j + 1])), __float_as_uint(round_tf32(v[4 * j + 2])),
               __float_as_uint(round_tf32(v[4 * j + 3])));
    }
  }
}
__device__ __forceinline__ void unpack8_bf16(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(b[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// bilinear mix of four 16-B vectors of packed 16-bit pairs (H2 = bf16x2 or
// fp16x2; p00, p10, p01, p11) in packed arithmetic:
// t0 = fma(p00, omr, p10*fr), t1 = fma(p01, omr, p11*fr), v = fma(t0, omc, t1*fc)
// (the weights 0, 0.25, 0.75, 1 are exact in both formats)
template <typename H2>
__device__ __forceinline__ void up_mix_h2(const uint4 (&q)[4], float omr, float fr, float omc,
                                          float fc, uint32_t (&out)[4]) {
  const H2 wr0 = splat2<H2>(omr), wr1 = splat2<H2>(fr);
  const H2 wc0 = splat2<H2>(omc), wc1 = splat2<H2>(fc);
  const H2* a = reinterpret_cast<const H2*>(&q[0]);
  const H2* b = reinterpret_cast<const H2*>(&q[1]);
  const H2* c = reinterpret_cast<const H2*>(&q[2]);
  const H2* d = reinterpret_cast<const H2*>(&q[3]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // explicit fused forms (one rounded product, one fma): the compiler may
    // not contract them differently per call site, so every caller (the
    // upsample kernel, the fused dec2.deconv2 epilogue) computes the same bits
    const H2 t0 = __hfma2(a[i], wr0, __hmul2_rn(b[i], wr1));
    const H2 t1 = __hfma2(c[i], wr0, __hmul2_rn(d[i], wr1));
    const H2 v = __hfma2(t0, wc0, __hmul2_rn(t1, wc1));
    out[i] = *reinterpret_cast<const uint32_t*>(&v);
  }
}

// elementwise max of four 16-B vectors of stored values (bf16x8 / fp32x4)
template <int KIND>
__device__ __forceinline__ uint4 max4(uint4 a, uint4 b, uint4 c, uint4 d) {
  uint4 r;
  uint32_t* ra = reinterpret_cast<uint32_t*>(&a);
  uint32_t* rb = reinterpret_cast<uint32_t*>(&b);
  uint32_t* rc = reinterpret_cast<uint32_t*>(&c);
  uint32_t* rd = reinterpret_cast<uint32_t*>(&d);
  uint32_t* rr = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (KIND != 1) {
      using H2 = Elem2T<KIND>;
      H2 x = __hmax2(__hmax2(*reinterpret_cast<H2*>(&ra[i]), *reinterpret_cast<H2*>(&rb[i])),
                     __hmax2(*reinterpret_cast<H2*>(&rc[i]), *reinterpret_cast<H2*>(&rd[i])));
      rr[i] = *reinterpret_cast<uint32_t*>(&x);
    } else {
      rr[i] = __float_as_uint(fmaxf(fmaxf(__uint_as_float(ra[i]), __uint_as_float(rb[i])),
                                    fmaxf(__uint_as_float(rc[i]), __uint_as_float(rd[i]))));
    }
  }
  return r;
}

constexpr int RT_EPI_WARPS = 8;
constexpr int RT_THREADS = 64 + 32 * RT_EPI_WARPS;
// k_conv_rows adds a pool warp (warp 10) for the fused 2x2 max-pool layers
constexpr int RT_POOL_WARP = 2 + RT_EPI_WARPS;
constexpr int ROWS_THREADS = RT_THREADS + 32;
// the two epilogue warps of TMEM lane quarter q (32 pixel rows)
__device__ __forceinline__ void quarter_bar(int q) {
  asm volatile("bar.sync %0, 64;" ::"r"(8 + q) : "memory");
}
__device__ __forceinline__ void epi_bar_rt() {
  asm volatile("bar.sync 2, %0;" ::"r"(32 * RT_EPI_WARPS) : "memory");
}

struct RowArgs {
  int a_bytes;    // (rows+2) * W * 128
  int row_bytes;  // W * 128: one dy shift
  int sa, sb;     // A / B ring depths
  int o_bytes;    // one output staging tile (BM * BN * elem); 0 = direct stores (head)
  int p_bytes;    // fused 2x2 max-pool staging tile (BM/4 * BN * elem); 0 = no pool
  int up2;        // MH = 2 at 16x16 (a tile = one whole map): store up2x(out) at 32x32 instead
  int pool_cta;   // fused pool by the epilogue warps on whole staged tiles (A/B switch)
};

// Row-tile implicit GEMM for hw in {16, 32}: an M tile is BM/W whole image
// rows, its activation operand one TMA box of rows+2 rows (OOB rows zero =
// the conv's padding), and the three dy taps read that box at descriptor
// offsets dy*W*128 B (a multiple of the 1024-B swizzle atom).
//   DX = false ("halo"): one box per (channel chunk, dx) loaded at x offset
//     dx-1 (OOB columns zero); per dy one MMA with N = BN into the single
//     accumulator. B stage = the three dy weight tiles of that (chunk, dx).
//   DX = true ("dx-in-N"): one box per chunk; per dy ONE MMA multiplies it by
//     the three dx taps' weights stacked along N (N = 3 BN, split in two for
//     BN = 128) into accumulators P_-1, P_0, P_+1 of the unshifted input,
//     combined in the epilogue as P_-1(x-1) + P_0(x) + P_+1(x+1) by lane
//     shuffles (acc_chunk<BN, true>). 1/3 of the activation traffic for 3x
//     the TMEM reads + shuffles in the epilogue.
// RES: the whole weight matrix stays resident in SMEM ([chunk][dy][dx]
// tiles). 8 epilogue warps (two per TMEM lane quarter) stage the tile in
// SMEM in the output map's swizzled layout; one thread TMA-stores it.
template <int KIND, int BN, bool RES, bool DX, int MH, bool PW = false>
__global__ void __launch_bounds__(PW ? ROWS_THREADS : RT_THREADS, 1)
    k_conv_rows(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const __grid_constant__ CUtensorMap mapO, const __grid_constant__ CUtensorMap mapP,
                const __grid_constant__ ConvArgs p, const __grid_constant__ RowArgs h) {
  pdl_wait();
  constexpr int B_TILE = BN * ROW_BYTES;
  constexpr int B3 = 3 * B_TILE;                       // one B stage: three weight tiles
  constexpr int ELEM = elem_bytes(KIND);
  constexpr int CEL = ROW_BYTES / ELEM;
  constexpr int NACCW = DX ? 3 * BN : BN;              // TMEM columns per M block
  // MH = 2: a work tile is two M blocks (BM rows each) sharing every A and B
  // stage (half the weight traffic per pixel for streamed-weight layers)
  // TMEM accumulator buffers: four when they fit (small-N layers, whose
  // per-tile epilogue latency is long next to their MMA time), else two / one
  constexpr int NACC = 4 * MH * NACCW <= 512 ? 4 : (2 * MH * NACCW <= 512 ? 2 : 1);
  static_assert(MH == 1 || (BN <= CEL && DX), "two-block tiles: one staging sub-tile, dx-in-N");
  constexpr int NSPLIT = NACCW <= 256 ? 1 : 2;
  constexpr int NMMA = NACCW / NSPLIT;
  constexpr int BPA = DX ? 3 : 1;                      // B stages per A stage
  constexpr uint32_t COLS = NACC * MH * NACCW;
  constexpr uint32_t TMEM_COLS = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512)));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int n_wtiles = 9 * p.cblocks;
  uint8_t* wres = smem;  // RES: tiles ordered [chunk][dy][dx]
  uint8_t* aring = smem + (RES ? n_wtiles * B_TILE : 0);
  uint8_t* bring = aring + h.sa * h.a_bytes;
  uint8_t* ostage = bring + (RES ? 0 : h.sb * B3);  // 2 x o_bytes, 1024-aligned
  uint8_t* pstage = ostage + (h.up2 ? 3 : 2) * h.o_bytes;  // 2 x p_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(pstage + 2 * h.p_bytes);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + 8;
  uint64_t* bfull = bars + 16;
  uint64_t* bempty = bars + 24;
  uint64_t* tfull = bars + 32;
  uint64_t* tempty = bars + 36;
  uint64_t* wfull = bars + 40;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 41);
  uint64_t* pfull = bars + 48;   // fused pool: the 4 lane quarters staged obuf
  uint64_t* pempty = bars + 50;  // fused pool: the pool warp has read obuf
  // fused 2x2 max-pool on the pool warp (single-block tiles, no up2): the
  // epilogue keeps its per-quarter staging and stores
  // (PW instantiations only: launched with the extra warp)
  constexpr bool POOL_WARP = PW;
  // the fused head epilogue (16 channels -> 3) is one 16-column chunk: the two
  // epilogue warp groups take alternate tiles (accumulator buffer = group)
  // instead of one group idling
  const bool HEAD_SPLIT = p.head && h.o_bytes == 0 && NACC % 2 == 0 && RT_EPI_WARPS == 8;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    for (int s = 0; s < h.sa; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < h.sb; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], HEAD_SPLIT ? RT_EPI_WARPS / 2 : RT_EPI_WARPS);
    }
    mbar_init(wfull, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pfull[b], 4);
      mbar_init(&pempty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.num_m_tiles * p.num_n_tiles;
  const int astages = DX ? p.cblocks : 3 * p.cblocks;  // A boxes per tile
  // N tiles of one M tile are adjacent in the schedule (the boxes are
  // re-read from L2, not DRAM)
  if (warp == 0) {
    if (lane == 0) {
      if (RES) {
        // (several N tiles: the grid is a multiple of num_n_tiles, so this
        // CTA's tiles all have N tile blockIdx.x % num_n_tiles: its weights)
        const int nt_res = int(blockIdx.x) % p.num_n_tiles;
        mbar_expect_tx(wfull, uint32_t(n_wtiles * B_TILE));
        for (int cb = 0; cb < p.cblocks; ++cb)
          for (int t = 0; t < 9; ++t)
            tma_load_2d(&mapB, wfull, wres + (cb * 9 + t) * B_TILE, (t * p.cblocks + cb) * CEL,
                        nt_res * BN);
      }
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt = tile % p.num_n_tiles, mt = tile / p.num_n_tiles;
        int n0 = mt / p.tiles_per_map;
        int y0 = (mt % p.tiles_per_map) * p.rows_per_tile;
        for (int as = 0; as < astages; ++as) {
          const int cb = DX ? as : as / 3, dxi = DX ? 1 : as % 3;
          mbar_wait(&aempty[sa], pa ^ 1);
          mbar_expect_tx(&afull[sa], uint32_t(h.a_bytes));
          tma_load_4d(&mapA, &afull[sa], aring + sa * h.a_bytes, cb * CEL, dxi - 1, y0 - 1, n0);
          if (++sa == h.sa) {
            sa = 0;
            pa ^= 1;
          }
          if (!RES) {
            for (int bs = 0; bs < BPA; ++bs) {
              mbar_wait(&bempty[sb], pb ^ 1);
              mbar_expect_tx(&bfull[sb], uint32_t(B3));
              uint8_t* dst = bring + sb * B3;
              // DX: the three dx tiles of (cb, dy = bs); halo: the three dy
              // tiles of (cb, dx)
              for (int j = 0; j < 3; ++j) {
                const int tap = DX ? bs * 3 + j : j * 3 + dxi;
                tma_load_2d(&mapB, &bfull[sb], dst + j * B_TILE, (tap * p.cblocks + cb) * CEL, nt * BN);
              }
              if (++sb == h.sb) {
                sb = 0;
                pb ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, BM, NMMA);
      if (RES) mbar_wait(wfull, 0);
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * MH * NACCW;
        bool first = true;
        for (int as = 0; as < astages; ++as) {
          const int cb = DX ? as : as / 3, dxi = DX ? 1 : as % 3;
          mbar_wait(&afull[sa], pa);
          tc_fence_after();
          const uint32_t a0 = smem_u32(aring + sa * h.a_bytes);
          uint32_t bstage = 0;
          if (!RES && !DX) {
            mbar_wait(&bfull[sb], pb);
            tc_fence_after();
            bstage = smem_u32(bring + sb * B3);
          }
#pragma unroll 1
          for (int dyi = 0; dyi < 3; ++dyi) {
            uint32_t bb;
            if (RES) {
              bb = smem_u32(wres + (cb * 9 + dyi * 3 + (DX ? 0 : dxi)) * B_TILE);
            } else if (DX) {
              mbar_wait(&bfull[sb], pb);
              tc_fence_after();
              bb = smem_u32(bring + sb * B3);
            } else {
              bb = bstage + dyi * B_TILE;
            }
            const uint32_t aa = a0 + dyi * h.row_bytes;
#pragma unroll
            for (int k = 0; k < ROW_BYTES / 32; ++k) {
#pragma unroll
              for (int mh = 0; mh < MH; ++mh)
#pragma unroll
                for (int sp = 0; sp < NSPLIT; ++sp)
                  tc_mma<KIND>(tmem_d + mh * NACCW + sp * NMMA,
                               sw128_desc(aa + mh * BM * ROW_BYTES + 32 * k),
                               sw128_desc(bb + sp * NMMA * ROW_BYTES + 32 * k), idesc,
                               first ? 0u : 1u);
              first = false;
            }
            if (!RES && DX) {
              tc_commit(&bempty[sb]);
              if (++sb == h.sb) {
                sb = 0;
                pb ^= 1;
              }
            }
          }
          if (!RES && !DX) {
            tc_commit(&bempty[sb]);
            if (++sb == h.sb) {
              sb = 0;
              pb ^= 1;
            }
          }
          tc_commit(&aempty[sa]);
          if (++sa == h.sa) {
            sa = 0;
            pa ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == RT_POOL_WARP) {
    if constexpr (PW) {
      // fused 2x2 max-pool (cnn.py:152-156) of each staged, already rounded
      // tile once its four lane quarters have staged it: BM/4 pooled pixels x
      // BN channels in the same swizzled layout, TMA-stored to the next level
      const int hw = p.hw, ho = hw >> 1, lho = __ffs(ho) - 1;
      constexpr int PPR = ROW_BYTES / 16;  // 16-B pieces per sub-tile row
      int obuf = 0, kt = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int nt = tile % p.num_n_tiles, mt = tile / p.num_n_tiles;
        const int n0 = mt / p.tiles_per_map;
        const int y0 = (mt % p.tiles_per_map) * p.rows_per_tile;
        mbar_wait(&pfull[obuf], (kt >> 1) & 1);
        uint8_t* ot = ostage + obuf * h.o_bytes;
        uint8_t* pt = pstage + obuf * h.p_bytes;
        if (lane == 0) bulk_wait_read1();  // the pool store of 2 tiles ago has read pt
        __syncwarp();
        constexpr int PIECES = BN * ELEM / 16;  // 16-B pieces per pooled pixel
#pragma unroll
        for (int it = 0; it < (BM / 4) * PIECES / 32; ++it) {
          const int e = lane + 32 * it;
          const int pr = e / PIECES, pc = e % PIECES;
          const int sub = pc / PPR, jj = pc % PPR;
          const int py = pr >> lho, px = pr & (ho - 1);  // ho is a power of two
          const int r00 = (2 * py) * hw + 2 * px;
          const uint32_t base = smem_u32(ot + sub * BM * ROW_BYTES);
          uint4 v[4];
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int rr = r00 + (w >> 1) * hw + (w & 1);
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[w].x), "=r"(v[w].y), "=r"(v[w].z), "=r"(v[w].w)
                         : "r"(base + rr * ROW_BYTES + ((jj ^ (rr & 7)) << 4)));
          }
          uint4 m4 = max4<KIND>(v[0], v[1], v[2], v[3]);
          sts128(smem_u32(pt + sub * (BM / 4) * ROW_BYTES) + pr * ROW_BYTES + ((jj ^ (pr & 7)) << 4),
                 m4.x, m4.y, m4.z, m4.w);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&pempty[obuf]);  // ot may be restaged
          for (int sb2 = 0; sb2 < BN / CEL; ++sb2)
            tma_store_4d(&mapP, pt + sb2 * (BM / 4) * ROW_BYTES, nt * BN + sb2 * CEL, 0, y0 >> 1, n0);
          bulk_commit();
        }
        obuf ^= 1;
        ++kt;
      }
      if (lane == 0) bulk_wait_all();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    // RT_EPI_WARPS / 4 warps per TMEM lane quarter split the 16-column chunks
    const int grp = (warp - 2) / 4;
    constexpr int CSTEP = 16 * (RT_EPI_WARPS / 4);
    // folded BN vectors in SMEM for the staged epilogue
    float* s_ep = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);
    const int ncout = p.num_n_tiles * BN;
    const uint32_t sep = (h.o_bytes && ncout <= EP_MAX) ? smem_u32(s_ep) : 0u;
    if (sep) {
      stage_ep(p, ncout, s_ep, threadIdx.x - 64, 32 * RT_EPI_WARPS);
      epi_bar_rt();
    }
    int acc = 0, obuf = 0, kt = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int nt = tile % p.num_n_tiles, mt = tile / p.num_n_tiles;
      if (HEAD_SPLIT && (acc & 1) != grp) {
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase0 = tmem_base + (uint32_t(q * 32) << 16) + acc * MH * NACCW;
      if (MH == 2 && h.up2) {
        // The tile is one whole 16x16 map: stage it (stored, rounded values),
        // then write its bilinear 2x upsample (cnn.py:159-174, the operation
        // order of k_up_nhwc) straight into the 32x32 concat buffer in four
        // 8-row chunks; the 16x16 output itself is never stored.
        uint8_t* lowb = ostage;  // + two 8-row output chunk buffers (3 x o_bytes)
        if (threadIdx.x == 64) bulk_wait_read0();
        epi_bar_rt();
#pragma unroll
        for (int mh = 0; mh < MH; ++mh)
          epilogue_stage<KIND, BN, DX, CSTEP>(p, tbase0 + mh * NACCW, (int64_t(mt) * MH + mh) * BM + row,
                                              nt, lowb + mh * BM * ROW_BYTES, 16 * grp, sep);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        epi_bar_rt();
        const uint32_t L0 = smem_u32(lowb);
        const int et = threadIdx.x - 64;
        for (int chk = 0; chk < 4; ++chk) {
          uint8_t* upb = ostage + (1 + (chk & 1)) * h.o_bytes;
          const uint32_t U0 = smem_u32(upb);
          if (chk > 1) {  // the store of chunk chk-2 has read this buffer
            if (threadIdx.x == 64) bulk_wait_read1();
            epi_bar_rt();
          }
          // one item = two vertically adjacent 2x2 output blocks (low-res
          // rows bi0, bi0 + 1) from their 4x3 low-res neighbourhood: 12 SMEM
          // reads per 8 outputs; each output mixes its four neighbours exactly
          // as k_up_nhwc does
          for (int e = et; e < 2 * 16 * 8; e += 32 * RT_EPI_WARPS) {
            const int j = e & 7, bj = (e >> 3) & 15;
            const int bi0 = 4 * chk + 2 * (e >> 7);  // low-res rows bi0, bi0 + 1
            uint4 nbq[4][3];
#pragma unroll
            for (int dr = 0; dr < 4; ++dr) {
              const int r = min(max(bi0 + dr - 1, 0), 15);
#pragma unroll
              for (int dc = 0; dc < 3; ++dc) {
                const int c = min(max(bj + dc - 1, 0), 15);
                const int rr = r * 16 + c;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(nbq[dr][dc].x), "=r"(nbq[dr][dc].y), "=r"(nbq[dr][dc].z),
                               "=r"(nbq[dr][dc].w)
                             : "r"(L0 + rr * ROW_BYTES + ((j ^ (rr & 7)) << 4)));
              }
            }
            const float fc_even = bj == 0 ? 0.f : 0.75f;
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
              const int bi = bi0 + hb;
              const float fr_even = bi == 0 ? 0.f : 0.75f;
#pragma unroll
              for (int a2 = 0; a2 < 2; ++a2) {
                const float fr = a2 ? 0.25f : fr_even;
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2) {
                  const float fc = b2 ? 0.25f : fc_even;
                  const uint4 q[4] = {nbq[hb + a2][b2], nbq[hb + a2 + 1][b2], nbq[hb + a2][b2 + 1],
                                      nbq[hb + a2 + 1][b2 + 1]};
                  uint32_t pk[4];
                  up_mix_h2<Elem2T<KIND>>(q, 1.f - fr, fr, 1.f - fc, fc, pk);
                  const int opx = ((2 * bi + a2) & 7) * 32 + 2 * bj + b2;  // pixel in the chunk
                  sts128(U0 + opx * ROW_BYTES + ((j ^ (opx & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
                }
              }
            }
          }
          fence_proxy_async();
          epi_bar_rt();
          if (threadIdx.x == 64) {
            tma_store_4d(&mapO, upb, nt * BN, 0, 8 * chk, mt);
            bulk_commit();
          }
        }
      } else if (h.o_bytes && (!h.p_bytes || POOL_WARP)) {
        // per lane quarter: its two warps stage their 32 pixel rows and one
        // thread stores them (mapO: 32-pixel boxes); no CTA-wide barrier
        uint8_t* ot = ostage + obuf * h.o_bytes;
        const bool issuer = grp == 0 && lane == 0;
        if (issuer) {
          bulk_wait_read1();  // this quarter's store of 2 tiles ago has read ot
          // and the pool warp has read it (its use before this one)
          if (POOL_WARP && kt >= 2) mbar_wait(&pempty[obuf], ((kt >> 1) - 1) & 1);
        }
        quarter_bar(q);
#pragma unroll
        for (int mh = 0; mh < MH; ++mh)
          epilogue_stage<KIND, BN, DX, CSTEP>(p, tbase0 + mh * NACCW, (int64_t(mt) * MH + mh) * BM + row,
                                              nt, ot + mh * BM * ROW_BYTES, 16 * grp, sep);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        fence_proxy_async();
        quarter_bar(q);
        if (issuer) {
          const int n0 = mt / p.tiles_per_map;
          const int y0 = (mt % p.tiles_per_map) * p.rows_per_tile;
#pragma unroll
          for (int mh = 0; mh < MH; ++mh)
            for (int sb2 = 0; sb2 < (BN + CEL - 1) / CEL; ++sb2)
              tma_store_4d(&mapO, ot + (sb2 * MH * BM + mh * BM + q * 32) * ROW_BYTES,
                           p.cout_off + nt * BN + sb2 * CEL, 0, y0 + (mh * BM + q * 32) / p.hw, n0);
          bulk_commit();
          if (POOL_WARP) mbar_arrive(&pfull[obuf]);  // this quarter's rows are staged
        }
        obuf ^= 1;
        ++kt;
      } else if (h.o_bytes) {
        uint8_t* ot = ostage + obuf * h.o_bytes;
        if (threadIdx.x == 64) bulk_wait_read1();  // the store issued 2 tiles ago has read ot
        epi_bar_rt();
#pragma unroll
        for (int mh = 0; mh < MH; ++mh)
          epilogue_stage<KIND, BN, DX, CSTEP>(p, tbase0 + mh * NACCW, (int64_t(mt) * MH + mh) * BM + row,
                                              nt, ot + mh * BM * ROW_BYTES, 16 * grp, sep);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        fence_proxy_async();
        epi_bar_rt();
        const int n0 = mt / p.tiles_per_map;
        const int y0 = (mt % p.tiles_per_map) * p.rows_per_tile;
        if (threadIdx.x == 64) {
          for (int sb2 = 0; sb2 < (BN + CEL - 1) / CEL; ++sb2)
            tma_store_4d(&mapO, ot + sb2 * MH * BM * ROW_BYTES, p.cout_off + nt * BN + sb2 * CEL, 0, y0, n0);
        }
        if (h.p_bytes) {
          // fused 2x2 max-pool (cnn.py:152-156) of the staged, already rounded
          // tile: BM/4 pooled pixels x BN channels, same swizzled layout
          uint8_t* pt = pstage + obuf * h.p_bytes;
          const int hw = p.hw, ho = hw >> 1;
          constexpr int PPR = ROW_BYTES / 16;  // 16-B pieces per sub-tile row
          for (int e = threadIdx.x - 64; e < (BM / 4) * (BN * ELEM / 16); e += 32 * RT_EPI_WARPS) {
            const int pr = e / (BN * ELEM / 16), pc = e % (BN * ELEM / 16);
            const int sub = pc / PPR, jj = pc % PPR;
            const int py = pr / ho, px = pr % ho;
            const int r00 = (2 * py) * hw + 2 * px;
            const uint32_t base = smem_u32(ot + sub * BM * ROW_BYTES);
            uint4 v[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const int rr = r00 + (w >> 1) * hw + (w & 1);
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v[w].x), "=r"(v[w].y), "=r"(v[w].z), "=r"(v[w].w)
                           : "r"(base + rr * ROW_BYTES + ((jj ^ (rr & 7)) << 4)));
            }
            uint4 m4 = max4<KIND>(v[0], v[1], v[2], v[3]);
            sts128(smem_u32(pt + sub * (BM / 4) * ROW_BYTES) + pr * ROW_BYTES + ((jj ^ (pr & 7)) << 4),
                   m4.x, m4.y, m4.z, m4.w);
          }
          fence_proxy_async();
          epi_bar_rt();
          if (threadIdx.x == 64)
            for (int sb2 = 0; sb2 < BN / CEL; ++sb2)
              tma_store_4d(&mapP, pt + sb2 * (BM / 4) * ROW_BYTES, nt * BN + sb2 * CEL, 0, y0 >> 1, n0);
        }
        if (threadIdx.x == 64) bulk_commit();
        obuf ^= 1;
      } else {
#pragma unroll
        for (int mh = 0; mh < MH; ++mh)
          epilogue_tile<KIND, BN, DX>(p, tbase0 + mh * NACCW, (int64_t(mt) * MH + mh) * BM + row, nt,
                                      HEAD_SPLIT ? 0 : 16 * grp, CSTEP);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0 && grp == 0 && h.o_bytes) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// The decoder head fused (bf16): head.deconv1 (64 -> 32) + BN + LeakyReLU,
// head.deconv2 (32 -> 16) + BN + LeakyReLU, conv_out (1x1, 16 -> 3) + ReLU,
// with head.deconv1's output living only in SMEM: the 32x32 layer's 64-channel
// padded output (537 MB per 4,096 maps) is neither written nor re-read.
// A CTA walks whole maps, 8 items of 4 output rows each, in row order, so
// every head.deconv1 row is computed once: item t computes rows 4t+1..4t+4
// (one M block, dx taps stacked along N = 96) and reuses rows 4t-1, 4t from
// item t-1; item 0 computes rows 0..7 (two blocks, rows 5..7 unused). The
// six rows 4t-1..4t+4 that head.deconv2 (N = 48, K = the 32 real channels)
// reads at dy offsets form A2[t & 1], written in the 128B-swizzled layout a
// TMA load would produce; rows outside the map are zero (head.deconv2's
// padding). A reused row stays in the registers of the warp that computed it
// and is written into the next item's buffer with that item's rows. Same products, fp32 accumulation groups and bf16 rounding of the
// intermediate as the two-kernel path (bit-identical, DRCB_NO_HEAD_FUSE).
//   warp 0: TMA (weights once; per item one input box, two stages)
//   warp 1: MMA: head.deconv1 of item i, then head.deconv2 of item i-1
//   warps 2-9: head.deconv1 epilogue of item i (two warps per lane quarter,
//              16 channels each), then the head.deconv2 + conv_out epilogue
//              of item i-1 (the warp group of i-1's parity)
constexpr int HF_ROW = 32 * ROW_BYTES;       // one 32-px row of 128-B pixels
constexpr int HF_A1 = 10 * HF_ROW;           // input box: 10 rows (item 0) / 6 rows
constexpr int HF_A2 = 6 * HF_ROW;            // rows 4t-1 .. 4t+4
constexpr int HF_W1 = 9 * 32 * ROW_BYTES;    // 9 tiles [dy][dx] of 32 rows
constexpr int HF_W2 = 9 * 16 * ROW_BYTES;    // 9 tiles of 16 rows
constexpr int HF_ACC1 = 2 * 96;              // TMEM columns per head.deconv1 accumulator
constexpr int HF_ACC2 = 2 * HF_ACC1;         // first head.deconv2 accumulator column

template <int KIND>
__global__ void __launch_bounds__(RT_THREADS, 1)
    k_head_fused(const __grid_constant__ CUtensorMap mapA10, const __grid_constant__ CUtensorMap mapA6,
                 const __grid_constant__ CUtensorMap mapW1, const __grid_constant__ CUtensorMap mapW2,
                 const __grid_constant__ ConvArgs p1, const __grid_constant__ ConvArgs p2, int nmaps) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* w1 = smem;
  uint8_t* w2 = w1 + HF_W1;
  uint8_t* a1 = w2 + HF_W2;      // 2 stages
  uint8_t* a2 = a1 + 2 * HF_A1;  // 2 buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(a2 + 2 * HF_A2);
  uint64_t* a1full = bars;         // [2]
  uint64_t* a1empty = bars + 2;    // [2]
  uint64_t* acc1full = bars + 4;   // [2]
  uint64_t* acc1empty = bars + 6;  // [2]
  uint64_t* a2full = bars + 8;     // [2]
  uint64_t* a2empty = bars + 10;   // [2]
  uint64_t* acc2full = bars + 12;  // [2]
  uint64_t* acc2empty = bars + 14; // [2]
  uint64_t* wfull = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA10);
    prefetch_map(&mapA6);
    prefetch_map(&mapW1);
    prefetch_map(&mapW2);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a1full[i], 1);
      mbar_init(&a1empty[i], 1);
      mbar_init(&acc1full[i], 1);
      mbar_init(&acc1empty[i], RT_EPI_WARPS);
      mbar_init(&a2full[i], RT_EPI_WARPS);
      mbar_init(&a2empty[i], 1);
      mbar_init(&acc2full[i], 1);
      mbar_init(&acc2empty[i], RT_EPI_WARPS / 2);
    }
    mbar_init(wfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int my_maps = nmaps > int(blockIdx.x) ? (nmaps - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int items = 8 * my_maps;
  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(wfull, uint32_t(HF_W1 + HF_W2));
      for (int t = 0; t < 9; ++t) {
        tma_load_2d(&mapW1, wfull, w1 + t * 32 * ROW_BYTES, t * 64, 0);
        tma_load_2d(&mapW2, wfull, w2 + t * 16 * ROW_BYTES, t * 64, 0);
      }
      for (int kt = 0; kt < items; ++kt) {
        const int s = kt & 1, t = kt & 7, n0 = int(blockIdx.x) + (kt >> 3) * int(gridDim.x);
        mbar_wait(&a1empty[s], ((kt >> 1) & 1) ^ 1);
        if (t == 0) {  // rows -1 .. 8
          mbar_expect_tx(&a1full[s], uint32_t(10 * HF_ROW));
          tma_load_4d(&mapA10, &a1full[s], a1 + s * HF_A1, 0, 0, -1, n0);
        } else {       // rows 4t .. 4t+5
          mbar_expect_tx(&a1full[s], uint32_t(6 * HF_ROW));
          tma_load_4d(&mapA6, &a1full[s], a1 + s * HF_A1, 0, 0, 4 * t, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc1 = make_idesc(KIND, BM, 96);
      constexpr uint32_t idesc2 = make_idesc(KIND, BM, 48);
      mbar_wait(wfull, 0);
      const uint32_t w1a = smem_u32(w1), w2a = smem_u32(w2);
      auto mma2 = [&](int kt) {  // head.deconv2 of item kt: 3 dy x 2 K steps
        const int b = kt & 1;
        mbar_wait(&a2full[b], (kt >> 1) & 1);
        mbar_wait(&acc2empty[b], ((kt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t a2a = smem_u32(a2 + b * HF_A2);
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            tc_mma<KIND>(tmem_base + HF_ACC2 + b * 48, sw128_desc(a2a + dy * HF_ROW + 32 * k),
                      sw128_desc(w2a + dy * 3 * 16 * ROW_BYTES + 32 * k), idesc2, (dy | k) ? 1u : 0u);
        tc_commit(&a2empty[b]);
        tc_commit(&acc2full[b]);
      };
      for (int kt = 0; kt < items; ++kt) {
        const int s = kt & 1, t = kt & 7;
        // head.deconv1 of item kt: 1 (item 0: 2) M blocks x 3 dy x 4 K steps
        mbar_wait(&a1full[s], (kt >> 1) & 1);
        mbar_wait(&acc1empty[s], ((kt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t a1a = smem_u32(a1 + s * HF_A1);
        const int nblk = t == 0 ? 2 : 1;
#pragma unroll 1
        for (int b = 0; b < nblk; ++b)
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int k = 0; k < ROW_BYTES / 32; ++k)
              tc_mma<KIND>(tmem_base + s * HF_ACC1 + b * 96,
                        sw128_desc(a1a + (4 * b + dy) * HF_ROW + 32 * k),
                        sw128_desc(w1a + dy * 3 * 32 * ROW_BYTES + 32 * k), idesc1, (dy | k) ? 1u : 0u);
        tc_commit(&a1empty[s]);
        tc_commit(&acc1full[s]);
        if (kt > 0) mma2(kt - 1);
      }
      if (items > 0) mma2(items - 1);
    }
  } else {
    const int q = warp & 3, grp = (warp - 2) / 4;
    const uint32_t tq = tmem_base + (uint32_t(q * 32) << 16);
    const uint32_t a2s = smem_u32(a2);
    const int c0 = 16 * grp, jb = 2 * grp;
    // one row of head.deconv1 outputs (this warp's 16 channels) into A2 slot
    auto put = [&](int buf, int slot, const uint32_t (&pk)[8]) {
      const int r = slot * 32 + lane;
      const uint32_t rowa = a2s + buf * HF_A2 + r * ROW_BYTES;
      sts128(rowa + (((jb + 0) ^ (r & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
      sts128(rowa + (((jb + 1) ^ (r & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
    };
    // folded BN vectors in registers: head.deconv1's 16 channels of this
    // warp, head.deconv2's 16 channels
    float e1a[16], e1b[16], e2a[16], e2b[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      e1a[i] = p1.ep_a[c0 + i];
      e1b[i] = p1.ep_b[c0 + i];
      e2a[i] = p2.ep_a[i];
      e2b[i] = p2.ep_b[i];
    }
    auto epi2 = [&](int kt) {  // head.deconv2 + conv_out of item kt (warp group kt & 1)
      const int b = kt & 1;
      if (grp != b) return;
      const int t = kt & 7, n0 = int(blockIdx.x) + (kt >> 3) * int(gridDim.x);
      mbar_wait(&acc2full[b], (kt >> 1) & 1);
      tc_fence_after();
      float acc[16];
      acc_chunk<16, true>(tq + HF_ACC2 + b * 48, 0, lane, 32, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc2empty[b]);
      // BN + LeakyReLU, then conv_out + ReLU (epilogue_tile's head branch)
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float x = acc[i] * e2a[i] + e2b[i];
        v[i] = x >= 0.f ? x : p2.slope * x;
      }
      const int pix = (4 * t + q) * 32 + lane;
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        float sum = p2.hw_b[o];
#pragma unroll
        for (int i = 0; i < 16; ++i) sum += p2.hw_w[o * 16 + i] * v[i];
        p2.pred[(int64_t(n0) * 3 + o) * 1024 + pix] = fmaxf(sum, 0.f);
      }
    };
    // a row of item kt-1 that item kt reuses (slot 4 / 5 -> slot 0 / 1),
    // kept in registers by the warp that computed it
    uint32_t carry[8];
    int carry_slot = -1;
    for (int kt = 0; kt < items; ++kt) {
      const int s = kt & 1, t = kt & 7;
      mbar_wait(&acc1full[s], (kt >> 1) & 1);
      mbar_wait(&a2empty[s], ((kt >> 1) & 1) ^ 1);  // head.deconv2 of item kt-2 has read A2[s]
      tc_fence_after();
      if (carry_slot >= 0) put(s, carry_slot, carry);
      carry_slot = -1;
      const int nblk = t == 0 ? 2 : 1;
#pragma unroll 1
      for (int b = 0; b < nblk; ++b) {
        // this quarter's head.deconv1 row: item 0 block b -> row 4b + q,
        // else row 4t + 1 + q
        const int row = t == 0 ? 4 * b + q : 4 * t + 1 + q;
        if (t == 0 && b == 1 && q > 0) {
          if (q == 1) {  // row -1 (slot 0 of item 0) is the map's zero padding
            const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            put(s, 0, z);
          }
          continue;  // rows 5..7 of item 0 are recomputed by item 1
        }
        float acc[16], v[16];
        acc_chunk<32, true>(tq + s * HF_ACC1 + b * 96, c0, lane, 32, acc);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x = acc[i] * e1a[i] + e1b[i];
          v[i] = x >= 0.f ? x : p1.slope * x;
        }
        const bool inside = row < 32;
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = pack2<KIND>(inside ? v[2 * i] : 0.f, inside ? v[2 * i + 1] : 0.f);
        const int slot = row - (4 * t - 1);  // slot in this item's A2 (rows 4t-1 ..)
        put(s, slot, pk);
        // rows 4t+3, 4t+4 are rows 4(t+1)-1, 4(t+1) of the next item
        if (t < 7 && (slot == 4 || slot == 5)) {
          carry_slot = slot - 4;
#pragma unroll
          for (int i = 0; i < 8; ++i) carry[i] = pk[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc1empty[s]);
      fence_proxy_async();  // A2 is read by the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&a2full[s]);
      if (kt > 0) epi2(kt - 1);
    }
    if (items > 0) epi2(items - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u));
  }
}
constexpr size_t head_fused_smem() {
  return 1024 + size_t(HF_W1) + HF_W2 + 2 * size_t(HF_A1) + 2 * size_t(HF_A2) + 256;
}

// ---------------------------------------------------------------------------
// CTA-pair row-tile conv (tcgen05.mma.cta_group::2, M = 256): the
// streamed-weight dx layers (dec1.deconv1 @32x32, dec2.deconv1 @16x16).
// A work tile is 256 output pixels; CTA rank r of the pair owns M rows
// [128 r, 128 r + 128) (its A box, its TMEM accumulator, its epilogue and
// store), and half of the N = 3 BN stacked dx weight rows ([1.5 BN r,
// 1.5 BN (r + 1))). Per SM that is the single-CTA kernel's A traffic with half
// its B traffic and B operand reads, and an accumulator of 3 BN columns per
// CTA, so two of them fit in TMEM: the epilogue of tile i overlaps the MMAs
// of tile i + 1 (the one-CTA MH = 2 kernel holds 6 BN columns per tile and
// must drain before the next tile starts).
//   both CTAs, warp 0: TMA producer (its own A box and B half; completion
//                      is signalled on the LEADER's full barriers)
//   leader, warp 1:    MMA issue (one thread), commits multicast to both
//   both CTAs, 2-9:    epilogue (arrive on the leader's TMEM-empty barrier)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_4d_cg2(const CUtensorMap* map, uint32_t bar_cluster, void* dst,
                                                int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_cg2(const CUtensorMap* map, uint32_t bar_cluster, void* dst,
                                                int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at the same SMEM offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}

template <int KIND, int BN, bool RES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RT_THREADS, 1)
    k_conv_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const __grid_constant__ CUtensorMap mapO, const __grid_constant__ ConvArgs p,
                const __grid_constant__ RowArgs h) {
  pdl_wait();
  static_assert(KIND != 1, "16-bit operands");
  constexpr int ELEM = 2;
  constexpr int CEL = ROW_BYTES / ELEM;
  static_assert(BN == CEL, "one 128-B staging sub-tile per pixel");
  constexpr int N = 3 * BN;                  // stacked dx accumulators per CTA row
  constexpr int BHALF = N / 2 * ROW_BYTES;   // this CTA's half of a (cb, dy) triple
  constexpr int BCH = BN / 2;                // rows per B box
  constexpr uint32_t TMEM_COLS = 2 * N <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // RES: this CTA's weight half stays resident, [cb][dy] triples
  uint8_t* wres = smem;
  uint8_t* aring = smem + (RES ? p.cblocks * 3 * BHALF : 0);
  uint8_t* bring = aring + h.sa * h.a_bytes;
  uint8_t* ostage = bring + (RES ? 0 : h.sb * BHALF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ostage + 2 * h.o_bytes);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + 8;
  uint64_t* bfull = bars + 16;
  uint64_t* bempty = bars + 24;
  uint64_t* tfull = bars + 32;
  uint64_t* tempty = bars + 34;
  uint64_t* wfull = bars + 36;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 37);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    for (int s = 0; s < h.sa; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < h.sb; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * RT_EPI_WARPS);  // both CTAs' epilogue warps
    }
    mbar_init(wfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.num_m_tiles;  // one N tile (cout = BN)
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int rows_cta = BM / p.hw;
  if (warp == 0) {
    if (lane == 0) {
      if (RES) {
        if (leader) mbar_expect_tx(wfull, uint32_t(2 * p.cblocks * 3 * BHALF));
        const uint32_t fw = mapa_rank(smem_u32(wfull), 0);
        for (int cb = 0; cb < p.cblocks; ++cb)
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const int s = int(rank) * (N / 2) + j * BCH;
              const int tap = dy * 3 + s / BN;
              tma_load_2d_cg2(&mapB, fw, wres + (cb * 3 + dy) * BHALF + j * BCH * ROW_BYTES,
                              (tap * p.cblocks + cb) * CEL, s % BN);
            }
      }
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        const int n0 = tile / p.tiles_per_map;
        const int y0 = (tile % p.tiles_per_map) * p.rows_per_tile + int(rank) * rows_cta;
        for (int cb = 0; cb < p.cblocks; ++cb) {
          mbar_wait(&aempty[sa], pa ^ 1);
          if (leader) mbar_expect_tx(&afull[sa], uint32_t(2 * h.a_bytes));
          tma_load_4d_cg2(&mapA, mapa_rank(smem_u32(&afull[sa]), 0), aring + sa * h.a_bytes, cb * CEL, 0,
                          y0 - 1, n0);
          if (++sa == h.sa) {
            sa = 0;
            pa ^= 1;
          }
          if (!RES)
          for (int dy = 0; dy < 3; ++dy) {
            mbar_wait(&bempty[sb], pb ^ 1);
            if (leader) mbar_expect_tx(&bfull[sb], uint32_t(2 * BHALF));
            const uint32_t fb = mapa_rank(smem_u32(&bfull[sb]), 0);
            uint8_t* dst = bring + sb * BHALF;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const int s = int(rank) * (N / 2) + j * BCH;  // stacked row: dx * BN + co
              const int tap = dy * 3 + s / BN;
              tma_load_2d_cg2(&mapB, fb, dst + j * BCH * ROW_BYTES, (tap * p.cblocks + cb) * CEL, s % BN);
            }
            if (++sb == h.sb) {
              sb = 0;
              pb ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, 2 * BM, N);
      if (RES) mbar_wait(wfull, 0);
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        bool first = true;
        for (int cb = 0; cb < p.cblocks; ++cb) {
          mbar_wait(&afull[sa], pa);
          tc_fence_after();
          const uint32_t a0 = smem_u32(aring + sa * h.a_bytes);
#pragma unroll 1
          for (int dy = 0; dy < 3; ++dy) {
            uint32_t bb;
            if (RES) {
              bb = smem_u32(wres + (cb * 3 + dy) * BHALF);
            } else {
              mbar_wait(&bfull[sb], pb);
              tc_fence_after();
              bb = smem_u32(bring + sb * BHALF);
            }
            const uint32_t aa = a0 + dy * h.row_bytes;
#pragma unroll
            for (int k = 0; k < ROW_BYTES / 32; ++k) {
              tc_mma_cg2(tmem_d, sw128_desc(aa + 32 * k), sw128_desc(bb + 32 * k), idesc, first ? 0u : 1u);
              first = false;
            }
            if (!RES) {
              tc_commit_cg2(&bempty[sb]);
              if (++sb == h.sb) {
                sb = 0;
                pb ^= 1;
              }
            }
          }
          tc_commit_cg2(&aempty[sa]);
          if (++sa == h.sa) {
            sa = 0;
            pa ^= 1;
          }
        }
        tc_commit_cg2(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int grp = (warp - 2) / 4;
    constexpr int CSTEP = 16 * (RT_EPI_WARPS / 4);
    float* s_ep = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);
    stage_ep(p, BN, s_ep, threadIdx.x - 64, 32 * RT_EPI_WARPS);
    epi_bar_rt();
    const uint32_t sep = smem_u32(s_ep);
    int acc = 0, obuf = 0;
    uint32_t acc_phase = 0;
    for (int tile = pair; tile < num_tiles; tile += npairs) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase0 = tmem_base + (uint32_t(q * 32) << 16) + acc * N;
      uint8_t* ot = ostage + obuf * h.o_bytes;
      const bool issuer = grp == 0 && lane == 0;  // per lane quarter (32 pixel rows)
      if (issuer) bulk_wait_read1();  // this quarter's store of 2 tiles ago has read ot
      quarter_bar(q);
      epilogue_stage<KIND, BN, true, CSTEP>(p, tbase0, (int64_t(tile) * 2 + rank) * BM + row, 0, ot,
                                            16 * grp, sep);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_rank(smem_u32(&tempty[acc]), 0));
      fence_proxy_async();
      quarter_bar(q);
      if (issuer) {
        const int n0 = tile / p.tiles_per_map;
        const int y0 = (tile % p.tiles_per_map) * p.rows_per_tile + int(rank) * rows_cta;
        tma_store_4d(&mapO, ot + q * 32 * ROW_BYTES, p.cout_off, 0, y0 + q * 32 / p.hw, n0);
        bulk_commit();
      }
      obuf ^= 1;
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0 && grp == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// enc1.conv1 (7 -> 64 channels @ 32x32) from the compact network input: NHWC
// with 8 channels per pixel (7 + one zero), 16 B (bf16) / 32 B (tf32) per
// pixel, 1/8 of a channel-padded layout's bytes. The im2col operand is built
// in SMEM: K value tap*8 + c of pixel (y, x) is channel c of pixel
// (y + tap/3 - 1, x + tap%3 - 1); 9 taps x 8 = 72 K values, zero-padded to
// whole 128-B swizzle rows (bf16: 2 K chunks, tf32: 3).
//   warp 0: TMA of the tile's input rows y0-1 .. y0+4 (OOB rows = 0)
//   warp 1: tcgen05.mma (M = 128, N = 64) into double-buffered TMEM
//   warps 2-5: build the im2col tile (one pixel per thread, 9 x 16-B pieces
//              per tap group; the x border is zeroed here)
//   warps 6-9: folded BN + LeakyReLU epilogue staged in SMEM, TMA store
constexpr int IN8_THREADS = 320;
constexpr int IN8_SI = 4, IN8_SA = 2;

template <int KIND>
__global__ void __launch_bounds__(IN8_THREADS, 1)
    k_conv_in8(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapB,
               const __grid_constant__ CUtensorMap mapO, const __grid_constant__ ConvArgs p) {
  pdl_wait();
  constexpr int ELEM = elem_bytes(KIND);
  constexpr int PX_BYTES = 8 * ELEM;                  // one input pixel
  constexpr int PPT = PX_BYTES / 16;                  // 16-B pieces per tap
  constexpr int NCH = (72 * ELEM + ROW_BYTES - 1) / ROW_BYTES;  // K chunks
  constexpr int BN = 64;
  constexpr int IN_BYTES = 6 * 32 * PX_BYTES;         // rows y0-1 .. y0+4
  constexpr int A_BYTES = NCH * BM * ROW_BYTES;
  constexpr int W_BYTES = NCH * BN * ROW_BYTES;
  constexpr int O_BYTES = BM * BN * ELEM;
  constexpr int CEL = ROW_BYTES / ELEM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                          // IN8_SA x A_BYTES
  uint8_t* sw = sa + IN8_SA * A_BYTES;         // W_BYTES
  uint8_t* so = sw + W_BYTES;                  // 2 x O_BYTES
  uint8_t* si = so + 2 * O_BYTES;              // IN8_SI x IN_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(si + IN8_SI * IN_BYTES);
  uint64_t* ifull = bars;
  uint64_t* iempty = bars + IN8_SI;
  uint64_t* afull = bars + 2 * IN8_SI;
  uint64_t* aempty = afull + IN8_SA;
  uint64_t* tfull = aempty + IN8_SA;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapX);
    prefetch_map(&mapB);
    for (int i = 0; i < IN8_SI; ++i) {
      mbar_init(&ifull[i], 1);
      mbar_init(&iempty[i], 4);
    }
    for (int i = 0; i < IN8_SA; ++i) {
      mbar_init(&afull[i], 4);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    mbar_init(wfull, 1);
    fence_barrier_init();
  }
  if (warp >= 2 && warp < 6) {
    // pieces no input pixel is scattered to (never rewritten): the K padding
    // and the x-border taps (dx = -1 at x = 0, dx = +1 at x = 31, the conv's
    // zero padding); zero them once in every A stage
    const int r = threadIdx.x - 64, x = r & 31;
    for (int st = 0; st < IN8_SA; ++st)
      for (int j = 0; j < NCH * 8; ++j) {
        const int t = j / PPT;
        const bool pad = j >= 9 * PPT || (x == 0 && t % 3 == 0) || (x == 31 && t % 3 == 2);
        if (pad)
          sts128(smem_u32(sa + st * A_BYTES + (j >> 3) * (BM * ROW_BYTES) + r * ROW_BYTES) +
                     (((j & 7) ^ (r & 7)) << 4),
                 0u, 0u, 0u, 0u);
      }
    fence_proxy_async();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.num_m_tiles;
  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(wfull, uint32_t(W_BYTES));
      for (int c = 0; c < NCH; ++c) tma_load_2d(&mapB, wfull, sw + c * BN * ROW_BYTES, c * CEL, 0);
      int st = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&iempty[st], ph ^ 1);
        mbar_expect_tx(&ifull[st], uint32_t(IN_BYTES));
        tma_load_4d(&mapX, &ifull[st], si + st * IN_BYTES, 0, 0, (tile & 7) * 4 - 1, tile >> 3);
        if (++st == IN8_SI) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(KIND, BM, BN);
      mbar_wait(wfull, 0);
      int st = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);
        mbar_wait(&afull[st], ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sa + st * A_BYTES), b0 = smem_u32(sw);
        // K steps of 32 B that hold real taps: the last chunk holds only tap 8
        // (its other steps would multiply zero padding)
        constexpr int KLAST = (72 * ELEM - (NCH - 1) * ROW_BYTES + 31) / 32;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int k = 0; k < (c == NCH - 1 ? KLAST : ROW_BYTES / 32); ++k)
            tc_mma<KIND>(tmem_base + acc * BN, sw128_desc(a0 + c * BM * ROW_BYTES + 32 * k),
                         sw128_desc(b0 + c * BN * ROW_BYTES + 32 * k), idesc, (c | k) ? 1u : 0u);
        tc_commit(&aempty[st]);
        tc_commit(&tfull[acc]);
        if (++st == IN8_SA) {
          st = 0;
          ph ^= 1;
        }
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp < 6) {
    // im2col builders, scatter form: each input pixel (6 rows y0-1 .. y0+4 of
    // 32) is read once and written to the (up to) 9 output pixels whose taps
    // it feeds: output (ry, x) tap t = (dy, dx) is input (ry + dy, x + dx - 1);
    // the x-border taps stay zero (zeroed once above), the y border comes
    // zero from the TMA (OOB rows)
    const int b = threadIdx.x - 64;
    int ist = 0, ast = 0;
    uint32_t iph = 0, aph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&ifull[ist], iph);
      mbar_wait(&aempty[ast], aph ^ 1);
      const uint32_t src = smem_u32(si + ist * IN_BYTES);
      const uint32_t dst = smem_u32(sa + ast * A_BYTES);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = b + 128 * h;  // input pixel of the tile's 6 x 32 window
        if (k >= 6 * 32) break;     // warp-uniform (k multiple of 32 per warp)
        const int iy = k >> 5, ix = k & 31;
#pragma unroll
        for (int qq = 0; qq < PPT; ++qq) {
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                       : "r"(src + k * PX_BYTES + 16 * qq));
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const int ry = iy - t / 3, x = ix - t % 3 + 1;
            if (ry < 0 || ry > 3 || x < 0 || x > 31) continue;
            const int r = ry * 32 + x, j = t * PPT + qq;
            sts128(dst + (j >> 3) * (BM * ROW_BYTES) + r * ROW_BYTES + (((j & 7) ^ (r & 7)) << 4), v0, v1,
                   v2, v3);
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&iempty[ist]);
        mbar_arrive(&afull[ast]);
      }
      if (++ist == IN8_SI) {
        ist = 0;
        iph ^= 1;
      }
      if (++ast == IN8_SA) {
        ast = 0;
        aph ^= 1;
      }
    }
  } else {
    // epilogue warps 6..9 -> TMEM lane quarter warp % 4
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int acc = 0, obuf = 0;
    uint32_t aph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int64_t m = int64_t(tile) * BM + row;
      uint8_t* ot = so + obuf * O_BYTES;
      // one warp per lane quarter = one image row: the warp stages and
      // TMA-stores its own 32 pixels (no barrier across the epilogue warps)
      if (lane == 0) bulk_wait_read1();  // this warp's store of 2 tiles ago has read ot
      __syncwarp();
      epilogue_stage<KIND, BN, false, 16>(p, tmem_base + (uint32_t(q * 32) << 16) + acc * BN, m, 0,
                                          ot, 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        for (int sb = 0; sb < BN / CEL; ++sb)
          tma_store_4d(&mapO, ot + (sb * BM + q * 32) * ROW_BYTES, p.cout_off + sb * CEL, 0,
                       (tile & 7) * 4 + q, tile >> 3);
        bulk_commit();
      }
      obuf ^= 1;
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128u));
  }
}

template <int KIND>
constexpr size_t in8_smem() {
  constexpr int ELEM = elem_bytes(KIND);
  constexpr int NCH = (72 * ELEM + ROW_BYTES - 1) / ROW_BYTES;
  return 1024 + size_t(IN8_SA) * NCH * BM * ROW_BYTES + size_t(NCH) * 64 * ROW_BYTES +
         2 * size_t(BM) * 64 * ELEM + size_t(IN8_SI) * 6 * 32 * 8 * ELEM + 256;
}

// ---------------------------------------------------------------------------
// NHWC helper kernels (element type T = bf16 or fp32)
template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <>
__device__ __forceinline__ float ldf<__half>(const __half* p) { return __half2float(*p); }
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <typename T>
__device__ __forceinline__ T stf(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 stf<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half stf<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ float stf<float>(float v) { return round_tf32(v); }

// 16-byte vectors of 8 bf16 / 4 fp32 channels
template <typename T>
struct Vec {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void unpack(const uint4& u, float* f);
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t = __bfloat1622float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void unpack<__half>(const uint4& u, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t = __half22float2(h[j]);
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void unpack<float>(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x);
  f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z);
  f[3] = __uint_as_float(u.w);
}
template <typename T>
__device__ __forceinline__ uint4 pack(const float* f);
template <>
__device__ __forceinline__ uint4 pack<__nv_bfloat16>(const float* f) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&b);
  }
  return u;
}
template <>
__device__ __forceinline__ uint4 pack<__half>(const float* f) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) w[j] = pack2<2>(f[2 * j], f[2 * j + 1]);
  return u;
}
template <>
__device__ __forceinline__ uint4 pack<float>(const float* f) {
  return make_uint4(__float_as_uint(round_tf32(f[0])), __float_as_uint(round_tf32(f[1])),
                    __float_as_uint(round_tf32(f[2])), __float_as_uint(round_tf32(f[3])));
}

// NCHW fp32 stack (n,7,32,32) -> compact NHWC network input (n_pad,32,32,8),
// channel 7 and padding maps zero; one thread per (pixel, 16-B piece)
template <typename T>
__global__ void k_stack_to_nhwc(const float* __restrict__ x, int64_t n, int64_t n_pad, int,
                                T* __restrict__ out) {
  pdl_wait();
  constexpr int V = Vec<T>::N;   // channels per 16-B piece
  constexpr int PP = 8 / V;      // pieces per pixel
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad * 1024 * PP) return;
  const int piece = int(i % PP);
  const int64_t px = i / PP;
  const int64_t map = px / 1024;
  const int pix = int(px % 1024);
  float f[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c = piece * V + j;
    f[j] = (c < 7 && map < n) ? __ldg(x + (map * 7 + c) * 1024 + pix) : 0.f;
  }
  reinterpret_cast<uint4*>(out)[i] = pack<T>(f);
}

// 2x2 max-pool of channel slice [off, off+C) of an NHWC buffer
// (cnn.py:152-156); compile-time shapes, one thread per (output pixel,
// 4 x 16 B channel groups)
template <typename T, int HW_OUT, int C>
__global__ void __launch_bounds__(256) k_pool_nhwc(const T* __restrict__ in, int c_tot, int off,
                                                   T* __restrict__ out, int64_t nmaps) {
  pdl_wait();
  constexpr int V = Vec<T>::N;
  constexpr int G = C / V;          // 16 B groups per pixel
  constexpr int GPT = G >= 4 ? 4 : G;  // groups per thread
  constexpr int TPP = G / GPT;       // threads per pixel
  constexpr int HI = 2 * HW_OUT;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nmaps * HW_OUT * HW_OUT * TPP) return;
  const int gq = int(i % TPP);
  const int64_t px = i / TPP;
  const int x = int(px % HW_OUT), y = int((px / HW_OUT) % HW_OUT);
  const int64_t n = px / (HW_OUT * HW_OUT);
  const T* p = in + ((n * HI + 2 * y) * HI + 2 * x) * c_tot + off;
  T* o = out + px * C;
#pragma unroll
  for (int k = 0; k < GPT; ++k) {
    const int g = k * TPP + gq;  // a pixel's threads cover adjacent 16-B groups (full sectors)
    float a[V], b[V], cc[V], d[V], m[V];
    unpack<T>(__ldg(reinterpret_cast<const uint4*>(p + g * V)), a);
    unpack<T>(__ldg(reinterpret_cast<const uint4*>(p + c_tot + g * V)), b);
    unpack<T>(__ldg(reinterpret_cast<const uint4*>(p + HI * c_tot + g * V)), cc);
    unpack<T>(__ldg(reinterpret_cast<const uint4*>(p + (HI + 1) * c_tot + g * V)), d);
#pragma unroll
    for (int j = 0; j < V; ++j) m[j] = fmaxf(fmaxf(a[j], b[j]), fmaxf(cc[j], d[j]));
    *reinterpret_cast<uint4*>(o + g * V) = pack<T>(m);
  }
}

// bilinear 2x (align_corners=False) of an NHWC buffer (C channels) into the
// leading channel slice of the decoder concat buffer (cnn.py:159-174), rows
// then columns like the reference. One thread per (2x2 output block, 16-B
// channel group), groups fastest: the 3x3 input neighbourhood is loaded once
// for four outputs and a warp's stores cover whole 32-B sectors.
template <typename T, int HW_IN, int C>
__global__ void __launch_bounds__(256) k_up_nhwc(const T* __restrict__ in, T* __restrict__ out,
                                                 int c_tot, int64_t nmaps) {
  pdl_wait();
  constexpr int V = Vec<T>::N;
  constexpr int G = C / V;
  constexpr int HO = 2 * HW_IN;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nmaps * HW_IN * HW_IN * G) return;
  const int g = int(t % G) * V;
  const int64_t blk = t / G;
  const int j = int(blk % HW_IN), i = int((blk / HW_IN) % HW_IN);
  const int64_t n = blk / (HW_IN * HW_IN);
  const T* b = in + n * HW_IN * HW_IN * C + g;
  if constexpr (sizeof(T) == 2) {
    // bf16 / fp16: packed mixing (up_mix_h2), the same arithmetic as the
    // upsample fused into dec2.deconv2's epilogue
    using H2 = typename std::conditional<std::is_same<T, __half>::value, __half2, __nv_bfloat162>::type;
    uint4 nbq[3][3];
#pragma unroll
    for (int dr = 0; dr < 3; ++dr) {
      const int r = min(max(i + dr - 1, 0), HW_IN - 1);
#pragma unroll
      for (int dc = 0; dc < 3; ++dc) {
        const int c = min(max(j + dc - 1, 0), HW_IN - 1);
        nbq[dr][dc] = __ldg(reinterpret_cast<const uint4*>(b + (r * HW_IN + c) * C));
      }
    }
    const float fr_even = i == 0 ? 0.f : 0.75f, fc_even = j == 0 ? 0.f : 0.75f;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const float fr = a ? 0.25f : fr_even;
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const float fc = bb ? 0.25f : fc_even;
        const uint4 q[4] = {nbq[a][bb], nbq[a + 1][bb], nbq[a][bb + 1], nbq[a + 1][bb + 1]};
        uint32_t o[4];
        up_mix_h2<H2>(q, 1.f - fr, fr, 1.f - fc, fc, o);
        const int64_t px = (n * HO + 2 * i + a) * HO + 2 * j + bb;
        *reinterpret_cast<uint4*>(out + px * c_tot + g) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  } else {
  // neighbourhood rows/cols i-1, i, i+1 (clamped; up_w only selects in-range ones)
  float nb[3][3][V];
#pragma unroll
  for (int dr = 0; dr < 3; ++dr) {
    const int r = min(max(i + dr - 1, 0), HW_IN - 1);
#pragma unroll
    for (int dc = 0; dc < 3; ++dc) {
      const int c = min(max(j + dc - 1, 0), HW_IN - 1);
      unpack<T>(__ldg(reinterpret_cast<const uint4*>(b + (r * HW_IN + c) * C)), nb[dr][dc]);
    }
  }
  // up_w in neighbourhood coordinates with compile-time indices: even
  // output 2i -> rows (i-1, i), weight 0.75 (0 at i = 0, where the clamped
  // row i-1 is row 0 and the result is row 0 exactly as in the reference);
  // odd 2i+1 -> rows (i, i+1 clamped), weight 0.25
  const float fr_even = i == 0 ? 0.f : 0.75f, fc_even = j == 0 ? 0.f : 0.75f;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const float fr = a ? 0.25f : fr_even, omr = 1.f - fr;
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const float fc = bb ? 0.25f : fc_even, omc = 1.f - fc;
      float v[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        float t0 = __fadd_rn(__fmul_rn(nb[a][bb][e], omr), __fmul_rn(nb[a + 1][bb][e], fr));
        float t1 = __fadd_rn(__fmul_rn(nb[a][bb + 1][e], omr), __fmul_rn(nb[a + 1][bb + 1][e], fr));
        v[e] = __fadd_rn(__fmul_rn(t0, omc), __fmul_rn(t1, fc));
      }
      const int64_t px = (n * HO + 2 * i + a) * HO + 2 * j + bb;
      *reinterpret_cast<uint4*>(out + px * c_tot + g) = pack<T>(v);
    }
  }
  }
}

template <typename T, int HW_OUT, int C>
void launch_pool(const T* in, int c_tot, int off, T* out, int64_t nmaps, cudaStream_t st) {
  constexpr int G = C / Vec<T>::N;
  constexpr int TPP = G / (G >= 4 ? 4 : G);
  int64_t tot = nmaps * HW_OUT * HW_OUT * TPP;
  launch_pdl(k_pool_nhwc<T, HW_OUT, C>, unsigned((tot + 255) / 256), 256, 0, st, in, c_tot, off, out, nmaps);
  count_launch();
}

template <typename T, int HW_IN, int C>
void launch_up(const T* in, T* out, int c_tot, int64_t nmaps, cudaStream_t st) {
  int64_t tot = nmaps * HW_IN * HW_IN * (C / Vec<T>::N);
  launch_pdl(k_up_nhwc<T, HW_IN, C>, unsigned((tot + 255) / 256), 256, 0, st, in, out, c_tot, nmaps);
  count_launch();
}

// shapes of the k = 64 / k = 32 U-Nets
template <typename T>
int pool_dispatch(const T* in, int c_tot, int off, int c, int hw_out, T* out, int64_t n,
                  cudaStream_t st) {
  if (hw_out == 16 && c == 64) launch_pool<T, 16, 64>(in, c_tot, off, out, n, st);
  else if (hw_out == 8 && c == 128) launch_pool<T, 8, 128>(in, c_tot, off, out, n, st);
  else if (hw_out == 4 && c == 256) launch_pool<T, 4, 256>(in, c_tot, off, out, n, st);
  else if (hw_out == 16 && c == 32) launch_pool<T, 16, 32>(in, c_tot, off, out, n, st);
  else if (hw_out == 8 && c == 64) launch_pool<T, 8, 64>(in, c_tot, off, out, n, st);
  else if (hw_out == 4 && c == 128) launch_pool<T, 4, 128>(in, c_tot, off, out, n, st);
  else return fail(DRCB_ECONFIG, "unsupported pool shape");
  return 0;
}

template <typename T>
int up_dispatch(const T* in, int c, int hw_in, T* out, int c_tot, int64_t n, cudaStream_t st) {
  if (hw_in == 4 && c == 512) launch_up<T, 4, 512>(in, out, c_tot, n, st);
  else if (hw_in == 8 && c == 256) launch_up<T, 8, 256>(in, out, c_tot, n, st);
  else if (hw_in == 16 && c == 128) launch_up<T, 16, 128>(in, out, c_tot, n, st);
  else if (hw_in == 4 && c == 256) launch_up<T, 4, 256>(in, out, c_tot, n, st);
  else if (hw_in == 8 && c == 128) launch_up<T, 8, 128>(in, out, c_tot, n, st);
  else if (hw_in == 16 && c == 64) launch_up<T, 16, 64>(in, out, c_tot, n, st);
  else return fail(DRCB_ECONFIG, "unsupported upsample shape");
  return 0;
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

CUtensorMapDataType tmap_dtype(int kind) {
  return kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                   : (kind == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// NHWC activation box of `box_c` channels (box_c * elem bytes = 32 / 64 /
// 128 B rows, swizzled at that width) x box_w x box_h x box_n
// (pitch: elements between pixels when the tensor is stored narrower than
// c_tot; 0 = c_tot)
int encode_act_c(CUtensorMap* m, const void* base, int kind, int c_tot, int hw, int64_t nmaps,
                 int box_c, int box_w, int box_h, int box_n, int pitch = 0) {
  auto enc = get_encode();
  if (!enc) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = elem_bytes(kind);
  const int rb = box_c * es;
  if (rb != 32 && rb != 64 && rb != 128) return fail(DRCB_ECONFIG, "activation box rows must be 32, 64 or 128 B");
  const int pc = pitch > 0 ? pitch : c_tot;
  cuuint64_t dims[4] = {cuuint64_t(std::min(c_tot, pc)), cuuint64_t(hw), cuuint64_t(hw), cuuint64_t(nmaps)};
  cuuint64_t strides[3] = {cuuint64_t(pc) * es, cuuint64_t(pc) * es * hw, cuuint64_t(pc) * es * hw * hw};
  cuuint32_t box[4] = {cuuint32_t(box_c), cuuint32_t(box_w), cuuint32_t(box_h), cuuint32_t(box_n)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle sw = rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(m, tmap_dtype(kind), 4,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled(activation) failed: " + std::to_string(int(r)));
  return 0;
}

// c_dim (0 = c_tot): channels that hold data; the box's channels beyond it
// are the TMA unit's out-of-bounds zero fill on loads (not read from HBM)
// and are dropped on stores. pitch (0 = c_tot): elements between pixels, for
// a tensor stored narrower than the 64-channel boxes (the training engine's
// 32- / 16-channel head layers)
int encode_act(CUtensorMap* m, const void* base, int kind, int c_tot, int hw, int64_t nmaps,
               int box_w, int box_h, int box_n, int c_dim = 0, int pitch = 0) {
  auto enc = get_encode();
  if (!enc) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = elem_bytes(kind);
  const int pc = pitch > 0 ? pitch : c_tot;
  const int cd = std::min(c_dim > 0 ? c_dim : c_tot, pc);
  cuuint64_t dims[4] = {cuuint64_t(cd), cuuint64_t(hw), cuuint64_t(hw), cuuint64_t(nmaps)};
  cuuint64_t strides[3] = {cuuint64_t(pc) * es, cuuint64_t(pc) * es * hw, cuuint64_t(pc) * es * hw * hw};
  cuuint32_t box[4] = {cuuint32_t(ROW_BYTES / es), cuuint32_t(box_w), cuuint32_t(box_h), cuuint32_t(box_n)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, tmap_dtype(kind), 4,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled(activation) failed: " + std::to_string(int(r)));
  return 0;
}

int encode_w(CUtensorMap* m, const void* base, int kind, int64_t k_tot, int rows, int bn) {
  auto enc = get_encode();
  if (!enc) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = elem_bytes(kind);
  cuuint64_t dims[2] = {cuuint64_t(k_tot), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(k_tot) * es};
  cuuint32_t box[2] = {cuuint32_t(ROW_BYTES / es), cuuint32_t(bn)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, tmap_dtype(kind), 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled(weights) failed: " + std::to_string(int(r)));
  return 0;
}

float host_round_tf32(float v) {
  uint32_t i;
  std::memcpy(&i, &v, 4);
  if ((i & 0x7f800000u) != 0x7f800000u) i = (i + 0x1000u) & 0xffffe000u;  // nearest, ties away
  float r;
  std::memcpy(&r, &i, 4);
  return r;
}

int pad_c(int c, int kind) {
  int g = ROW_BYTES / elem_bytes(kind);
  return ((c + g - 1) / g) * g;
}

// pack conv-form weights (cout, cin, 3, 3) into K-major (cout_pad, 9*cin_pad)
int prepare_layer(NetImpl& net, ConvLayer& L, int kind) {
  if (L.tc_kind == kind) return 0;
  L.in8 = (L.name == "enc1.conv1" && L.cin <= 8);
  // in8: K = 9 taps x 8 channels rounded up to whole 128-B rows
  const int cinp = L.in8 ? ((72 * elem_bytes(kind) + ROW_BYTES - 1) / ROW_BYTES) * (ROW_BYTES / elem_bytes(kind))
                         : pad_c(L.cin, kind);
  // output channels are padded to the next layer's K granularity; padded
  // channels get zero weights and zero epilogue vectors, so they hold exact
  // zeros (head.deconv1's k/2 outputs feed a K-padded input). The fused head
  // layer only needs the UMMA minimum N of 16.
  // A row-tile layer (hw >= 16) with fewer outputs than one 128-B row
  // (bf16 head.deconv1: 32) computes N = cout rounded to 16 and its epilogue
  // zero-fills the rest of the row, which the next layer's K padding reads.
  const int cel = ROW_BYTES / elem_bytes(kind);
  const int coutp = (L.name == "head.deconv2") ? 16
                    : (L.hw >= 16 && L.cout < cel && L.name != "enc1.conv1") ? (L.cout + 15) / 16 * 16
                                                    : pad_c(L.cout, kind);
  L.cin_pad = cinp;
  L.cout_pad = coutp;
  const int64_t ktot = L.in8 ? cinp : int64_t(9) * cinp;
  // K index of (input channel ci, tap t) in the packed operand
  auto kidx = [&](int ci, int t) -> int64_t { return L.in8 ? t * 8 + ci : int64_t(t) * cinp + ci; };
  std::vector<float> a(coutp, 0.f), b(coutp, 0.f);
  for (int c = 0; c < L.cout; ++c) {
    a[c] = L.scale[c];
    b[c] = L.bias[c] * L.scale[c] + L.shift[c];
  }
  size_t nel = size_t(coutp) * ktot;
  void* dw = nullptr;
  if (kind == 0) {
    std::vector<__nv_bfloat16> w(nel, __float2bfloat16(0.f));
    for (int co = 0; co < L.cout; ++co)
      for (int ci = 0; ci < L.cin; ++ci)
        for (int t = 0; t < 9; ++t)
          w[size_t(co) * ktot + kidx(ci, t)] = __float2bfloat16(L.w[(size_t(co) * L.cin + ci) * 9 + t]);
    if (cudaMalloc(&dw, nel * 2) != cudaSuccess) return fail(DRCB_ECUDA, "cudaMalloc weights");
    cudaMemcpy(dw, w.data(), nel * 2, cudaMemcpyHostToDevice);
  } else if (kind == 2) {
    std::vector<__half> w(nel, __float2half_rn(0.f));
    for (int co = 0; co < L.cout; ++co)
      for (int ci = 0; ci < L.cin; ++ci)
        for (int t = 0; t < 9; ++t)
          w[size_t(co) * ktot + kidx(ci, t)] = __float2half_rn(L.w[(size_t(co) * L.cin + ci) * 9 + t]);
    if (cudaMalloc(&dw, nel * 2) != cudaSuccess) return fail(DRCB_ECUDA, "cudaMalloc weights");
    cudaMemcpy(dw, w.data(), nel * 2, cudaMemcpyHostToDevice);
  } else {
    std::vector<float> w(nel, 0.f);
    for (int co = 0; co < L.cout; ++co)
      for (int ci = 0; ci < L.cin; ++ci)
        for (int t = 0; t < 9; ++t)
          w[size_t(co) * ktot + kidx(ci, t)] = host_round_tf32(L.w[(size_t(co) * L.cin + ci) * 9 + t]);
    if (cudaMalloc(&dw, nel * 4) != cudaSuccess) return fail(DRCB_ECUDA, "cudaMalloc weights");
    cudaMemcpy(dw, w.data(), nel * 4, cudaMemcpyHostToDevice);
  }
  net.allocs.push_back(dw);
  L.d_wtc = dw;
  float *da = nullptr, *db = nullptr;
  cudaMalloc(&da, coutp * 4);
  cudaMalloc(&db, coutp * 4);
  net.allocs.push_back(da);
  net.allocs.push_back(db);
  cudaMemcpy(da, a.data(), coutp * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), coutp * 4, cudaMemcpyHostToDevice);
  L.d_ep_a = da;
  L.d_ep_b = db;
  L.tc_kind = kind;
  return 0;
}

// SMs the persistent tensor-core kernels spread over (DRCB_CONV_SMS caps it:
// an A/B of the U-Net's throughput on fewer SMs under the power limit)
inline int conv_sms() {
  const int nsm = sm_count();
  static const int cap = [] {
    const char* e = getenv("DRCB_CONV_SMS");
    return e ? atoi(e) : 0;
  }();
  return cap > 0 ? std::min(cap, nsm) : nsm;
}

template <int KIND, int BN, int STAGES>
int launch_bn(const CUtensorMap& mA, const CUtensorMap& mB, const ConvArgs& a, cudaStream_t st) {
  using SM = Smem<KIND, BN, STAGES>;
  auto kern = k_conv_tc<KIND, BN, STAGES>;
  static DeviceFlags attr;
  smem_attr_once(attr, kern, SM::TOTAL);
  const int nsm = conv_sms();
  int tiles = a.num_m_tiles * a.num_n_tiles;
  int grid = tiles < nsm ? tiles : nsm;
  launch_pdl(kern, grid, NUM_THREADS, SM::TOTAL, st, mA, mB, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_conv_tc");
}

template <int KIND, int BN, bool RES, bool DX, int MH = 1, bool PW = false>
int launch_rows_bn(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mO,
                   const CUtensorMap& mP, const ConvArgs& a, const RowArgs& h, size_t smem,
                   cudaStream_t st) {
  auto kern = k_conv_rows<KIND, BN, RES, DX, MH, PW>;
  static DeviceFlags attr;
  smem_attr_once(attr, kern, 227 * 1024);
  const int nsm = conv_sms();
  int tiles = a.num_m_tiles * a.num_n_tiles;
  int grid = tiles < nsm ? tiles : nsm;
  // resident weights with several N tiles: a CTA keeps one N tile's weights,
  // so the grid is a multiple of the N tiles (the schedule's stride then
  // keeps every CTA on its N tile)
  if (RES && a.num_n_tiles > 1) grid = std::min(a.num_m_tiles, nsm / a.num_n_tiles) * a.num_n_tiles;
  launch_pdl(kern, grid, PW ? ROWS_THREADS : RT_THREADS, smem, st, mA, mB, mO, mP, a, h);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_conv_rows");
}

template <int KIND, bool RES>
int launch_pair64(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mO,
                  const ConvArgs& a, const RowArgs& h, size_t smem, cudaStream_t st) {
  auto kern = k_conv_pair<KIND, 64, RES>;
  static DeviceFlags attr;
  smem_attr_once(attr, kern, 227 * 1024);
  const int nsm = conv_sms();
  const int pairs = std::min(a.num_m_tiles, nsm / 2);
  launch_pdl(kern, 2 * pairs, RT_THREADS, smem, st, mA, mB, mO, a, h);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_conv_pair");
}

template <int KIND, bool DX>
int launch_rows(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mO,
                const CUtensorMap& mP, const ConvArgs& a, const RowArgs& h, bool res, size_t smem,
                cudaStream_t st) {
  // the fused-pool skip convs (enc1.conv2: resident dx, BN 64; enc2.conv2:
  // streamed halo, BN 128) with the pool warp
  if (h.o_bytes && h.p_bytes && !h.up2 && !h.pool_cta) {
    if (DX && res && a.bn == 64) return launch_rows_bn<KIND, 64, true, DX, 1, true>(mA, mB, mO, mP, a, h, smem, st);
    if (!DX && !res && a.bn == 128)
      return launch_rows_bn<KIND, 128, false, DX, 1, true>(mA, mB, mO, mP, a, h, smem, st);
    return fail(DRCB_ECONFIG, "fused pool: no pool-warp instantiation for this layer shape");
  }
#define ROWS_CASE(BNV)                                                                  \
  case BNV:                                                                             \
    return res ? launch_rows_bn<KIND, BNV, true, DX>(mA, mB, mO, mP, a, h, smem, st)    \
               : launch_rows_bn<KIND, BNV, false, DX>(mA, mB, mO, mP, a, h, smem, st);
  switch (a.bn) {
    ROWS_CASE(16)
    ROWS_CASE(32)
    ROWS_CASE(64)
    ROWS_CASE(128)
  }
#undef ROWS_CASE
  return fail(DRCB_ECONFIG, "unsupported N tile (row-tile kernel)");
}

// stage counts keep smem <= ~200 KB: BN=256 -> 48 KB/stage
template <int KIND>
int launch_conv(const CUtensorMap& mA, const CUtensorMap& mB, const ConvArgs& a, cudaStream_t st) {
  switch (a.bn) {
    case 16: return launch_bn<KIND, 16, 8>(mA, mB, a, st);
    case 32: return launch_bn<KIND, 32, 8>(mA, mB, a, st);
    case 64: return launch_bn<KIND, 64, 6>(mA, mB, a, st);
    case 128: return launch_bn<KIND, 128, 5>(mA, mB, a, st);
    case 256: return launch_bn<KIND, 256, 4>(mA, mB, a, st);
  }
  return fail(DRCB_ECONFIG, "unsupported N tile");
}

struct Buf {
  void* p;
  int c;   // channels (NHWC)
  int hw;
  int c_real = 0;  // channels holding data when fewer than c (0: all), see encode_act
  int pitch = 0;   // elements between pixels when stored narrower than c (0: c)
};

// one conv layer: in (NHWC, c_in_tot == layer cin_pad) -> out slice
// N tile: the largest of 256 / 128 / 64 / 32 / 16 (<= cap) dividing cout_pad
int n_tile(int cout_pad, int cap) {
  for (int b = cap; b >= 16; b /= 2)
    if (cout_pad % b == 0) return b;
  return 16;
}

// dx-in-N vs halo for a row-tile layer (measured on B200)
bool rows_use_dx(const ConvLayer& L, int kind) {
  (void)kind;
  const bool pooled = L.name.rfind("enc", 0) == 0;  // encoder convs feed a max-pool
  // 16x16: dx (with two-block tiles) wins once the streamed weights dominate
  // (cin >= 128) unless the epilogue also pools (dec2.deconv2: 289 vs 302 us;
  // enc2.conv1: halo 178 vs 196 us; enc2.conv2 + pool: halo 302 vs 318 us)
  return L.hw == 32 || L.cin_pad >= 256 || (L.hw == 16 && L.cin_pad >= 128 && !pooled);
}

// enc1.conv1 through k_conv_in8 (input: 8-channel NHWC, out: BN + LeakyReLU)
template <int KIND>
int run_in8(NetImpl& net, ConvLayer& L, const Buf& in, const Buf& out, int cout_off, int64_t nmaps,
            cudaStream_t st) {
  if (in.c != 8 || L.hw != 32 || L.cout_pad != 64)
    return fail(DRCB_ECONTRACT, "enc1.conv1 expects the 8-channel 32x32 input and 64 outputs");
  ConvArgs a;
  std::memset(&a, 0, sizeof(a));
  a.hw = 32;
  a.maps_per_tile = 1;
  a.rows_per_tile = 4;
  a.tiles_per_map = 8;
  a.num_m_tiles = int(nmaps * 8);
  a.num_n_tiles = 1;
  a.bn = 64;
  a.cout = 64;
  a.cout_tot = out.c;
  a.cout_off = cout_off;
  a.ep_a = L.d_ep_a;
  a.ep_b = L.d_ep_b;
  a.slope = net.slope;
  a.out = out.p;
  auto enc = get_encode();
  if (!enc) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int es = elem_bytes(KIND);
  CUtensorMap mX, mB, mO;
  cuuint64_t dims[4] = {8, 32, 32, cuuint64_t(nmaps)};
  cuuint64_t strides[3] = {cuuint64_t(8 * es), cuuint64_t(8 * es * 32), cuuint64_t(8 * es * 1024)};
  cuuint32_t box[4] = {8, 32, 6, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&mX, tmap_dtype(KIND), 4,
                   in.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DRCB_ECUDA, "cuTensorMapEncodeTiled(in8) failed: " + std::to_string(int(r)));
  int rc = encode_w(&mB, L.d_wtc, KIND, L.cin_pad, 64, 64);
  if (rc) return rc;
  rc = encode_act(&mO, out.p, KIND, out.c, 32, nmaps, 32, 1, 1);  // one row per lane quarter
  if (rc) return rc;
  auto kern = k_conv_in8<KIND>;
  constexpr size_t smem = in8_smem<KIND>();
  static DeviceFlags attr;
  smem_attr_once(attr, kern, int(smem));
  const int nsm = conv_sms();
  int grid = a.num_m_tiles < nsm ? a.num_m_tiles : nsm;
  launch_pdl(kern, grid, IN8_THREADS, smem, st, mX, mB, mO, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_conv_in8");
}

template <int KIND>
int run_layer(NetImpl& net, ConvLayer& L, const Buf& in, const Buf& out, int cout_off,
              int64_t nmaps, cudaStream_t st, float* pred = nullptr, const Buf* up = nullptr,
              const Buf* pool = nullptr) {
  int rc = prepare_layer(net, L, KIND);
  if (rc) return rc;
  if (L.in8) return run_in8<KIND>(net, L, in, out, cout_off, nmaps, st);
  if (in.c != L.cin_pad) return fail(DRCB_ECONTRACT, "tc layer input channels mismatch for " + L.name);
  const int hw = L.hw;
  ConvArgs a;
  std::memset(&a, 0, sizeof(a));
  a.hw = hw;
  if (hw * hw >= BM) {
    a.maps_per_tile = 1;
    a.rows_per_tile = BM / hw;
    a.tiles_per_map = hw * hw / BM;
  } else {
    a.maps_per_tile = BM / (hw * hw);
    a.rows_per_tile = hw;
    a.tiles_per_map = 1;
  }
  a.num_m_tiles = int(nmaps * hw * hw / BM);
  a.cblocks = L.cin_pad / (ROW_BYTES / elem_bytes(KIND));
  a.num_kb = 9 * a.cblocks;
  a.bn = n_tile(L.cout_pad, 256);
  a.num_n_tiles = L.cout_pad / a.bn;
  a.cout = pred ? L.cout_pad : L.cout_pad;  // padded channels carry exact zeros
  a.cout_tot = out.c;
  a.cout_off = cout_off;
  a.ep_a = L.d_ep_a;
  a.ep_b = L.d_ep_b;
  a.slope = net.slope;
  a.out = out.p;
  if (pred) {
    const ConvLayer& H = net.layers[16];
    a.head = 1;
    a.pred = pred;
    for (int o = 0; o < 3; ++o) {
      for (int j = 0; j < 16; ++j) a.hw_w[o * 16 + j] = j < H.cin ? H.w[o * H.cin + j] : 0.f;
      a.hw_b[o] = H.bias[o];
    }
  }
  CUtensorMap mA, mB;
  if (hw >= 16 && !getenv("DRCB_NO_ROWS")) {
    // row-tile kernel (hw 16/32); DRCB_ROWS=dx|halo overrides the variant
    static const char* mode_env = getenv("DRCB_ROWS");
    const bool dx = mode_env ? std::strcmp(mode_env, "dx") == 0 : rows_use_dx(L, KIND);
    a.bn = n_tile(L.cout_pad, KIND != 1 ? 128 : 64);
    a.num_n_tiles = L.cout_pad / a.bn;
    RowArgs rz;
    rz.up2 = 0;
    rz.pool_cta = 0;
    rz.row_bytes = hw * ROW_BYTES;
    rz.a_bytes = (a.rows_per_tile + 2) * hw * ROW_BYTES;
    int b_tile = a.bn * ROW_BYTES;
    int w_bytes = 9 * a.cblocks * b_tile;
    rz.o_bytes = pred ? 0 : BM * std::max(a.bn, ROW_BYTES / elem_bytes(KIND)) * elem_bytes(KIND);
    rz.p_bytes = (pool && rz.o_bytes) ? rz.o_bytes / 4 : 0;
    const int budget = 216 * 1024 - 2 * rz.o_bytes - 2 * rz.p_bytes;  // of 227 KB
    // resident weights: one N tile's weights per CTA (several N tiles: the
    // dgrad of dec1.deconv1, 64 -> 192 channels; 1,101 -> ~830 us per 4,096
    // samples against the streamed two-block kernel)
    const bool no_res_multi = getenv("DRCB_NO_RES_MULTI") != nullptr;
    bool res = (a.num_n_tiles == 1 || (!no_res_multi && a.num_n_tiles <= sm_count())) &&
               w_bytes + 3 * rz.a_bytes <= budget;
    int budget_res = budget;
    // weights that do not fit at 3 A stages: 64-wide N tiles with at least
    // DRCB_RES_STAGES A stages (default 2) may (the 16x16 convs with 128
    // input channels: 144 KB per N tile; dec2.deconv1's dgrad, 128 -> 384
    // channels, 880 -> 695 us; the 128 -> 128 ones 293 -> 234 us, B = 4,096)
    if (!res && !no_res_multi && KIND != 1 && dx && a.bn >= 64 && !pool && !pred && !up) {
      const char* e = getenv("DRCB_RES_STAGES");
      const int min_st = e ? std::max(1, atoi(e)) : 2;
      const int o64 = BM * 64 * elem_bytes(KIND), w64 = 9 * a.cblocks * 64 * ROW_BYTES;
      const int bud64 = 216 * 1024 - 2 * o64;
      if (w64 + min_st * rz.a_bytes <= bud64) {
        a.bn = 64;
        a.num_n_tiles = L.cout_pad / 64;
        b_tile = 64 * ROW_BYTES;
        rz.o_bytes = o64;
        budget_res = bud64;
        w_bytes = w64;
        res = true;
      }
    }
    if (res) {
      rz.sb = 1;
      rz.sa = std::min(8, (budget_res - w_bytes) / rz.a_bytes);
    } else if (dx) {
      // B triples are consumed three per A box
      rz.sa = std::min(4, std::max(2, budget / (4 * rz.a_bytes)));
      rz.sb = std::min(8, (budget - rz.sa * rz.a_bytes) / (3 * b_tile));
    } else {
      rz.sa = rz.sb = std::min(8, budget / (rz.a_bytes + 3 * b_tile));
    }
    // streamed-weight dx layers (dec1.deconv1, dec2.deconv1): two M blocks per
    // work tile share each weight stage (half the L2 weight traffic per
    // pixel; at 16x16 the tile is the whole map)
    const bool two = dx && !res && KIND != 1 && a.bn <= 128 && L.cout_pad % 64 == 0 &&
                     rz.o_bytes && !rz.p_bytes && getenv("DRCB_NO_MH2") == nullptr;
    if (two) {
      a.bn = 64;  // two M blocks x 3 dx accumulators of 64 columns = 384 TMEM columns
      a.num_n_tiles = L.cout_pad / 64;
      b_tile = 64 * ROW_BYTES;
      rz.o_bytes = BM * 64 * 2;
      a.rows_per_tile = 2 * BM / hw;
      a.tiles_per_map = hw * hw / (2 * BM);
      a.num_m_tiles = int(nmaps * a.tiles_per_map);
      rz.a_bytes = (a.rows_per_tile + 2) * hw * ROW_BYTES;
      rz.o_bytes *= 2;
      const int bud2 = 216 * 1024 - 2 * rz.o_bytes;
      rz.sa = 2;
      rz.sb = std::min(8, (bud2 - rz.sa * rz.a_bytes) / (3 * b_tile));
    }
    // streamed-weight dx layers without a fused upsample: CTA-pair kernel
    // (M = 256 across two SMs, double-buffered TMEM)
    if (KIND != 1 && dx && !res && L.cout_pad == 64 && rz.o_bytes && !rz.p_bytes && !up &&
        getenv("DRCB_NO_PAIR") == nullptr) {
      RowArgs pz = rz;
      ConvArgs pa = a;
      pa.bn = 64;
      pa.num_n_tiles = 1;
      pa.rows_per_tile = 2 * BM / hw;           // per pair tile
      pa.tiles_per_map = hw * hw / (2 * BM);
      pa.num_m_tiles = int(nmaps * pa.tiles_per_map);
      pz.a_bytes = (BM / hw + 2) * hw * ROW_BYTES;
      pz.o_bytes = BM * 64 * 2;
      pz.p_bytes = 0;
      pz.up2 = 0;
      const int bhalf = 96 * ROW_BYTES;
      // this CTA's half of the weights resident when it fits next to three
      // A stages (dec1.deconv1: 3 x 3 x 12 KB)
      const int wbytes = a.cblocks * 3 * bhalf;
      const bool pres = wbytes + 3 * pz.a_bytes + 2 * pz.o_bytes <= 216 * 1024 &&
                        getenv("DRCB_PAIR_STREAM") == nullptr;
      if (pres) {
        pz.sb = 1;
        pz.sa = std::min(8, (216 * 1024 - 2 * pz.o_bytes - wbytes) / pz.a_bytes);
      } else {
        pz.sa = 4;
        pz.sb = std::min(8, (216 * 1024 - 2 * pz.o_bytes - pz.sa * pz.a_bytes) / bhalf);
      }
      CUtensorMap pA, pB, pO;
      rc = encode_act(&pA, in.p, KIND, in.c, hw, nmaps, hw, BM / hw + 2, 1, in.c_real, in.pitch);
      if (rc) return rc;
      rc = encode_w(&pB, L.d_wtc, KIND, int64_t(9) * L.cin_pad, L.cout_pad, 32);
      if (rc) return rc;
      rc = encode_act(&pO, out.p, KIND, out.c, hw, nmaps, hw, 32 / hw, 1);  // per-quarter boxes
      if (rc) return rc;
      const size_t smem = 1024 + (pres ? size_t(wbytes) : size_t(pz.sb) * bhalf) + size_t(pz.sa) * pz.a_bytes +
                          2 * size_t(pz.o_bytes) + 512 + 8 * EP_MAX;
      constexpr int KP = KIND == 1 ? 0 : KIND;  // never reached for tf32 (16-bit operands only)
      return pres ? launch_pair64<KP, true>(pA, pB, pO, pa, pz, smem, st)
                  : launch_pair64<KP, false>(pA, pB, pO, pa, pz, smem, st);
    }
    // resident-weight 32x32 dx layers: two M blocks (8 rows) per work tile
    // halve the per-tile fixed costs and the halo re-reads (10 rows loaded
    // per 8 computed instead of 6 per 4)
    // (head.deconv1 / head.deconv2; at BN = 64 the 40 KB A stages leave too
    // few of them and the layer slows down)
    bool two_res = !two && dx && res && KIND != 1 && a.bn <= 32 && hw == 32 && !rz.p_bytes &&
                   !up && getenv("DRCB_NO_MH2") == nullptr;
    if (two_res) {
      const int a2 = (2 * BM / hw + 2) * hw * ROW_BYTES;
      const int bud2 = 216 * 1024 - 4 * rz.o_bytes;
      const int sa2 = std::min(8, (bud2 - w_bytes) / a2);
      if (sa2 >= 2) {
        a.rows_per_tile = 2 * BM / hw;
        a.tiles_per_map = hw * hw / (2 * BM);
        a.num_m_tiles = int(nmaps * a.tiles_per_map);
        rz.a_bytes = a2;
        rz.o_bytes *= 2;
        rz.sa = sa2;
      } else {
        two_res = false;
      }
    }
    // 16x16 two-block tiles hold whole maps: the epilogue can write the 2x
    // upsample of the output into the next level's concat buffer itself
    const bool up_after = up && !(two && hw == 16);  // no whole-map tile: separate pass
    if (up && !up_after) {
      rz.up2 = 1;
      rz.sb = 2;  // room for the low-res tile + two output chunk buffers
    }
    // fused pools run on the kernel's pool warp (per-quarter output stores);
    // DRCB_POOL_CTA: the CTA-wide staged-tile pool of the epilogue warps
    const bool pool_cta = getenv("DRCB_POOL_CTA") != nullptr;
    // pool-warp instantiations: enc1.conv2 (resident dx, BN 64) and enc2.conv2
    // (streamed halo, BN 128); other shapes keep the CTA-wide pool
    const bool pw_shape = (dx && res && a.bn == 64) || (!dx && !res && a.bn == 128);
    rz.pool_cta = (pool_cta || !pw_shape) ? 1 : 0;
    if (rz.sa >= 2 && (res || rz.sb >= 2)) {
      rc = encode_act(&mA, in.p, KIND, in.c, hw, nmaps, hw, a.rows_per_tile + 2, 1, in.c_real, in.pitch);
      if (rc) return rc;
      rc = encode_w(&mB, L.d_wtc, KIND, int64_t(9) * L.cin_pad, L.cout_pad, a.bn);
      if (rc) return rc;
      CUtensorMap mO, mP;
      if (rz.up2) {
        rc = encode_act(&mO, up->p, KIND, up->c, 2 * hw, nmaps, 2 * hw, 8, 1);
        if (rc) return rc;
      } else if (rz.o_bytes) {
        // whole-tile boxes with the fused pool, else per-lane-quarter (32 px)
        rc = encode_act(&mO, out.p, KIND, out.c, hw, nmaps, hw, (rz.p_bytes && rz.pool_cta) ? a.rows_per_tile : 32 / hw, 1);
        if (rc) return rc;
      }
      if (rz.p_bytes) {
        rc = encode_act(&mP, pool->p, KIND, pool->c, hw / 2, nmaps, hw / 2, a.rows_per_tile / 2, 1);
        if (rc) return rc;
      } else {
        mP = mO;
      }
      size_t smem = 1024 + size_t(res ? w_bytes : 0) + size_t(rz.sa) * rz.a_bytes +
                    size_t(res ? 0 : rz.sb * 3 * b_tile) + (rz.up2 ? 3 : 2) * size_t(rz.o_bytes) +
                    2 * size_t(rz.p_bytes) + 512 + 8 * EP_MAX;
      if constexpr (KIND != 1) {
        if (two) rc = launch_rows_bn<KIND, 64, false, true, 2>(mA, mB, mO, mP, a, rz, smem, st);
        if (two_res) {
          switch (a.bn) {
            case 16: rc = launch_rows_bn<KIND, 16, true, true, 2>(mA, mB, mO, mP, a, rz, smem, st); break;
            default: rc = launch_rows_bn<KIND, 32, true, true, 2>(mA, mB, mO, mP, a, rz, smem, st); break;
          }
        }
      }
      if ((!two && !two_res) || KIND == 1)
        rc = dx ? launch_rows<KIND, true>(mA, mB, mO, mP, a, rz, res, smem, st)
                : launch_rows<KIND, false>(mA, mB, mO, mP, a, rz, res, smem, st);
      if (rc || !up_after) return rc;
      using T = ElemT<KIND>;
      return up_dispatch<T>(static_cast<const T*>(out.p), L.cout_pad, hw, static_cast<T*>(up->p),
                            up->c, nmaps, st);
    }
    a.bn = n_tile(L.cout_pad, 256);
    a.num_n_tiles = L.cout_pad / a.bn;
  }
  // few M tiles (small batches of the 4x4 / 8x8 layers): narrower N tiles
  // until the work tiles cover the SMs; each output's K order is unchanged
  // (same bits), the A tiles are re-read per N tile from L2
  static const bool no_nsplit = getenv("DRCB_NO_NSPLIT") != nullptr;
  if (!pred && !no_nsplit) {
    while (a.bn > 64 && int64_t(a.num_m_tiles) * (L.cout_pad / a.bn) < sm_count()) a.bn /= 2;
    a.num_n_tiles = L.cout_pad / a.bn;
  }
  int box_w = hw, box_h = a.maps_per_tile == 1 ? a.rows_per_tile : hw, box_n = a.maps_per_tile;
  rc = encode_act(&mA, in.p, KIND, in.c, hw, nmaps, box_w, box_h, box_n, in.c_real, in.pitch);
  if (rc) return rc;
  rc = encode_w(&mB, L.d_wtc, KIND, int64_t(9) * L.cin_pad, L.cout_pad, a.bn);
  if (rc) return rc;
  rc = launch_conv<KIND>(mA, mB, a, st);
  if (rc || !pool) return rc;
  // this path has no fused pool: run the separate pass
  using T = ElemT<KIND>;
  return pool_dispatch<T>(static_cast<const T*>(out.p), out.c, cout_off, L.cout_pad, hw / 2,
                          static_cast<T*>(pool->p), nmaps, st);
}

// head.deconv1 + head.deconv2 + conv_out in one kernel (16-bit; see k_head_fused)
template <int KIND>
int run_head_fused(NetImpl& net, ConvLayer& L1, ConvLayer& L2, const Buf& in, int64_t nmaps,
                   float* pred, cudaStream_t st) {
  int rc = prepare_layer(net, L1, KIND);
  if (rc) return rc;
  rc = prepare_layer(net, L2, KIND);
  if (rc) return rc;
  if (in.c != 64 || in.hw != 32 || L1.cin_pad != 64 || L1.cout_pad != 32 || L2.cin_pad != 64 ||
      L2.cout_pad != 16)
    return fail(DRCB_ECONTRACT, "fused head expects 64 -> 32 -> 16 channels at 32x32");
  ConvArgs p1, p2;
  std::memset(&p1, 0, sizeof(p1));
  std::memset(&p2, 0, sizeof(p2));
  p1.hw = p2.hw = 32;
  p1.ep_a = L1.d_ep_a;
  p1.ep_b = L1.d_ep_b;
  p1.slope = p2.slope = net.slope;
  p1.cout = 32;
  p2.ep_a = L2.d_ep_a;
  p2.ep_b = L2.d_ep_b;
  p2.cout = 16;
  p2.head = 1;
  p2.pred = pred;
  const ConvLayer& H = net.layers[16];
  for (int o = 0; o < 3; ++o) {
    for (int j = 0; j < 16; ++j) p2.hw_w[o * 16 + j] = j < H.cin ? H.w[o * H.cin + j] : 0.f;
    p2.hw_b[o] = H.bias[o];
  }
  CUtensorMap mA10, mA6, mW1, mW2;
  rc = encode_act(&mA10, in.p, KIND, in.c, 32, nmaps, 32, 10, 1);
  if (rc) return rc;
  rc = encode_act(&mA6, in.p, KIND, in.c, 32, nmaps, 32, 6, 1);
  if (rc) return rc;
  rc = encode_w(&mW1, L1.d_wtc, KIND, int64_t(9) * L1.cin_pad, L1.cout_pad, 32);
  if (rc) return rc;
  rc = encode_w(&mW2, L2.d_wtc, KIND, int64_t(9) * L2.cin_pad, L2.cout_pad, 16);
  if (rc) return rc;
  constexpr size_t smem = head_fused_smem();
  static DeviceFlags attr;
  smem_attr_once(attr, k_head_fused<KIND>, int(smem));
  const int nsm = conv_sms();
  const int grid = nmaps < nsm ? int(nmaps) : nsm;  // whole maps per CTA
  launch_pdl(k_head_fused<KIND>, grid, RT_THREADS, smem, st, mA10, mA6, mW1, mW2, p1, p2, int(nmaps));
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_head_fused");
}

template <int KIND>
int forward_kind(NetImpl& net, const float* x, float* y, int64_t n, cudaStream_t st,
                 const void* x_nhwc = nullptr) {
  using T = ElemT<KIND>;
  const int k = net.k;
  if (k != 64)  // buffer plan: concat/skip slices are whole 64-channel rows only at k = 64
    return fail(DRCB_ECONFIG, "tensor-core path supports k = 64 (use net_mode fp32 for other k)");
  auto& Ls = net.layers;
  const int64_t np = ((n + 7) / 8) * 8;  // 4x4 tiles hold 8 maps
  auto P = [&](int c) { return pad_c(c, KIND); };
  // buffer plan (elements per map): channels padded to the K granularity
  struct Spec { int c, hw; };
  const Spec specs[] = {
      {8, 32},          // 0 x0: compact input, 7 channels + 1 zero
      {P(k), 32},       // 1 e32
      {3 * k, 32},      // 2 c1 [up(2k) | s1(k)]
      {P(k), 16},       // 3 p1
      {2 * k, 16},      // 4 e16
      {6 * k, 16},      // 5 c2
      {2 * k, 8},       // 6 p2
      {4 * k, 8},       // 7 e8
      {12 * k, 8},      // 8 c3
      {4 * k, 4},       // 9 p3
      {8 * k, 4},       // 10 b0
      {8 * k, 4},       // 11 b1
      {4 * k, 8},       // 12 d8
      {2 * k, 16},      // 13 d16
      {P(k), 32},       // 14 d32
      {P(k / 2), 32},   // 15 h1
  };
  constexpr int NBUF = 16;
  size_t off[NBUF + 1];
  off[0] = 0;
  for (int i = 0; i < NBUF; ++i) {
    size_t bytes = size_t(np) * specs[i].hw * specs[i].hw * specs[i].c * sizeof(T);
    off[i + 1] = off[i] + ((bytes + 1023) & ~size_t(1023));
  }
  uint8_t* base = nullptr;
  DRCB_CUDA(cudaMallocAsync((void**)&base, off[NBUF], st));
  Buf B[NBUF];
  for (int i = 0; i < NBUF; ++i) B[i] = Buf{base + off[i], specs[i].c, specs[i].hw};
  int rc = 0;
  // input stack -> NHWC padded (skipped when the caller already wrote it)
  if (x_nhwc) {
    B[0].p = const_cast<void*>(x_nhwc);
  } else {
    int64_t tot = np * 1024 * (8 / Vec<T>::N);
    launch_pdl(k_stack_to_nhwc<T>, unsigned((tot + 255) / 256), 256, 0, st, x, n, np, B[0].c, (T*)B[0].p);
    count_launch();
  }
  auto pool = [&](const Buf& in, int off_c, int c, const Buf& out) {
    rc |= pool_dispatch<T>((const T*)in.p, in.c, off_c, c, out.hw, (T*)out.p, np, st);
  };
  auto up = [&](const Buf& in, int c, const Buf& out) {
    rc |= up_dispatch<T>((const T*)in.p, c, in.hw, (T*)out.p, out.c, np, st);
  };
  // encoder
  rc |= run_layer<KIND>(net, Ls[0], B[0], B[1], 0, np, st);
  // the 32x32 / 16x16 skip convs also write their 2x2 max-pool (fused)
  const bool fpool = getenv("DRCB_NO_FUSED_POOL") == nullptr;
  rc |= run_layer<KIND>(net, Ls[1], B[1], B[2], 2 * k, np, st, nullptr, nullptr,
                        fpool ? &B[3] : nullptr);                   // s1 -> c1[2k:3k]
  if (!fpool) pool(B[2], 2 * k, k, B[3]);
  rc |= run_layer<KIND>(net, Ls[2], B[3], B[4], 0, np, st);
  rc |= run_layer<KIND>(net, Ls[3], B[4], B[5], 4 * k, np, st, nullptr, nullptr,
                        fpool ? &B[6] : nullptr);                   // s2 -> c2[4k:6k]
  if (!fpool) pool(B[5], 4 * k, 2 * k, B[6]);
  rc |= run_layer<KIND>(net, Ls[4], B[6], B[7], 0, np, st);
  rc |= run_layer<KIND>(net, Ls[5], B[7], B[8], 8 * k, np, st);   // s3 -> c3[8k:12k]
  pool(B[8], 8 * k, 4 * k, B[9]);
  rc |= run_layer<KIND>(net, Ls[6], B[9], B[10], 0, np, st);
  rc |= run_layer<KIND>(net, Ls[7], B[10], B[11], 0, np, st);
  up(B[11], 8 * k, B[8]);
  // decoder
  rc |= run_layer<KIND>(net, Ls[8], B[8], B[7], 0, np, st);
  rc |= run_layer<KIND>(net, Ls[9], B[7], B[12], 0, np, st);
  up(B[12], 4 * k, B[5]);
  rc |= run_layer<KIND>(net, Ls[10], B[5], B[4], 0, np, st);
  // dec2.deconv2's whole-map tiles write up2x straight into c1 (k_conv_rows up2)
  const bool fup16 = KIND != 1 && getenv("DRCB_NO_UP16") == nullptr;
  rc |= run_layer<KIND>(net, Ls[11], B[4], B[13], 0, np, st, nullptr, fup16 ? &B[2] : nullptr);
  if (!fup16) up(B[13], 2 * k, B[2]);
  rc |= run_layer<KIND>(net, Ls[12], B[2], B[1], 0, np, st);
  rc |= run_layer<KIND>(net, Ls[13], B[1], B[14], 0, np, st);
  if (rc) {
    cudaFreeAsync(base, st);
    return rc;
  }
  // predictions for the n real maps
  float* pred = y;
  float* tmp = nullptr;
  if (np != n) {
    DRCB_CUDA(cudaMallocAsync((void**)&tmp, size_t(np) * 3 * 1024 * 4, st));
    pred = tmp;
  }
  if (KIND != 1 && getenv("DRCB_NO_HEAD_FUSE") == nullptr) {
    // head.deconv1 + head.deconv2 + conv_out + ReLU in one kernel
    rc = run_head_fused<KIND>(net, Ls[14], Ls[15], B[14], np, pred, st);
  } else {
    rc = run_layer<KIND>(net, Ls[14], B[14], B[15], 0, np, st);
    // head.deconv2 + conv_out + ReLU fused
    if (!rc) rc = run_layer<KIND>(net, Ls[15], B[15], B[14], 0, np, st, pred);
  }
  if (tmp) {
    DRCB_CUDA(cudaMemcpyAsync(y, tmp, size_t(n) * 3 * 1024 * 4, cudaMemcpyDeviceToDevice, st));
    DRCB_CUDA(cudaFreeAsync(tmp, st));
  }
  DRCB_CUDA(cudaFreeAsync(base, st));
  return rc;
}

}  // namespace tc

// input already NHWC (n rounded up to 8 maps, channels padded to the K
// granularity, zeros in the padding): used by the frame driver
// Maps per forward pass: the layer chain runs over chunks of this many maps
// (a multiple of 8; bounds the activation footprint, ~1.5 MB per map in
// 16-bit). Measured inside the bench frame (config 3, 4,096 maps, fp16): one
// pass 5.15-5.17 ms, two chunks of 2,048 5.23 ms, four of 1,024 5.47 ms
// (standalone, tools/net_time.py, two chunks looked 6 % faster: it does not
// carry over to the frame). DRCB_NET_CHUNK overrides (A/B).
int64_t net_chunk() {
  static const int64_t c = [] {
    const char* e = getenv("DRCB_NET_CHUNK");
    const int64_t v = e ? atoll(e) : 8192;
    return std::max<int64_t>(8, v / 8 * 8);
  }();
  return c;
}

int forward_tc_nhwc(NetImpl& net, const void* x_nhwc, float* y, int64_t n, int mode,
                    cudaStream_t st) {
  keep_pool_memory();
  const int64_t chunk = net_chunk();
  const size_t es = mode == DRCB_NET_TF32 ? 4 : 2;  // compact input: 8 channels per pixel
  for (int64_t d = 0; d < n; d += chunk) {
    const int64_t c = n - d < chunk ? n - d : chunk;
    const void* xs = static_cast<const uint8_t*>(x_nhwc) + size_t(d) * 1024 * 8 * es;
    float* ys = y + d * 3 * 1024;
    int rc = mode == DRCB_NET_BF16   ? tc::forward_kind<0>(net, nullptr, ys, c, st, xs)
             : mode == DRCB_NET_FP16 ? tc::forward_kind<2>(net, nullptr, ys, c, st, xs)
             : mode == DRCB_NET_TF32 ? tc::forward_kind<1>(net, nullptr, ys, c, st, xs)
                                     : fail(DRCB_ECONFIG, "unknown tensor-core net mode");
    if (rc) return rc;
  }
  return 0;
}

int tc_input_channels(int) { return 8; }  // compact NHWC input (7 + 1 zero channel)

// One tensor-core conv on caller buffers (the training engine's forward and
// dgrad): NHWC bf16 in (nmaps a multiple of 8, cin_pad channels), packed
// K-major weights [cout_pad][9 * cin_pad], epilogue y = acc * a + b then
// LeakyReLU(slope) (slope 1 = identity) into out's channel slice.
// in_pitch (0 = cin_pad): elements between input pixels when the input is
// stored narrower than its 64-channel K blocks; out_ctot below 64 likewise
// stores the output narrow (the TMA store drops the box's other channels)
int tc_conv_bf16(int cin, int cout, int hw, int64_t nmaps, const void* in, int cin_pad, void* out,
                 int out_ctot, int out_coff, const void* wpacked, int cout_pad, const float* ep_a,
                 const float* ep_b, float slope, cudaStream_t st, int in_pitch) {
  NetImpl net;
  net.slope = slope;
  ConvLayer L;
  L.name = "train";
  L.cin = cin;
  L.cout = cout;
  L.hw = hw;
  L.cin_pad = cin_pad;
  L.cout_pad = cout_pad;
  L.d_wtc = const_cast<void*>(wpacked);
  L.d_ep_a = const_cast<float*>(ep_a);
  L.d_ep_b = const_cast<float*>(ep_b);
  L.tc_kind = 0;
  // channels past cin (rounded to 8) hold zeros (or a shared buffer's stale
  // values) that meet zero weights: not read (TMA zero fill)
  const int c_real = cin < cin_pad ? (cin + 7) / 8 * 8 : 0;
  tc::Buf bi{const_cast<void*>(in), cin_pad, hw, c_real, in_pitch}, bo{out, out_ctot, hw};
  return tc::run_layer<0>(net, L, bi, bo, out_coff, nmaps, st);
}

// enc1.conv1 of the training engine through the inference in8 kernel: the
// 8-channel NHWC input (x0), weights packed [64][128] with K index tap * 8 +
// channel (zeros beyond 72), epilogue y = acc * a + b then LeakyReLU(slope)
int tc_conv_in8_bf16(int64_t nmaps, const void* in, void* out, int out_ctot, const void* w8,
                     const float* ep_a, const float* ep_b, float slope, cudaStream_t st) {
  NetImpl net;
  net.slope = slope;
  ConvLayer L;
  L.name = "enc1.conv1";
  L.cin = 8;
  L.cout = 64;
  L.hw = 32;
  L.in8 = true;
  L.cin_pad = 128;
  L.cout_pad = 64;
  L.tc_kind = 0;
  L.d_wtc = const_cast<void*>(w8);
  L.d_ep_a = const_cast<float*>(ep_a);
  L.d_ep_b = const_cast<float*>(ep_b);
  tc::Buf bi{const_cast<void*>(in), 8, 32}, bo{out, out_ctot, 32};
  return tc::run_in8<0>(net, L, bi, bo, 0, nmaps, st);
}

int forward_tc(NetImpl& net, const float* x, float* y, int64_t n, int mode, cudaStream_t st) {
  if (n <= 0) return 0;
  keep_pool_memory();
  // (also bounds the activation footprint, ~1.5 MB/map in bf16)
  const int64_t chunk = net_chunk();
  for (int64_t d = 0; d < n; d += chunk) {
    int64_t c = n - d < chunk ? n - d : chunk;
    const float* xs = x + d * 7 * 1024;
    float* ys = y + d * 3 * 1024;
    int rc = mode == DRCB_NET_BF16   ? tc::forward_kind<0>(net, xs, ys, c, st)
             : mode == DRCB_NET_FP16 ? tc::forward_kind<2>(net, xs, ys, c, st)
             : mode == DRCB_NET_TF32 ? tc::forward_kind<1>(net, xs, ys, c, st)
                                     : fail(DRCB_ECONFIG, "unknown tensor-core net mode");
    if (rc) return rc;
  }
  return 0;
}

}  // namespace drcb

// ---------------------------------------------------------------------------
// single-layer harness (tests only): identity epilogue (a=1, b=0, slope 1),
// host arrays. x: (n,hw,hw,cin) fp32 NHWC, w: (cout,cin,3,3), y: (n,hw,hw,cout)
extern "C" int drcb_debug_conv(int32_t mode, int32_t cin, int32_t cout, int32_t hw, int64_t n,
                               const float* x, const float* w, float* y) {
  using namespace drcb;
  using namespace drcb::tc;
  const int kind = mode == DRCB_NET_BF16 ? 0 : (mode == DRCB_NET_FP16 ? 2 : 1);
  NetImpl net;
  net.k = 64;
  net.slope = 1.0f;
  ConvLayer L;
  L.name = "debug";
  L.cin = cin;
  L.cout = cout;
  L.hw = hw;
  L.w.assign(w, w + size_t(cout) * cin * 9);
  L.bias.assign(cout, 0.f);
  L.scale.assign(cout, 1.f);
  L.shift.assign(cout, 0.f);
  int rc = prepare_layer(net, L, kind);
  if (rc) return rc;
  const int es = elem_bytes(kind);
  const int cinp = L.cin_pad, coutp = L.cout_pad;
  const int64_t np = ((n + 7) / 8) * 8;
  const size_t px = size_t(np) * hw * hw;
  std::vector<uint8_t> hx(px * cinp * es, 0);
  for (int64_t i = 0; i < n * hw * hw; ++i)
    for (int c = 0; c < cin; ++c) {
      float v = x[i * cin + c];
      if (kind == 0) {
        __nv_bfloat16 b = __float2bfloat16(v);
        std::memcpy(&hx[(i * cinp + c) * 2], &b, 2);
      } else if (kind == 2) {
        __half b = __float2half_rn(v);
        std::memcpy(&hx[(i * cinp + c) * 2], &b, 2);
      } else {
        std::memcpy(&hx[(i * cinp + c) * 4], &v, 4);
      }
    }
  void *dx = nullptr, *dy = nullptr;
  DRCB_CUDA(cudaMalloc(&dx, hx.size()));
  DRCB_CUDA(cudaMalloc(&dy, px * coutp * es));
  cudaMemcpy(dx, hx.data(), hx.size(), cudaMemcpyHostToDevice);
  Buf in{dx, cinp, hw}, out{dy, coutp, hw};
  rc = kind == 0 ? run_layer<0>(net, L, in, out, 0, np, 0)
       : kind == 2 ? run_layer<2>(net, L, in, out, 0, np, 0)
                   : run_layer<1>(net, L, in, out, 0, np, 0);
  if (!rc) {
    std::vector<uint8_t> hy(px * coutp * es);
    cudaMemcpy(hy.data(), dy, hy.size(), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = cuda_fail(e, "drcb_debug_conv");
    for (int64_t i = 0; i < n * hw * hw; ++i)
      for (int c = 0; c < cout; ++c) {
        if (kind == 0) {
          __nv_bfloat16 b;
          std::memcpy(&b, &hy[(i * coutp + c) * 2], 2);
          y[i * cout + c] = __bfloat162float(b);
        } else if (kind == 2) {
          __half b;
          std::memcpy(&b, &hy[(i * coutp + c) * 2], 2);
          y[i * cout + c] = __half2float(b);
        } else {
          std::memcpy(&y[i * cout + c], &hy[(i * coutp + c) * 4], 4);
        }
      }
  }
  cudaFree(dx);
  cudaFree(dy);
  for (void* p : net.allocs) cudaFree(p);
  return rc;
}
