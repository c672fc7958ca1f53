// drcb_cnn.cu — DRCW weights container, network handle and the fp32 SIMT
// forward pass (the exact-parity engine for drc.cnn.forward, cnn.py:193-215).
// The tensor-core engines live in drcb_conv_tc.cu.
#include <cmath>
#include <cstring>

#include "drcb_net.h"

namespace drcb {

std::map<std::string, std::vector<uint32_t>> architecture(int k) {
  // cnn.py:39-78
  std::map<std::string, std::vector<uint32_t>> t;
  auto conv = [&](const std::string& n, uint32_t ci, uint32_t co, uint32_t ks) {
    t[n + ".weight"] = {co, ci, ks, ks};
    t[n + ".bias"] = {co};
  };
  auto deconv = [&](const std::string& n, uint32_t ci, uint32_t co) {
    t[n + ".weight"] = {ci, co, 3, 3};
    t[n + ".bias"] = {co};
  };
  auto bn = [&](const std::string& n, uint32_t c) {
    for (const char* s : {"gamma", "beta", "running_mean", "running_var"}) t[n + "." + s] = {c};
  };
  uint32_t K = uint32_t(k);
  uint32_t w[3][2] = {{7, K}, {K, 2 * K}, {2 * K, 4 * K}};
  for (int i = 0; i < 3; ++i) {
    std::string p = "enc" + std::to_string(i + 1);
    conv(p + ".conv1", w[i][0], w[i][1], 3);
    bn(p + ".bn1", w[i][1]);
    conv(p + ".conv2", w[i][1], w[i][1], 3);
    bn(p + ".bn2", w[i][1]);
  }
  conv("bott.conv1", 4 * K, 8 * K, 3);
  bn("bott.bn1", 8 * K);
  conv("bott.conv2", 8 * K, 8 * K, 3);
  bn("bott.bn2", 8 * K);
  uint32_t dec[3][3] = {{3, 8 * K, 4 * K}, {2, 4 * K, 2 * K}, {1, 2 * K, K}};
  for (auto& d : dec) {
    std::string p = "dec" + std::to_string(d[0]);
    deconv(p + ".deconv1", d[1] + d[2], d[2]);
    bn(p + ".bn1", d[2]);
    deconv(p + ".deconv2", d[2], d[2]);
    bn(p + ".bn2", d[2]);
  }
  deconv("head.deconv1", K, K / 2);
  bn("head.bn1", K / 2);
  deconv("head.deconv2", K / 2, K / 4);
  bn("head.bn2", K / 4);
  conv("head.conv_out", K / 4, 3, 1);
  return t;
}

namespace {

struct Reader {
  const uint8_t* p;
  size_t len, off = 0;
  bool take(void* dst, size_t n) {
    if (off + n > len) return false;
    std::memcpy(dst, p + off, n);
    off += n;
    return true;
  }
};

int format_error(const std::string& msg, size_t offset) {
  return fail(DRCB_EFORMAT, msg + " (byte offset " + std::to_string(offset) + ")");
}

template <typename T>
T* dev_copy(NetImpl& net, const std::vector<T>& v) {
  void* p = nullptr;
  if (cudaMalloc(&p, v.size() * sizeof(T)) != cudaSuccess) return nullptr;
  net.allocs.push_back(p);
  cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return static_cast<T*>(p);
}

}  // namespace

// ---------------------------------------------------------------------------
// fp32 SIMT kernels (NCHW). Each thread owns one output pixel and 8 output
// channels; weights are read warp-uniformly.
namespace {

constexpr int CO_PER_THREAD = 8;

template <int KS>
__global__ void __launch_bounds__(256) k_conv_f32(const float* __restrict__ in, int cin_tot,
                                                  int cin_off, int cin, const float* __restrict__ w,
                                                  const float* __restrict__ bias,
                                                  const float* __restrict__ scale,
                                                  const float* __restrict__ shift, int act,
                                                  float slope, float* __restrict__ out,
                                                  int cout_tot, int cout_off, int cout, int hw) {
  int n = blockIdx.z;
  int co0 = blockIdx.y * CO_PER_THREAD;
  int pix = blockIdx.x * blockDim.x + threadIdx.x;
  int npx = hw * hw;
  if (pix >= npx) return;
  int y = pix / hw, x = pix % hw;
  const float* ib = in + (size_t(n) * cin_tot + cin_off) * npx;
  float acc[CO_PER_THREAD];
#pragma unroll
  for (int j = 0; j < CO_PER_THREAD; ++j) acc[j] = 0.f;
  const int R = KS / 2;
  for (int ci = 0; ci < cin; ++ci) {
    const float* ip = ib + size_t(ci) * npx;
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      int yy = y + ky - R;
#pragma unroll
      for (int kx = 0; kx < KS; ++kx) {
        int xx = x + kx - R;
        float v = (yy >= 0 && yy < hw && xx >= 0 && xx < hw) ? __ldg(ip + yy * hw + xx) : 0.f;
#pragma unroll
        for (int j = 0; j < CO_PER_THREAD; ++j) {
          int co = co0 + j;
          if (co < cout) acc[j] += v * __ldg(w + ((size_t(co) * cin + ci) * KS + ky) * KS + kx);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CO_PER_THREAD; ++j) {
    int co = co0 + j;
    if (co >= cout) break;
    float v = acc[j] + (bias ? bias[co] : 0.f);
    if (act == 1) {
      v = __fadd_rn(__fmul_rn(v, scale[co]), shift[co]);
      v = v >= 0.f ? v : __fmul_rn(slope, v);
    } else if (act == 2) {
      v = fmaxf(v, 0.f);
    }
    out[(size_t(n) * cout_tot + cout_off + co) * npx + pix] = v;
  }
}

// maxpool2x2 (cnn.py:152-156)
__global__ void k_maxpool_f32(const float* __restrict__ in, int c_tot, int c_off, int c,
                              float* __restrict__ out, int hw_out, int64_t total) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int x = int(i % hw_out);
  int64_t r = i / hw_out;
  int y = int(r % hw_out);
  r /= hw_out;
  int ch = int(r % c);
  int64_t n = r / c;
  int hw_in = 2 * hw_out;
  const float* p = in + ((n * c_tot + c_off + ch) * hw_in + 2 * y) * hw_in + 2 * x;
  float m = fmaxf(fmaxf(p[0], p[1]), fmaxf(p[hw_in], p[hw_in + 1]));
  out[i] = m;
}

// 2x bilinear, align_corners=False, rows then columns exactly as
// upsample_bilinear2x2 (cnn.py:159-174) in fp32 without FMA.
__device__ __forceinline__ void up_weights(int o, int n, int& i0, int& i1, float& fr) {
  double src = fmax((double(o) + 0.5) / 2.0 - 0.5, 0.0);
  int a = int(src);
  i0 = a < n - 1 ? a : n - 1;
  i1 = i0 + 1 < n - 1 ? i0 + 1 : n - 1;
  fr = float(src - double(i0));
}

__global__ void k_upsample_f32(const float* __restrict__ in, int c, int hw_in,
                               float* __restrict__ out, int c_tot, int64_t total) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int hw_out = 2 * hw_in;
  int x = int(i % hw_out);
  int64_t r = i / hw_out;
  int y = int(r % hw_out);
  r /= hw_out;
  int ch = int(r % c);
  int64_t n = r / c;
  int r0, r1, c0, c1;
  float fr, fc;
  up_weights(y, hw_in, r0, r1, fr);
  up_weights(x, hw_in, c0, c1, fc);
  const float* p = in + (n * c + ch) * hw_in * hw_in;
  float omr = __fsub_rn(1.f, fr), omc = __fsub_rn(1.f, fc);
  float t0 = __fadd_rn(__fmul_rn(p[r0 * hw_in + c0], omr), __fmul_rn(p[r1 * hw_in + c0], fr));
  float t1 = __fadd_rn(__fmul_rn(p[r0 * hw_in + c1], omr), __fmul_rn(p[r1 * hw_in + c1], fr));
  out[((n * c_tot + ch) * hw_out + y) * hw_out + x] = __fadd_rn(__fmul_rn(t0, omc), __fmul_rn(t1, fc));
}

}  // namespace

int conv_f32(const ConvLayer& L, const float* in, int cin_tot, int cin_off, float* out,
             int cout_tot, int cout_off, int64_t n, float slope, cudaStream_t st) {
  int npx = L.hw * L.hw;
  dim3 grid((npx + 255) / 256, (L.cout + CO_PER_THREAD - 1) / CO_PER_THREAD, unsigned(n));
  int act = L.mode >= 0 ? L.mode : (L.act ? 1 : 2);
  if (L.ksize == 3)
    k_conv_f32<3><<<grid, 256, 0, st>>>(in, cin_tot, cin_off, L.cin, L.d_w, L.d_bias, L.d_scale,
                                        L.d_shift, act, slope, out, cout_tot, cout_off, L.cout,
                                        L.hw);
  else
    k_conv_f32<1><<<grid, 256, 0, st>>>(in, cin_tot, cin_off, L.cin, L.d_w, L.d_bias, L.d_scale,
                                        L.d_shift, act, slope, out, cout_tot, cout_off, L.cout,
                                        L.hw);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_conv_f32");
}

int maxpool_f32(const float* in, int c_tot, int c_off, int c, int hw_out, float* out, int64_t n,
                cudaStream_t st) {
  int64_t total = n * c * hw_out * hw_out;
  k_maxpool_f32<<<unsigned((total + 255) / 256), 256, 0, st>>>(in, c_tot, c_off, c, out, hw_out,
                                                                total);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_maxpool_f32");
}

int upsample_f32(const float* in, int c, int hw_in, float* out, int c_tot, int64_t n,
                 cudaStream_t st) {
  int64_t total = n * c * 4 * hw_in * hw_in;
  k_upsample_f32<<<unsigned((total + 255) / 256), 256, 0, st>>>(in, c, hw_in, out, c_tot, total);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e, "k_upsample_f32");
}

// fp32 forward over n maps, NCHW (cnn.py:193-215). Encoder skips are written
// straight into the skip slices of the decoder concat buffers, upsampled
// tensors into their leading slices, so torch.cat/np.concatenate never runs.
int forward_f32(const NetImpl& net, const float* x, float* y, int64_t n, cudaStream_t st) {
  const int k = net.k;
  const auto& Ls = net.layers;
  const size_t sz[] = {
      size_t(3 * k) * 1024, size_t(k) * 1024, size_t(k) * 1024, size_t(k) * 256,     // c1 e32 d32 p1
      size_t(6 * k) * 256,  size_t(2 * k) * 256, size_t(2 * k) * 256, size_t(2 * k) * 64,  // c2 e16 d16 p2
      size_t(12 * k) * 64,  size_t(4 * k) * 64, size_t(4 * k) * 64, size_t(4 * k) * 16,    // c3 e8 d8 p3
      size_t(8 * k) * 16,   size_t(8 * k) * 16, size_t(k / 2) * 1024, size_t(k / 4) * 1024};  // b0 b1 h1 h2
  constexpr int NB = 16;
  size_t per = 0;
  for (size_t v : sz) per += v;
  float* buf = nullptr;
  DRCB_CUDA(cudaMallocAsync((void**)&buf, per * size_t(n) * sizeof(float), st));
  float* B[NB];
  float* cur = buf;
  for (int i = 0; i < NB; ++i) {
    B[i] = cur;
    cur += sz[i] * size_t(n);
  }
  float *c1 = B[0], *e32 = B[1], *d32 = B[2], *p1 = B[3], *c2 = B[4], *e16 = B[5], *d16 = B[6],
        *p2 = B[7], *c3 = B[8], *e8 = B[9], *d8 = B[10], *p3 = B[11], *b0 = B[12], *b1 = B[13],
        *h1 = B[14], *h2 = B[15];
  const float s = net.slope;
  int rc = 0;
  rc |= conv_f32(Ls[0], x, 7, 0, e32, k, 0, n, s, st);
  rc |= conv_f32(Ls[1], e32, k, 0, c1, 3 * k, 2 * k, n, s, st);
  rc |= maxpool_f32(c1, 3 * k, 2 * k, k, 16, p1, n, st);
  rc |= conv_f32(Ls[2], p1, k, 0, e16, 2 * k, 0, n, s, st);
  rc |= conv_f32(Ls[3], e16, 2 * k, 0, c2, 6 * k, 4 * k, n, s, st);
  rc |= maxpool_f32(c2, 6 * k, 4 * k, 2 * k, 8, p2, n, st);
  rc |= conv_f32(Ls[4], p2, 2 * k, 0, e8, 4 * k, 0, n, s, st);
  rc |= conv_f32(Ls[5], e8, 4 * k, 0, c3, 12 * k, 8 * k, n, s, st);
  rc |= maxpool_f32(c3, 12 * k, 8 * k, 4 * k, 4, p3, n, st);
  rc |= conv_f32(Ls[6], p3, 4 * k, 0, b0, 8 * k, 0, n, s, st);
  rc |= conv_f32(Ls[7], b0, 8 * k, 0, b1, 8 * k, 0, n, s, st);
  rc |= upsample_f32(b1, 8 * k, 4, c3, 12 * k, n, st);
  rc |= conv_f32(Ls[8], c3, 12 * k, 0, e8, 4 * k, 0, n, s, st);
  rc |= conv_f32(Ls[9], e8, 4 * k, 0, d8, 4 * k, 0, n, s, st);
  rc |= upsample_f32(d8, 4 * k, 8, c2, 6 * k, n, st);
  rc |= conv_f32(Ls[10], c2, 6 * k, 0, e16, 2 * k, 0, n, s, st);
  rc |= conv_f32(Ls[11], e16, 2 * k, 0, d16, 2 * k, 0, n, s, st);
  rc |= upsample_f32(d16, 2 * k, 16, c1, 3 * k, n, st);
  rc |= conv_f32(Ls[12], c1, 3 * k, 0, e32, k, 0, n, s, st);
  rc |= conv_f32(Ls[13], e32, k, 0, d32, k, 0, n, s, st);
  rc |= conv_f32(Ls[14], d32, k, 0, h1, k / 2, 0, n, s, st);
  rc |= conv_f32(Ls[15], h1, k / 2, 0, h2, k / 4, 0, n, s, st);
  rc |= conv_f32(Ls[16], h2, k / 4, 0, y, 3, 0, n, s, st);
  DRCB_CUDA(cudaFreeAsync(buf, st));
  return rc;
}

}  // namespace drcb

using namespace drcb;

extern "C" int drcb_net_create(const void* drcw, size_t len, DrcbNet** out) {
  if (!drcw || !out) return fail(DRCB_ECONTRACT, "drcb_net_create: null argument");
  *out = nullptr;
  Reader r{static_cast<const uint8_t*>(drcw), len};
  char magic[4];
  if (!r.take(magic, 4)) return format_error("truncated while reading magic", r.len);
  if (std::memcmp(magic, "DRCW", 4) != 0) return format_error("bad magic, not a DRCW file", 0);
  uint32_t version, slope_bits, count;
  if (!r.take(&version, 4) || !r.take(&slope_bits, 4))
    return format_error("truncated while reading header", r.len);
  if (version != 1) return format_error("unsupported DRCW version " + std::to_string(version), 4);
  if (!r.take(&count, 4)) return format_error("truncated while reading tensor count", r.len);
  DrcbNet* net = new DrcbNet();
  NetImpl& N = net->impl;
  N.version = version;
  N.slope_bits = slope_bits;
  std::memcpy(&N.slope, &slope_bits, 4);
  for (uint32_t t = 0; t < count; ++t) {
    uint16_t nlen;
    if (!r.take(&nlen, 2)) { delete net; return format_error("truncated while reading name length", r.len); }
    std::string name(nlen, '\0');
    if (!r.take(&name[0], nlen)) { delete net; return format_error("truncated while reading tensor name", r.len); }
    uint8_t rank;
    if (!r.take(&rank, 1)) { delete net; return format_error("truncated while reading rank", r.len); }
    std::vector<uint32_t> dims(rank);
    if (!r.take(dims.data(), 4 * size_t(rank))) {
      delete net;
      return format_error("truncated while reading " + name + " dims", r.len);
    }
    size_t cnt = 1;
    for (uint32_t d : dims) cnt *= d;
    std::vector<float> data(cnt);
    if (!r.take(data.data(), 4 * cnt)) {
      delete net;
      return format_error("truncated while reading " + name + " data", r.len);
    }
    N.tensors[name] = std::move(data);
    N.shapes[name] = dims;
  }
  if (r.off != r.len) { delete net; return format_error("trailing bytes after last tensor", r.off); }
  auto it = N.shapes.find("enc1.conv1.weight");
  if (it == N.shapes.end() || it->second.empty()) {
    delete net;
    return fail(DRCB_EFORMAT, "missing tensor 'enc1.conv1.weight'");
  }
  N.k = int(it->second[0]);
  if (N.k < 4 || N.k % 4 != 0) {
    delete net;
    return fail(DRCB_EFORMAT, "base width must be a positive multiple of 4, got " + std::to_string(N.k));
  }
  auto arch = architecture(N.k);
  for (auto& kv : arch)
    if (!N.shapes.count(kv.first)) {
      delete net;
      return fail(DRCB_EFORMAT, "missing tensor '" + kv.first + "'");
    }
  for (auto& kv : N.shapes)
    if (!arch.count(kv.first)) {
      delete net;
      return fail(DRCB_EFORMAT, "unexpected tensor '" + kv.first + "'");
    }
  for (auto& kv : arch)
    if (N.shapes[kv.first] != kv.second) {
      delete net;
      return fail(DRCB_EFORMAT, "shape mismatch for '" + kv.first + "'");
    }
  for (auto& kv : N.tensors) N.n_params += int64_t(kv.second.size());

  // layer table in forward order; deconvs converted to conv form
  struct Spec { const char* name; const char* bn; int cin, cout, hw, ks; bool deconv; };
  const int k = N.k;
  std::vector<Spec> specs = {
      {"enc1.conv1", "enc1.bn1", 7, k, 32, 3, false},
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
      {"head.conv_out", "", k / 4, 3, 32, 1, false},
  };
  cudaGetDevice(&N.device);
  for (const Spec& sp : specs) {
    ConvLayer L;
    L.name = sp.name;
    L.bn = sp.bn;
    L.cin = sp.cin;
    L.cout = sp.cout;
    L.hw = sp.hw;
    L.ksize = sp.ks;
    L.act = sp.bn[0] != '\0';
    const std::vector<float>& W = N.tensors[L.name + ".weight"];
    L.w.resize(size_t(L.cout) * L.cin * L.ksize * L.ksize);
    if (sp.deconv) {
      // (cin, cout, 3, 3) -> conv (cout, cin, 3, 3) flipped (cnn.py:124-131)
      for (int co = 0; co < L.cout; ++co)
        for (int ci = 0; ci < L.cin; ++ci)
          for (int ky = 0; ky < 3; ++ky)
            for (int kx = 0; kx < 3; ++kx)
              L.w[((size_t(co) * L.cin + ci) * 3 + ky) * 3 + kx] =
                  W[((size_t(ci) * L.cout + co) * 3 + (2 - ky)) * 3 + (2 - kx)];
    } else {
      L.w = W;
    }
    L.bias = N.tensors[L.name + ".bias"];
    L.scale.assign(L.cout, 1.f);
    L.shift.assign(L.cout, 0.f);
    if (L.act) {
      const auto& g = N.tensors[L.bn + ".gamma"];
      const auto& b = N.tensors[L.bn + ".beta"];
      const auto& m = N.tensors[L.bn + ".running_mean"];
      const auto& v = N.tensors[L.bn + ".running_var"];
      for (int c = 0; c < L.cout; ++c) {
        float var = v[c] + 1e-5f;  // float32 + weak python float (cnn.py:136)
        if (!(var > 0.f)) {
          delete net;
          return fail(DRCB_EFORMAT, "nonpositive running_var + eps");
        }
        float sc = g[c] / sqrtf(var);
        L.scale[c] = sc;
        L.shift[c] = b[c] - m[c] * sc;
      }
    }
    L.d_w = dev_copy(N, L.w);
    L.d_bias = dev_copy(N, L.bias);
    L.d_scale = dev_copy(N, L.scale);
    L.d_shift = dev_copy(N, L.shift);
    if (!L.d_w || !L.d_bias || !L.d_scale || !L.d_shift) {
      delete net;
      return fail(DRCB_ECUDA, "cudaMalloc failed for network weights");
    }
    N.layers.push_back(std::move(L));
  }
  *out = net;
  return 0;
}

extern "C" void drcb_net_destroy(DrcbNet* net) {
  if (!net) return;
  for (void* p : net->impl.allocs) cudaFree(p);
  delete net;
}

extern "C" int drcb_net_info(const DrcbNet* net, int64_t* out4) {
  if (!net || !out4) return fail(DRCB_ECONTRACT, "drcb_net_info: null argument");
  out4[0] = net->impl.k;
  out4[1] = net->impl.n_params;
  out4[2] = net->impl.version;
  out4[3] = net->impl.slope_bits;
  return 0;
}
