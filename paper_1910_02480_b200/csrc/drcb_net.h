// drcb_net.h — the DrcbNet handle: parsed DRCW weights, folded batch norm,
// per-layer device buffers for the fp32 SIMT path and the tcgen05 path.
#pragma once
#include <map>
#include <string>
#include <vector>

#include "drcb_internal.h"

namespace drcb {

// One 3x3 (or 1x1) convolution layer in conv form: transposed convolutions
// are stored pre-flipped with channel axes swapped (cnn.py:124-131).
struct ConvLayer {
  std::string name;      // e.g. "enc1.conv1", "dec3.deconv1"
  std::string bn;        // e.g. "enc1.bn1" ("" for head.conv_out)
  int cin = 0, cout = 0, ksize = 3, hw = 32;
  bool act = true;       // BN + LeakyReLU epilogue
  int mode = -1;         // SIMT epilogue override: 0 bias only, 1 BN+LReLU, 2 bias+ReLU
  // host copies
  std::vector<float> w;      // (cout, cin, k, k) conv form
  std::vector<float> bias;   // (cout)
  std::vector<float> scale;  // folded BN scale (cnn.py:134-141), fp32
  std::vector<float> shift;  // folded BN shift
  // device (fp32 SIMT path)
  float *d_w = nullptr, *d_bias = nullptr, *d_scale = nullptr, *d_shift = nullptr;
  // device (tensor-core path): K-major packed operand, fused epilogue vectors
  void* d_wtc = nullptr;     // (cout_pad, 9 * cin_pad) bf16 or fp32 (tf32)
  float *d_ep_a = nullptr, *d_ep_b = nullptr;  // y = acc * a + b, then LeakyReLU
  int cin_pad = 0, cout_pad = 0;
  int tc_kind = -1;          // which operand format d_wtc holds
  // enc1.conv1 on the tensor cores reads the compact 8-channel NHWC input and
  // builds its im2col operand in SMEM (k_conv_in8): K value tap * 8 + c
  bool in8 = false;
};

struct NetImpl {
  int k = 0;
  float slope = 0.01f;
  uint32_t slope_bits = 0;
  uint32_t version = 1;
  int64_t n_params = 0;
  std::map<std::string, std::vector<float>> tensors;
  std::map<std::string, std::vector<uint32_t>> shapes;
  std::vector<ConvLayer> layers;  // 16 layers in forward order
  std::vector<void*> allocs;
  int device = 0;
};

std::map<std::string, std::vector<uint32_t>> architecture(int k);
}  // namespace drcb

struct DrcbNet {
  drcb::NetImpl impl;
};
