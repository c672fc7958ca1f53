// drcb_train.h — the DrcbTrainer handle shared by the training engines:
// drcb_train.cu (fp32 CUDA-core parity engine, Adam, export, NCCL plumbing)
// and drcb_train_tc.cu (the NHWC bf16 tensor-core engine). Not part of the ABI.
#pragma once
#include <string>
#include <vector>

#include "drcb_net.h"

namespace drcb {
namespace train {

constexpr int NL = 17;  // 16 conv/deconv + BN layers and head.conv_out
constexpr float MOMENTUM = 0.1f;
constexpr float EPS = 1e-5f;

// one layer of MapAutoencoder (model.py:20-88) in the flat parameter buffer
struct TL {
  std::string name, bn;
  int cin, cout, hw, ks;
  bool deconv, has_bn;
  int64_t w, b, g, be;  // offsets in the flat parameter buffer
  int64_t rm, rv;       // offsets in the running-stats buffer
  int64_t nw;           // weight element count
};

struct TcEngine;  // drcb_train_tc.cu
void tc_engine_destroy(TcEngine* e);

}  // namespace train
}  // namespace drcb

struct DrcbTrainer {
  int k = 0;
  float slope = 0.01f;
  uint32_t slope_bits = 0;
  std::vector<drcb::train::TL> L;
  int64_t n_params = 0, n_running = 0;
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr, *running = nullptr;
  float *wf = nullptr, *wt = nullptr;  // conv-form / dgrad-form weights (all layers)
  std::vector<int64_t> wf_off;
  float lr = 1e-4f, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
  int64_t* d_step = nullptr;  // Adam step counter (device; graph-replay safe)
  float* d_coef = nullptr;     // {lr / bc1, sqrt(bc2)} of the current step
  void* comm = nullptr;  // ncclComm_t or NULL
  int world = 1;
  std::vector<void*> allocs;
  int mode = 0;  // 0 = fp32 CUDA cores (parity), 2 = bf16 tensor cores (NHWC engine)
  drcb::train::TcEngine* tc = nullptr;
  // a reduction hook replacing NCCL (loopback ranks in one process, or a
  // host callback such as a gloo all-reduce): drcb_trainer_set_reducer
  DrcbReduceFn reduce_fn = nullptr;
  void* reduce_user = nullptr;
  // bucketed gradient all-reduce (NCCL): a side stream + one event per layer
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_ev[18] = {};
  cudaEvent_t sync_ev[2] = {};  // SyncBN all-reduces routed through comm_stream
};

namespace drcb {
namespace train {
// the NHWC bf16 tensor-core step (drcb_train_tc.cu): forward, loss, backward
// into T->grads (gradient all-reduce and Adam stay with the caller)
int tc_step(DrcbTrainer* T, const float* x, const float* y, int64_t n, double** loss_dev_sum,
            cudaStream_t st);
// sum-all-reduce over the data-parallel ranks through the trainer's
// communicator: the reduction hook if set, else NCCL (no-op for one rank)
int trainer_allreduce(DrcbTrainer* T, void* buf, size_t count, int is_double, cudaStream_t st);
// the flat-buffer range [off, off + count) of layer l's parameters
void layer_param_range(const DrcbTrainer* T, int l, int64_t& off, int64_t& count);
}  // namespace train
}  // namespace drcb
