// C-ABI entry points of the network phases (network.py:90-126).  Layers are
// dispatched to the tcgen05 trunk kernels when one exists for the geometry
// (trunk_tc.cu), otherwise to the generic SIMT kernels (net_simt.cu).
#include "common.cuh"

#include <string.h>

#include <atomic>

namespace dqn {

int simt_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                       const dqn_binding *b, int32_t *flags);
int simt_layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                        const dqn_binding *b);
int simt_layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                     const dqn_binding *b, int32_t *flags);
int64_t simt_scratch_floats(const dqn_net_desc *net, int batch);
int simt_validate(const dqn_net_desc *net);
bool tc_layer_supported(const dqn_net_desc *net, int l, int phase);
int64_t tc_scratch_floats(const dqn_net_desc *net, int batch);
int tc_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                     const dqn_binding *b);
int tc_layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                      const dqn_binding *b);
int tc_layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                   const dqn_binding *b, int32_t *flags);
bool conv1_wgrad_u8_ok(const dqn_net_desc *net);
int conv1_wgrad_u8_tc(cudaStream_t st, const dqn_net_desc *net, const uint8_t *x,
                      const float *dy, float *grads, float *scratch, int *counters, int batch,
                      int32_t *flags);
int lin_wgrad_smallk(cudaStream_t st, const float *x, const float *dy, int B, int F, int N,
                     float *gw, float *gb, int32_t *flags);
int small_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                        const dqn_binding *b);

// tcgen05 trunk for supported geometries unless the descriptor asks for SIMT
static bool use_tc(const dqn_net_desc *net, int l, int phase) {
  return net->algo != 1 && tc_layer_supported(net, l, phase);
}

// SIMT and tcgen05 partial buffers share the front of the scratch; the
// split-K tile-counter table (kTileCounters ints) always sits after both.
constexpr int64_t kTileCounters = 16384;   // == tc::kMaxTiles
static int64_t scratch_need(const dqn_net_desc *net, int batch) {
  const int64_t a = simt_scratch_floats(net, batch), b = tc_scratch_floats(net, batch);
  return (a > b ? a : b) + kTileCounters;
}

static int layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                         const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  const bool hidden = l != net->n_layers - 1 && net->algo != 1 &&
                      (L.kind == DQN_LAYER_CONV || L.kind == DQN_LAYER_LINEAR);
  // acting-sized batches: layers without a tcgen05 kernel (e.g. the desk
  // net's 16-filter conv1: 24.3 -> 4.1 us at batch 1) take the small-batch
  // kernel instead of the batched SIMT GEMM; tcgen05 layers stay (faster
  // also at batch 1: a linear layer as one output pixel walks K serially in
  // the small kernel -- desk act 59 vs 64 us, Atari 65 vs 112 us)
  if (hidden && b->batch <= 4 && !use_tc(net, l, 0))
    return small_layer_forward(st, net, l, params, b);
  if (use_tc(net, l, 0)) return tc_layer_forward(st, net, l, params, b);
  return simt_layer_forward(st, net, l, params, b, flags);
}
static int layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                          const dqn_binding *b) {
  if (use_tc(net, l, 1)) return tc_layer_backward(st, net, l, params, b);
  return simt_layer_backward(st, net, l, params, b);
}
// flags (optional): every written gradient is checked for non-finite values
// fc1's wgrad is an outer-product sum over the batch rows: the FMA kernel's
// short CTAs leave SMs to the dgrad chain that 200 one-block tcgen05 CTAs
// hold (measured +0.6 % in the learner)
static int layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                       const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  // hidden linear layers at learner batch sizes: the small-K FMA kernel
  // (a tcgen05 form -- both operands TMA-loaded and transposed in smem, one
  // 32-k stage, 100 CTAs -- measured 18.8 vs 12.9 us and -5 % in the learner)
  if (L.kind == DQN_LAYER_LINEAR && l != net->n_layers - 1 && l > 0 && b->batch <= 64 &&
      net->algo != 1)
    return lin_wgrad_smallk(st, b->act[l - 1], b->dact[l], b->batch,
                            L.in_h * L.in_w * L.in_c, L.out_c, grads + L.w_off,
                            grads + L.b_off, flags);
  // the uint8 first conv straight from the frames (csrc/wgrad_u8.cu)
  if (l == 0 && conv1_wgrad_u8_ok(net)) {
    const int rc = conv1_wgrad_u8_tc(st, net, (const uint8_t *)b->x, b->dact[0], grads,
                                     b->scratch,
                                     reinterpret_cast<int *>(b->scratch + b->scratch_floats -
                                                             kTileCounters),
                                     b->batch, flags);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
  }
  if (use_tc(net, l, 2)) return tc_layer_wgrad(st, net, l, grads, b, flags);
  return simt_layer_wgrad(st, net, l, grads, b, flags);
}

namespace {
thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace dqn

using namespace dqn;

extern "C" const char *dqn_last_error(void) { return g_err; }
extern "C" int dqn_abi_version(void) { return 5; }
extern "C" int dqn_has_tcgen05(void) { return 1; }
extern "C" int64_t dqn_launch_count(void) { return g_launches.load(); }

extern "C" int64_t dqn_net_scratch_floats(const dqn_net_desc *net, int32_t batch) {
  if (simt_validate(net) != DQN_OK || batch < 1) return -1;
  return scratch_need(net, batch);
}

static int check_binding(const dqn_net_desc *net, const dqn_binding *b) {
  int st = simt_validate(net);
  if (st) return st;
  if (!b || b->batch < 1 || !b->x) {
    set_error("binding: batch/input missing");
    return DQN_ERR_INVALID_ARG;
  }
  if (b->scratch_floats < scratch_need(net, b->batch)) {
    set_error("binding: scratch too small (%lld < %lld floats)", (long long)b->scratch_floats,
              (long long)scratch_need(net, b->batch));
    return DQN_ERR_INVALID_ARG;
  }
  for (int l = 0; l < net->n_layers; ++l)
    if (!b->act[l]) {
      set_error("binding: act[%d] missing", l);
      return DQN_ERR_INVALID_ARG;
    }
  return DQN_OK;
}

extern "C" int dqn_net_forward(void *stream, const dqn_net_desc *net, const float *params,
                               const dqn_binding *bind, int32_t *flags) {
  int st = check_binding(net, bind);
  if (st) return st;
  for (int l = 0; l < net->n_layers; ++l) {
    st = layer_forward(as_stream(stream), net, l, params, bind, flags);
    if (st) return st;
  }
  return DQN_OK;
}

extern "C" int dqn_net_backward(void *stream, const dqn_net_desc *net, const float *params,
                                const dqn_binding *bind, const float *dq) {
  int st = check_binding(net, bind);
  if (st) return st;
  const int L = net->n_layers;
  for (int l = 0; l < L; ++l)
    if (!bind->dact[l]) {
      set_error("binding: dact[%d] missing", l);
      return DQN_ERR_INVALID_ARG;
    }
  cudaStream_t s = as_stream(stream);
  // y.grad = dq (network.py:112)
  if (dq != bind->dact[L - 1]) {
    st = cuda_status(cudaMemcpyAsync(bind->dact[L - 1], dq,
                                     sizeof(float) * bind->batch * net->layer[L - 1].out_c,
                                     cudaMemcpyDeviceToDevice, s),
                     "backward: copy dq");
    if (st) return st;
  }
  for (int l = L - 1; l >= 0; --l) {
    st = layer_backward(s, net, l, params, bind);
    if (st) return st;
  }
  return DQN_OK;
}

extern "C" int dqn_net_wgrad(void *stream, const dqn_net_desc *net, float *grads,
                             const dqn_binding *bind) {
  int st = check_binding(net, bind);
  if (st) return st;
  for (int l = net->n_layers - 1; l >= 0; --l) {
    st = layer_wgrad(as_stream(stream), net, l, grads, bind, nullptr);
    if (st) return st;
  }
  return DQN_OK;
}

extern "C" int dqn_net_layer(void *stream, const dqn_net_desc *net, const float *params,
                             float *grads, const dqn_binding *bind, int32_t layer, int32_t phase,
                             int32_t *flags) {
  int st = check_binding(net, bind);
  if (st) return st;
  if (layer < 0 || layer >= net->n_layers) {
    set_error("net_layer: layer %d out of range", layer);
    return DQN_ERR_INVALID_ARG;
  }
  switch (phase) {
    case 0: return layer_forward(as_stream(stream), net, layer, params, bind, flags);
    case 1: return layer_backward(as_stream(stream), net, layer, params, bind);
    case 2: return layer_wgrad(as_stream(stream), net, layer, grads, bind, flags);
    default: set_error("net_layer: bad phase %d", phase); return DQN_ERR_INVALID_ARG;
  }
}
