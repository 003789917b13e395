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
int tc_layer_forward_group(cudaStream_t st, const dqn_net_desc *net, int l,
                           const float *on_params, const dqn_binding *on_b,
                           const float *tg_params, const dqn_binding *tg_b, float *scratch,
                           int *counters);
int64_t tc_forward_group_scratch(const dqn_net_desc *net, int upto, int batch);
int lin_wgrad_smallk(cudaStream_t st, const float *x, const float *dy, int B, int F, int N,
                     float *gw, float *gb, int32_t *flags);
int small_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                        const dqn_binding *b);
int conv_wgrad_u8_smallk(cudaStream_t st, const uint8_t *xt, const float *dy, int M, int N, int P,
                         float *gw, float *gb, float *scratch, int64_t scratch_floats,
                         int32_t *flags);

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

// opt-in (DQN_B200_SMALL_FWD_ROWS=n): forwards of at most n rows use the
// small-batch SIMT kernel for hidden conv / linear layers.  Measured at batch
// 1: conv layers 4-15 us, but a linear layer is a single output pixel (N/32
// CTAs walking K = 2048-3136 serially: 35-53 us), so the act forward is
// faster on the tcgen05 path (desk 59 vs 64 us, Atari 65 vs 112 us) -> off.
static int small_batch_rows() {
  static const int n = [] {
    const char *e = getenv("DQN_B200_SMALL_FWD_ROWS");
    return e ? atoi(e) : 0;
  }();
  return n;
}
static int layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                         const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  const bool hidden = l != net->n_layers - 1 && net->algo != 1 &&
                      (L.kind == DQN_LAYER_CONV || L.kind == DQN_LAYER_LINEAR);
  // acting-sized batches: layers without a tcgen05 kernel (e.g. the desk
  // net's 16-filter conv1: 24.3 -> 4.1 us at batch 1) take the small-batch
  // kernel instead of the batched SIMT GEMM; tcgen05 layers stay (faster)
  if (hidden && ((b->batch <= 4 && !use_tc(net, l, 0)) || b->batch <= small_batch_rows()))
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
// hold (measured +0.6 % in the learner); DQN_B200_LIN_WGRAD_SIMT=0 turns it off
static bool lin_wgrad_simt_enabled() {
  const char *e = getenv("DQN_B200_LIN_WGRAD_SIMT");
  return !(e && e[0] == '0');
}
// opt-in: the FMA reduction measured 31.8 us vs 17.7 us for the tcgen05 wgrad
static bool conv_u8_wgrad_simt_enabled() {
  const char *e = getenv("DQN_B200_CONV1_WGRAD_SIMT");
  return e && e[0] == '1';
}
static int layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                       const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  // hidden linear layers at learner batch sizes: the small-K FMA kernel
  if (L.kind == DQN_LAYER_LINEAR && l != net->n_layers - 1 && l > 0 && b->batch <= 64 &&
      net->algo != 1 && lin_wgrad_simt_enabled())
    return lin_wgrad_smallk(st, b->act[l - 1], b->dact[l], b->batch,
                            L.in_h * L.in_w * L.in_c, L.out_c, grads + L.w_off,
                            grads + L.b_off, flags);
  // the uint8 first conv from its transposed patch operand: FMA reduction
  if (l == 0 && net->input_u8 && b->xt && L.kind == DQN_LAYER_CONV && b->batch <= 64 &&
      net->algo != 1 && conv_u8_wgrad_simt_enabled()) {
    const int M = L.fh * L.fw * L.in_c, P = b->batch * L.out_h * L.out_w;
    const int rc = conv_wgrad_u8_smallk(st, b->xt, b->dact[0], M, L.out_c, P, grads + L.w_off,
                                        grads + L.b_off, b->scratch,
                                        b->scratch_floats - kTileCounters, flags);
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
extern "C" int dqn_abi_version(void) { return 3; }
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

extern "C" int64_t dqn_net_forward_group_scratch(const dqn_net_desc *net, int32_t upto,
                                                 int32_t batch) {
  if (!net || upto < 0 || upto > net->n_layers || batch < 1) return -1;
  return tc_forward_group_scratch(net, upto, batch) + kTileCounters;
}

extern "C" int dqn_net_forward_group(void *stream, const dqn_net_desc *net,
                                     const float *on_params, const dqn_binding *on_bind,
                                     const float *tg_params, const dqn_binding *tg_bind,
                                     int32_t upto, float *scratch, int64_t scratch_floats,
                                     int32_t *flags) {
  int st = check_binding(net, on_bind);
  if (st) return st;
  st = check_binding(net, tg_bind);
  if (st) return st;
  if (upto < 0 || upto > net->n_layers || on_bind->batch != 2 * tg_bind->batch || !scratch ||
      scratch_floats < dqn_net_forward_group_scratch(net, upto, tg_bind->batch)) {
    set_error("forward_group: need on batch = 2 x target batch, upto <= layers, scratch");
    return DQN_ERR_INVALID_ARG;
  }
  cudaStream_t s = as_stream(stream);
  int *counters = reinterpret_cast<int *>(scratch + scratch_floats - kTileCounters);
  for (int l = 0; l < upto; ++l) {
    if (use_tc(net, l, 0)) {
      st = tc_layer_forward_group(s, net, l, on_params, on_bind, tg_params, tg_bind, scratch,
                                  counters);
    } else {
      st = layer_forward(s, net, l, on_params, on_bind, flags);
      if (!st) st = layer_forward(s, net, l, tg_params, tg_bind, flags);
    }
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
