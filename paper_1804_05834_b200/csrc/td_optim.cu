// Fused Double-DQN target / TD-loss kernel and the fused RMSprop optimizer.
//
//   compute_target_double / _dqn   agent.py:58-73   -> td_loss_kernel
//   learn_step loss block          agent.py:110-124 -> td_loss_kernel
//   RmsProp.step                   optim.py:36-47   -> rms_scan_kernel + rms_apply_kernel
//   clip_gradients                 optim.py:61-75   -> sqnorm kernels + scale
//   sync_target                    optim.py:78-89   -> cudaMemcpyAsync
//
// TD arithmetic is fp64 with explicit _rn intrinsics in the reference's
// operation order; RMSprop is fp32 _rn in the order numpy evaluates
// optim.py:44-46 under NEP-50 weak-scalar promotion, so it is bit-exact given
// identical gradients.
#include "common.cuh"
#include "td_row.cuh"

#include <algorithm>

namespace dqn {
namespace {

constexpr int kTdThreads = 256;

__global__ void __launch_bounds__(kTdThreads)
td_loss_kernel(const float *__restrict__ q_on, const float *__restrict__ q_next_on,
               const float *__restrict__ q_next_tg, const int64_t *__restrict__ actions,
               const double *__restrict__ rewards, const uint8_t *__restrict__ terminals,
               const double *__restrict__ weights, int B, int nA, double gamma, int flags,
               double *__restrict__ targets, double *__restrict__ td,
               double *__restrict__ losses, float *__restrict__ dq, double *__restrict__ stats) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ double s_abs[kTdThreads], s_loss[kTdThreads];
  const int t = threadIdx.x;
  double acc_abs = 0.0, acc_loss = 0.0;
  for (int j = t; j < B; j += blockDim.x) {
    double ad, l;
    td_row(j, q_on, q_next_on, q_next_tg, actions, rewards, terminals, weights, nA, gamma, flags,
           targets, td, losses, dq, ad, l);
    acc_abs = __dadd_rn(acc_abs, ad);
    acc_loss = __dadd_rn(acc_loss, l);
  }
  if (stats == nullptr) return;
  s_abs[t] = acc_abs;
  s_loss[t] = acc_loss;
  __syncthreads();
  for (int s = kTdThreads / 2; s > 0; s >>= 1) {
    if (t < s) {
      s_abs[t] = __dadd_rn(s_abs[t], s_abs[t + s]);
      s_loss[t] = __dadd_rn(s_loss[t], s_loss[t + s]);
    }
    __syncthreads();
  }
  if (t == 0) {
    stats[0] = s_abs[0];
    stats[1] = s_loss[0];
  }
}

// -------------------------------------------------------------- RMSprop

__global__ void rms_scan_kernel(const float *__restrict__ g, int64_t n, int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, DQN_FLAG_NONFINITE_GRAD);
}

__device__ __forceinline__ void rms_one(float &w, float &g, float &a, float lr, float rho,
                                        float omr, float eps) {
  a = __fmul_rn(a, rho);                                          // acc *= decay
  a = __fadd_rn(a, __fmul_rn(omr, __fmul_rn(g, g)));              // acc += (1-decay)*g^2
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, g), __fadd_rn(__fsqrt_rn(a), eps)));
  g = 0.f;
}

__global__ void rms_apply_kernel(float *__restrict__ w, float *__restrict__ g,
                                 float *__restrict__ acc, int64_t n, float lr, float rho,
                                 float omr, float eps, const int32_t *__restrict__ flags,
                                 int32_t *flag_out) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  // completion signal for the host: every earlier kernel of the update has
  // finished (and its host-memory results were fenced) once this runs
  if (flag_out && blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    *(volatile int32_t *)flag_out = *flags;
  }
  // optim.py:38-40: a non-finite gradient aborts the step before any update;
  // any earlier failure of this step (the reference would have raised before
  // reaching the optimizer) does too.  Flags are sticky until the host reads.
  if (*flags & (DQN_FLAG_NONFINITE_GRAD | DQN_FLAG_NONFINITE_OUT | DQN_FLAG_ZERO_TOTAL |
                DQN_FLAG_BAD_PRIORITY | DQN_FLAG_INDEX))
    return;
  const int64_t n4 = n / 4;
  float4 *w4 = reinterpret_cast<float4 *>(w);
  float4 *g4 = reinterpret_cast<float4 *>(g);
  float4 *a4 = reinterpret_cast<float4 *>(acc);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 wv = w4[i], gv = g4[i], av = a4[i];
    rms_one(wv.x, gv.x, av.x, lr, rho, omr, eps);
    rms_one(wv.y, gv.y, av.y, lr, rho, omr, eps);
    rms_one(wv.z, gv.z, av.z, lr, rho, omr, eps);
    rms_one(wv.w, gv.w, av.w, lr, rho, omr, eps);
    w4[i] = wv;
    g4[i] = gv;
    a4[i] = av;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    rms_one(w[i], g[i], acc[i], lr, rho, omr, eps);
}

// ---------------------------------------------------------- grad clipping

constexpr int kNormBlocks = 148;

__global__ void sqnorm_partial_kernel(const float *__restrict__ g, int64_t n,
                                      double *__restrict__ partial) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)g[i];
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sqnorm_final_kernel(double *__restrict__ partial, int nb, double max_norm,
                                    double *__restrict__ norm_out) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < nb; ++i) s = __dadd_rn(s, partial[i]);
  const double norm = sqrt(s);
  *norm_out = norm;
  // scale factor (float32), or 0 meaning "no clipping"
  partial[nb] = (norm > max_norm && norm > 0.0) ? (double)(float)(max_norm / norm) : 0.0;
}

__global__ void grad_scale_kernel(float *__restrict__ g, int64_t n,
                                  const double *__restrict__ scale_p) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const double sd = *scale_p;
  if (sd == 0.0) return;
  const float s = (float)sd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] = __fmul_rn(g[i], s);
}

}  // namespace
}  // namespace dqn

using namespace dqn;

extern "C" int dqn_td_loss(void *stream, const float *q_online, const float *q_next_online,
                           const float *q_next_target, const int64_t *actions,
                           const double *rewards, const uint8_t *terminals,
                           const double *weights, int32_t batch, int32_t n_actions, double gamma,
                           int32_t flags, double *targets, double *td, double *losses, float *dq,
                           double *stats) {
  DQN_CHECK_ARG(q_online && q_next_target && actions && rewards && terminals && weights && targets &&
                    td && losses && dq && batch >= 1 && n_actions >= 1,
                "td_loss: bad args");
  DQN_CHECK_ARG(!(flags & DQN_TD_DOUBLE) || q_next_online, "td_loss: double needs q_next_online");
  launch_k(td_loss_kernel, 1, kTdThreads, 0, as_stream(stream), 
      q_online, q_next_online, q_next_target, actions, rewards, terminals, weights, batch,
      n_actions, gamma, flags, targets, td, losses, dq, stats);
  DQN_LAUNCH_CHECK("td_loss");
  return DQN_OK;
}

extern "C" int dqn_rmsprop_step(void *stream, float *w, float *g, float *acc, int64_t n, float lr,
                                float rho, float one_minus_rho, float eps, int32_t *flags) {
  DQN_CHECK_ARG(w && g && acc && flags && n >= 0, "rmsprop: bad args");
  DQN_CHECK_ARG(((uintptr_t)w | (uintptr_t)g | (uintptr_t)acc) % 16 == 0,
                "rmsprop: buffers must be 16-byte aligned");
  if (n == 0) return DQN_OK;
  cudaStream_t st = as_stream(stream);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  launch_k(rms_scan_kernel, blocks, 256, 0, st, g, n, flags);
  DQN_LAUNCH_CHECK("rms_scan");
  const int blocks4 = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, 148 * 4));
  launch_k(rms_apply_kernel, blocks4, 256, 0, st, w, g, acc, n, lr, rho, one_minus_rho, eps, flags,
           (int32_t *)nullptr);
  DQN_LAUNCH_CHECK("rms_apply");
  return DQN_OK;
}

// The apply kernel alone: for gradients whose producers flagged non-finite
// values as they wrote them (dqn_net_layer phase 2 with flags, dqn_head_td);
// the step is skipped on any error flag exactly as in dqn_rmsprop_step.
#ifdef DQN_TC_TRACE
int g_rms_cap = 148 * 8;
extern "C" void dqn_rms_set_cap(int c) { g_rms_cap = c; }
#else
constexpr int g_rms_cap = 148 * 8;
#endif

extern "C" int dqn_rmsprop_apply(void *stream, float *w, float *g, float *acc, int64_t n,
                                 float lr, float rho, float one_minus_rho, float eps,
                                 int32_t *flags, int32_t *flag_out) {
  DQN_CHECK_ARG(w && g && acc && flags && n >= 0, "rmsprop: bad args");
  DQN_CHECK_ARG(((uintptr_t)w | (uintptr_t)g | (uintptr_t)acc) % 16 == 0,
                "rmsprop: buffers must be 16-byte aligned");
  if (n == 0) return DQN_OK;
  const int cap = g_rms_cap;                            // measured best in the learner graph
  const int blocks4 = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, cap));
  launch_k(rms_apply_kernel, blocks4, 256, 0, as_stream(stream), w, g, acc, n, lr, rho,
           one_minus_rho, eps, flags, flag_out);
  DQN_LAUNCH_CHECK("rms_apply");
  return DQN_OK;
}

extern "C" int dqn_clip_gradients(void *stream, float *g, int64_t n, double max_norm,
                                  double *norm_out) {
  DQN_CHECK_ARG(g && norm_out && n >= 0, "clip: bad args");
  // partial sums live in a process-wide scratch allocated once
  static double *partial = nullptr;
  if (!partial) {
    int st = cuda_status(cudaMalloc(&partial, sizeof(double) * (kNormBlocks + 1)), "clip scratch");
    if (st) return st;
  }
  cudaStream_t st = as_stream(stream);
  launch_k(sqnorm_partial_kernel, kNormBlocks, 256, 0, st, g, n, partial);
  DQN_LAUNCH_CHECK("sqnorm_partial");
  launch_k(sqnorm_final_kernel, 1, 32, 0, st, partial, kNormBlocks, max_norm, norm_out);
  DQN_LAUNCH_CHECK("sqnorm_final");
  launch_k(grad_scale_kernel, kNormBlocks, 256, 0, st, g, n, partial + kNormBlocks);
  DQN_LAUNCH_CHECK("grad_scale");
  return DQN_OK;
}

extern "C" int dqn_sync_target(void *stream, float *dst, const float *src, int64_t n) {
  DQN_CHECK_ARG(dst && src && n >= 0, "sync_target: bad args");
  return cuda_status(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice,
                                     as_stream(stream)),
                     "sync_target");
}

// --- CUDA graphs with per-node priorities ---------------------------------
// torch.cuda.CUDAGraph(keep_graph=True) captures the learner update; the
// graph is instantiated here with cudaGraphInstantiateFlagUseNodePriority so
// the kernel-node priorities set by launch_k (= the capturing stream's
// priority) order CTA dispatch between the critical chain and side streams.
extern "C" int dqn_graph_instantiate(void *graph, int use_node_priority, void **exec_out) {
  DQN_CHECK_ARG(graph && exec_out, "graph_instantiate: null pointer");
  cudaGraphExec_t ex = nullptr;
  const unsigned long long fl = use_node_priority ? cudaGraphInstantiateFlagUseNodePriority : 0;
  const int rc = cuda_status(cudaGraphInstantiateWithFlags(&ex, (cudaGraph_t)graph, fl),
                             "graph_instantiate");
  if (rc != DQN_OK) return rc;
  *exec_out = (void *)ex;
  return DQN_OK;
}

extern "C" int dqn_graph_launch(void *exec, void *stream) {
  return cuda_status(cudaGraphLaunch((cudaGraphExec_t)exec, as_stream(stream)), "graph_launch");
}

extern "C" int dqn_graph_destroy(void *exec) {
  if (!exec) return DQN_OK;
  return cuda_status(cudaGraphExecDestroy((cudaGraphExec_t)exec), "graph_destroy");
}
