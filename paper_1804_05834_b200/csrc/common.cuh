// Shared helpers for libdqn_b200: error plumbing and exact-arithmetic
// intrinsics.  Parity-critical code uses explicit __d*_rn / __f*_rn so that
// nvcc never contracts a mul+add into an FMA the reference did not do.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <stdlib.h>

#include <utility>

#include "../../include/dqn_b200.h"

namespace dqn {

void set_error(const char *fmt, ...);
void note_launch();   // counts kernel launches issued by the library (dqn_launch_count)

inline int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return DQN_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return DQN_ERR_CUDA;
}

// After a launch: report configuration errors without synchronising.
inline int launch_status(const char *what) {
  return cuda_status(cudaGetLastError(), what);
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ void raise_flag(int32_t *flags, int32_t bit) {
  if (flags) atomicOr(flags, bit);
}

// Gradient producers flag non-finite values as they write them, so an
// optimizer step that follows only them need not rescan the gradients
// (dqn_rmsprop_apply; optim.py:38-40 semantics).
__device__ __forceinline__ void note_grad(int32_t *flags, float v) {
  if (flags && !isfinite(v)) atomicOr(flags, DQN_FLAG_NONFINITE_GRAD);
}
__device__ __forceinline__ void acc_grad(float *g, float s, int32_t *flags) {
  const float v = __fadd_rn(*g, s);
  *g = v;
  note_grad(flags, v);
}
__device__ __forceinline__ void note_grad4(int32_t *flags, float4 v) {
  if (flags && !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w)))
    atomicOr(flags, DQN_FLAG_NONFINITE_GRAD);
}

constexpr int kNumSMs = 148;

// Programmatic dependent launch: every kernel of the library is launched with
// programmatic stream serialization (launch_k), so it may be scheduled while
// the previous kernel of its stream drains.  Each kernel therefore
//   * calls pdl_trigger() first -- its own dependent may be scheduled once all
//     of this grid's CTAs are resident (a waiting dependent never holds SMs
//     this grid still needs);
//   * calls pdl_wait() before its first global access that depends on (or
//     overwrites data of) earlier kernels: it returns once every prerequisite
//     grid has completed and its memory is visible.
// Prologue work before pdl_wait (TMEM allocation, barrier setup, index math
// on kernel parameters) overlaps the previous kernel's tail.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  pdl_trigger();
  pdl_wait();
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("DQN_B200_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Kernel-node priority = the launching stream's priority, so a CUDA graph
// instantiated with cudaGraphInstantiateFlagUseNodePriority (dqn_graph_
// instantiate) schedules the learner's critical dgrad chain ahead of the
// side-stream wgrads when both have CTAs waiting for an SM.
inline cudaLaunchAttribute priority_attr(cudaStream_t st) {
  int prio = 0;
  if (cudaStreamGetPriority(st, &prio) != cudaSuccess) {
    (void)cudaGetLastError();
    prio = 0;
  }
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributePriority;
  a.val.priority = prio;
  return a;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Layer geometry in NHWC terms (linear layers: H = W = OH = OW = 1).
struct Geo {
  int H, W, C;       // input
  int OH, OW, N;     // output
  int fh, fw, sh, sw;
};

inline Geo geo_of(const dqn_layer_desc &L) {
  Geo g;
  g.H = L.in_h; g.W = L.in_w; g.C = L.in_c;
  g.OH = L.out_h; g.OW = L.out_w; g.N = L.out_c;
  g.fh = L.fh; g.fw = L.fw; g.sh = L.sh; g.sw = L.sw;
  return g;
}

}  // namespace dqn

#define DQN_CHECK_ARG(cond, ...)              \
  do {                                        \
    if (!(cond)) {                            \
      dqn::set_error(__VA_ARGS__);            \
      return DQN_ERR_INVALID_ARG;             \
    }                                         \
  } while (0)

#define DQN_LAUNCH_CHECK(what)                 \
  do {                                         \
    int _st = dqn::launch_status(what);        \
    if (_st != DQN_OK) return _st;             \
    dqn::note_launch();                        \
  } while (0)
