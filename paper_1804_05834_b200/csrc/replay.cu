// Replay side of the learner hot path: the uint8 frame ring gather and the
// fp64 proportional-priority sum tree.
//
// Reference: /root/reference/pkg/src/deepq/replay.py
//   ReplayMemory._gather          replay.py:104-115   -> ring_gather_kernel
//   SumTree.set / find            replay.py:155-181   -> tree_* kernels
//   PrioritizedReplay.sample      replay.py:215-229   -> tree_sample_kernel
//   PrioritizedReplay.update_priorities  232-241      -> tree_update_kernel
//   PrioritizedReplay.store       replay.py:207-210   -> tree_store_kernel
//
// HBM layout: the heap keeps the reference's 1-indexed layout
// (nodes[0] unused, leaf i at nodes[2^depth + i], replay.py:141-143), fp64,
// 16 MiB at 1M leaves.  Tree arithmetic uses __dadd_rn/__dmul_rn/__ddiv_rn so
// internal nodes, query masses and sampled indices are bit-identical to the
// reference given the same uniforms.
#include "common.cuh"
#include "tree_descend.cuh"
#include "bulk_copy.cuh"

#include <math.h>

#include <mutex>

namespace dqn {
namespace {

// ------------------------------------------------------------- frame ring

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void ring_fill_hash_kernel(uint64_t *__restrict__ out, int64_t total_words,
                                      int64_t first_word, uint64_t base) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < total_words; i += stride) out[i] = splitmix64(base | (uint64_t)(first_word + i));
}

// One CTA copies a 16 KiB chunk of one sampled slot (state or next state).
// 16-byte vector loads, four in flight per thread; slot strides are
// multiples of 16 B for the Atari ring (28,224 B).
constexpr int kGatherThreads = 256;
constexpr int kGatherUnroll = 4;
constexpr int kGatherChunk = kGatherThreads * kGatherUnroll;  // int4 per CTA

__global__ void __launch_bounds__(kGatherThreads)
ring_gather_vec_kernel(const int4 *__restrict__ states, const int4 *__restrict__ next_states,
                       int64_t slot_vecs, const int64_t *__restrict__ idx,
                       int4 *__restrict__ out_s, int4 *__restrict__ out_s2,
                       const int64_t *__restrict__ actions, const double *__restrict__ rewards,
                       const uint8_t *__restrict__ terminals, int64_t *out_a, double *out_r,
                       uint8_t *out_t) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  // blockIdx.x = sample * chunks + chunk (grid.y would cap k at 65,535)
  const int64_t nchunks = (slot_vecs + kGatherChunk - 1) / kGatherChunk;
  const int64_t j = blockIdx.x / nchunks, chunk = blockIdx.x - j * nchunks;
  const int which = blockIdx.y;
  const int64_t slot = __ldg(idx + j);
  if (chunk == 0 && which == 0 && threadIdx.x == 0) {   // the sample's metadata
    if (out_a) out_a[j] = actions[slot];
    if (out_r) out_r[j] = rewards[slot];
    if (out_t) out_t[j] = terminals[slot];
  }
  const int4 *src = which ? next_states : states;
  int4 *dst = which ? out_s2 : out_s;
  if (dst == nullptr) return;
  const int4 *s = src + slot * slot_vecs;
  int4 *d = dst + j * slot_vecs;
  const int64_t base = chunk * kGatherChunk + threadIdx.x;
  int4 v[kGatherUnroll];
#pragma unroll
  for (int u = 0; u < kGatherUnroll; ++u) {
    int64_t e = base + u * kGatherThreads;
    if (e < slot_vecs) v[u] = __ldg(s + e);
  }
#pragma unroll
  for (int u = 0; u < kGatherUnroll; ++u) {
    int64_t e = base + u * kGatherThreads;
    if (e < slot_vecs) d[e] = v[u];
  }
}

// The same gather through the TMA bulk-copy engine: one CTA per (sample,
// state | next state), one thread moves the whole slot global -> shared ->
// global (cp.async.bulk); thread 1 copies the sample's metadata.
__global__ void __launch_bounds__(32)
ring_gather_tma_kernel(const uint8_t *__restrict__ states, const uint8_t *__restrict__ next_states,
                       int64_t slot_bytes, const int64_t *__restrict__ idx,
                       uint8_t *__restrict__ out_s, uint8_t *__restrict__ out_s2,
                       const int64_t *__restrict__ actions, const double *__restrict__ rewards,
                       const uint8_t *__restrict__ terminals, int64_t *out_a, double *out_r,
                       uint8_t *out_t) {
  pdl_begin();
  extern __shared__ __align__(128) uint8_t slot_buf[];
  __shared__ uint64_t bar;
  const int j = blockIdx.x, which = blockIdx.y;
  const int64_t slot = __ldg(idx + j);
  if (threadIdx.x == 0) bc_mbar_init(&bar);
  __syncthreads();
  if (threadIdx.x == 0)
    bulk_copy_via_smem(slot_buf, &bar, (which ? next_states : states) + slot * slot_bytes,
                       (which ? out_s2 : out_s) + (int64_t)j * slot_bytes, (uint32_t)slot_bytes);
  if (threadIdx.x == 1 && which == 0) {
    if (out_a) out_a[j] = actions[slot];
    if (out_r) out_r[j] = rewards[slot];
    if (out_t) out_t[j] = terminals[slot];
  }
}

__global__ void ring_gather_bytes_kernel(const uint8_t *__restrict__ states,
                                         const uint8_t *__restrict__ next_states,
                                         int64_t slot_bytes, const int64_t *__restrict__ idx,
                                         uint8_t *__restrict__ out_s, uint8_t *__restrict__ out_s2) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int64_t j = blockIdx.x;                 // one CTA per sample and frame
  const int which = blockIdx.y;
  const uint8_t *src = which ? next_states : states;
  uint8_t *dst = which ? out_s2 : out_s;
  if (dst == nullptr) return;
  const int64_t slot = idx[j];
  for (int64_t e = threadIdx.x; e < slot_bytes; e += blockDim.x)
    dst[j * slot_bytes + e] = src[slot * slot_bytes + e];
}

__global__ void ring_gather_meta_kernel(const int64_t *__restrict__ actions,
                                        const double *__restrict__ rewards,
                                        const uint8_t *__restrict__ terminals,
                                        const int64_t *__restrict__ idx, int k,
                                        int64_t *out_a, double *out_r, uint8_t *out_t) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  int64_t s = idx[j];
  if (out_a) out_a[j] = actions[s];
  if (out_r) out_r[j] = rewards[s];
  if (out_t) out_t[j] = terminals[s];
}

// ReplayMemory.store_many (replay.py:91-102) for n staged transitions: slot
// (cursor + i) % capacity <- transition i, raw bytes of each state (any ring
// dtype); the sources may be pinned host memory read in place.  CTA (i, w)
// copies state (w = 0) / next state (w = 1) of transition i; CTA (i, 0)
// also the metadata, CTA (0, 0) the new size.
__global__ void __launch_bounds__(256)
ring_store_kernel(uint8_t *__restrict__ states, uint8_t *__restrict__ next_states,
                  int64_t slot_bytes, int64_t *__restrict__ actions, double *__restrict__ rewards,
                  uint8_t *__restrict__ terminals, int64_t capacity, int64_t cursor,
                  const uint8_t *__restrict__ src_s, const uint8_t *__restrict__ src_s2,
                  const int64_t *__restrict__ src_a, const double *__restrict__ src_r,
                  const uint8_t *__restrict__ src_t, int64_t *size_dev, int64_t new_size) {
  pdl_begin();
  const int i = blockIdx.x, w = blockIdx.y;
  const int64_t slot = (cursor + i) % capacity;
  const uint8_t *src = (w ? src_s2 : src_s) + (int64_t)i * slot_bytes;
  uint8_t *dst = (w ? next_states : states) + slot * slot_bytes;
  if (slot_bytes % 16 == 0 && ((uintptr_t)src | (uintptr_t)dst) % 16 == 0) {
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
    int4 *d4 = reinterpret_cast<int4 *>(dst);
    for (int64_t e = threadIdx.x; e < slot_bytes / 16; e += blockDim.x) d4[e] = s4[e];
  } else {
    for (int64_t e = threadIdx.x; e < slot_bytes; e += blockDim.x) dst[e] = src[e];
  }
  if (w == 0 && threadIdx.x == 0) {
    actions[slot] = src_a[i];
    rewards[slot] = src_r[i];
    terminals[slot] = src_t[i] ? 1 : 0;
    if (i == 0 && size_dev) *size_dev = new_size;
  }
}

// --------------------------------------------------------------- sum tree

// tree_descend (SumTree.find descent) lives in tree_descend.cuh (shared with dp.cu)

// PrioritizedReplay.sample for k <= blockDim (one CTA): stratified masses,
// descent, probabilities, IS weights and their batch-max normalisation.
__global__ void tree_sample_kernel(const double *__restrict__ nodes, int depth,
                                   const int64_t *__restrict__ size_p,
                                   const double *__restrict__ u, int k,
                                   const double *__restrict__ beta_p, int64_t *__restrict__ idx,
                                   double *__restrict__ prob, double *__restrict__ weight,
                                   int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ double red[32];
  const int j = threadIdx.x;
  const double total = nodes[1];
  if (!(total > 0.0)) {                        // replay.py:221-222
    if (j == 0) raise_flag(flags, DQN_FLAG_ZERO_TOTAL);
    if (j < k) { idx[j] = 0; prob[j] = 0.0; weight[j] = 0.0; }
    return;
  }
  const double beta = *beta_p;
  const int64_t size = *size_p;
  const double hi = nextafter(total, 0.0);
  const double seg = __ddiv_rn(total, (double)k);                 // segment = total / k
  double w = 0.0;
  if (j < k) {
    const double q = __dmul_rn(__dadd_rn((double)j, u[j]), seg);  // (arange + u) * seg
    double leaf;
    const int64_t i = tree_descend(nodes, depth, q, hi, &leaf);
    const double p = __ddiv_rn(leaf, total);
    w = pow(__dmul_rn((double)size, p), -beta);                   // (size * P)^-beta
    idx[j] = i;
    prob[j] = p;
  }
  // block max of w (order-free, exact)
  double m = w;
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((j & 31) == 0) red[j >> 5] = m;
  __syncthreads();
  if (j < 32) {
    double v = (j < (int)((blockDim.x + 31) >> 5)) ? red[j] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (j == 0) red[0] = v;
  }
  __syncthreads();
  if (j < k) weight[j] = __ddiv_rn(w, red[0]);                    // w /= w.max()
}

// PrioritizedReplay.sample + ReplayMemory._gather in ONE launch (the
// learner's first kernel): CTA (x, j, which) for j < k descends query j
// itself (thread 0; the same arithmetic as tree_sample_kernel) and copies its
// share of state / next state j, CTA (0, j, 0) also the metadata; the extra
// CTA row y = k descends all k queries for the IS weights (batch max) and
// writes idx / prob / weight.  Results identical to tree_sample + ring_gather.
template <bool TMA>
__global__ void __launch_bounds__(kGatherThreads)
sample_gather_kernel(const double *__restrict__ nodes, int depth, const int64_t *__restrict__ size_p,
                     const double *__restrict__ u, int k, const double *__restrict__ beta_p,
                     int64_t *__restrict__ idx, double *__restrict__ prob,
                     double *__restrict__ weight, int32_t *flags, const int4 *__restrict__ states,
                     const int4 *__restrict__ next_states, int64_t slot_vecs,
                     int4 *__restrict__ out_s, int4 *__restrict__ out_s2,
                     const int64_t *__restrict__ actions, const double *__restrict__ rewards,
                     const uint8_t *__restrict__ terminals, int64_t *out_a, double *out_r,
                     uint8_t *out_t) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int j = blockIdx.y;
  const double total = nodes[1];
  const bool ok = total > 0.0;
  if (j == k) {                                   // the weights CTA
    if (blockIdx.x != 0 || blockIdx.z != 0) return;
    __shared__ double red[kGatherThreads / 32];
    sample_is_weights_block(nodes, depth, size_p, u, k, beta_p, idx, prob, weight, flags, red);
    return;
  }
  __shared__ int64_t s_slot;
  if (threadIdx.x < 32) {                         // warp 0: eight levels per round trip
    int64_t i = 0;
    if (ok)
      i = warp_tree_descend(nodes, depth,
                            __dmul_rn(__dadd_rn((double)j, u[j]), __ddiv_rn(total, (double)k)),
                            nextafter(total, 0.0));
    if (threadIdx.x == 0) s_slot = i;
    // without a weights CTA (weight == nullptr: the IS weights come from a
    // separate dqn_tree_sample launch off the critical path) the gather CTAs
    // record the sampled slots themselves
    if (weight == nullptr && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.z == 0) idx[j] = i;
  }
  __syncthreads();
  const int64_t slot = s_slot;
  const int which = blockIdx.z;
  // the transition's metadata, by another thread than the one moving the
  // frame (and after it is started): three reads in flight, then the writes
  if (threadIdx.x == 1 && blockIdx.x == 0 && blockIdx.z == 0) {
    const int64_t av = out_a ? actions[slot] : 0;
    const double rv = out_r ? rewards[slot] : 0.0;
    const uint8_t tv = out_t ? terminals[slot] : 0;
    if (out_a) out_a[j] = av;
    if (out_r) out_r[j] = rv;
    if (out_t) out_t[j] = tv;
  }
  if constexpr (TMA) {             // one CTA per frame: the TMA engine moves the slot
    extern __shared__ __align__(128) uint8_t slot_buf[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
      bc_mbar_init(&bar);
      const int64_t bytes = slot_vecs * 16;
      bulk_copy_via_smem(slot_buf, &bar,
                         reinterpret_cast<const uint8_t *>(which ? next_states : states) + slot * bytes,
                         reinterpret_cast<uint8_t *>(which ? out_s2 : out_s) + (int64_t)j * bytes,
                         (uint32_t)bytes);
    }
    return;
  }
  const int4 *s = (which ? next_states : states) + slot * slot_vecs;
  int4 *d = (which ? out_s2 : out_s) + (int64_t)j * slot_vecs;
  const int64_t base = (int64_t)blockIdx.x * kGatherChunk + threadIdx.x;
  int4 v[kGatherUnroll];
#pragma unroll
  for (int uu = 0; uu < kGatherUnroll; ++uu) {
    const int64_t e = base + uu * kGatherThreads;
    if (e < slot_vecs) v[uu] = __ldg(s + e);
  }
#pragma unroll
  for (int uu = 0; uu < kGatherUnroll; ++uu) {
    const int64_t e = base + uu * kGatherThreads;
    if (e < slot_vecs) d[e] = v[uu];
  }
}

// Large-k sampler (SURVEY §8(d) microbenchmark; the learner's k <= 1024 use
// tree_sample_kernel / the fused sample+gather): a persistent grid whose CTAs
// stage the top kTopLevels levels of the heap (nodes [0, 2^top): 64 KB) in
// shared memory once, then descend their queries -- the first top - 1
// levels from shared memory, the remaining levels from global memory four
// per dependent round trip (tree_descend_from).  Same compare / subtract
// sequence as the reference's loop (replay.py:172-181): identical indices.
// Consecutive threads take consecutive strata, so a warp's queries share
// their upper path and land on neighbouring leaves.
// Pass 1 also reduces the raw IS weights to a per-CTA max; the last CTA to
// finish (ticket) reduces those to the batch max for pass 2.
constexpr int kTopLevels = 13;
constexpr int kSampleThreads = 512;

__global__ void __launch_bounds__(kSampleThreads)
tree_sample_raw_kernel(const double *nodes, int depth, const int64_t *size_p, const double *u,
                       int k, const double *beta_p, int64_t *__restrict__ idx,
                       double *__restrict__ prob, double *__restrict__ weight,
                       double *block_max, double *gmax, unsigned int *ticket, int32_t *flags) {
  // no __restrict__ on the inputs: their loads must stay below the PDL wait
  extern __shared__ double s_top[];
  __shared__ double red[kSampleThreads / 32];
  __shared__ bool s_last;
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int top = depth < kTopLevels ? depth : kTopLevels;
  for (int i = threadIdx.x; i < (1 << top); i += blockDim.x) s_top[i] = nodes[i];
  __syncthreads();
  const double total = s_top[1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double m = 0.0;
  if (!(total > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(flags, DQN_FLAG_ZERO_TOTAL);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += stride) {
      idx[j] = 0; prob[j] = 0.0; weight[j] = 0.0;
    }
    m = 1.0;
  } else {
    const double beta = *beta_p;
    const double size = (double)*size_p;
    const double seg = __ddiv_rn(total, (double)k), hi = nextafter(total, 0.0);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += stride) {
      double q = fmin(fmax(__dmul_rn(__dadd_rn((double)j, u[j]), seg), 1e-300), hi);
      int64_t n = 1;
      int l = 0;
      for (; l < top - 1; ++l) {                    // children of level l sit below 2^top
        const double ls = s_top[2 * n];
        const bool right = q > ls;
        if (right) q = __dsub_rn(q, ls);            // q -= left_sum * go_right
        n = 2 * n + (right ? 1 : 0);
      }
      double leaf;
      const int64_t i = tree_descend_from(nodes, depth, n, l, q, &leaf);
      const double p = __ddiv_rn(leaf, total);
      const double w = pow(__dmul_rn(size, p), -beta);
      idx[j] = i;
      prob[j] = p;
      weight[j] = w;
      m = fmax(m, w);
    }
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = fmax(v, red[i]);
    block_max[blockIdx.x] = v;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v = fmax(v, __ldcg(block_max + b));
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
    *gmax = mx;
    *ticket = 0;                                    // graph-replay safe
  }
}

__global__ void tree_sample_norm_kernel(double *__restrict__ weight, int k, const double *gmax) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const double mx = *gmax;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    weight[j] = __ddiv_rn(weight[j], mx);
}

__global__ void tree_find_kernel(const double *__restrict__ nodes, int depth,
                                 const double *__restrict__ q, int64_t n, int64_t *__restrict__ idx,
                                 int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const double total = nodes[1];
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (!(total > 0.0)) {
    if (j == 0) raise_flag(flags, DQN_FLAG_ZERO_TOTAL);
    return;
  }
  const double hi = nextafter(total, 0.0);
  for (; j < n; j += (int64_t)gridDim.x * blockDim.x) idx[j] = tree_descend(nodes, depth, q[j], hi);
}

constexpr int kTreeThreads = 1024;

// Recompute the ancestors of the leaves in leaf_ids[0..n) level by level.
// Each internal node is a pure function of its two children, so duplicate
// writers store identical bits and the result equals the reference's
// sequential set() calls.
__device__ void tree_fix_ancestors(double *nodes, int depth, const int64_t *leaf_node, int n) {
  for (int l = 1; l <= depth; ++l) {
    __syncthreads();
    if ((int)threadIdx.x < n) {
      const int64_t a = leaf_node[threadIdx.x] >> l;
      nodes[a] = __dadd_rn(nodes[2 * a], nodes[2 * a + 1]);
    }
  }
  __syncthreads();
}

// update_priorities (replay.py:232-241) and set (155-165).  mode 0: leaf
// value = (|td| + eps)^alpha; mode 1: leaf value = td (raw SumTree.set).
// One CTA walks the batch in chunks of 1024 in batch order.
__global__ void __launch_bounds__(kTreeThreads)
tree_update_kernel(double *__restrict__ nodes, int depth, const int64_t *__restrict__ limit_p,
                   int64_t limit_v,
                   const int64_t *__restrict__ idx, const double *__restrict__ td, int k,
                   double alpha, double eps, double *__restrict__ max_p, int32_t *flags,
                   int mode) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ int64_t s_node[kTreeThreads];
  __shared__ int s_first_bad;
  __shared__ double s_red[32];
  const int t = threadIdx.x;
  const int64_t limit = limit_p ? *limit_p : limit_v;
  // the reference raises before update_priorities when the step already
  // failed (empty/zero-mass sample, non-finite network output)
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) return;
  if (t == 0) s_first_bad = k;
  __syncthreads();
  // first invalid position in batch order (index range, then value)
  for (int j = t; j < k; j += blockDim.x) {
    const int64_t i = idx[j];
    bool bad = (i < 0 || i >= limit);
    if (!bad) {
      double v = (mode == 0) ? __dadd_rn(fabs(td[j]), eps) : td[j];
      if (mode == 0) v = pow(v, alpha);
      bad = !(v >= 0.0) || isinf(v);
    }
    if (bad) atomicMin(&s_first_bad, j);
  }
  __syncthreads();
  const int kk = s_first_bad;
  const int64_t base = int64_t(1) << depth;
  for (int c0 = 0; c0 < kk; c0 += blockDim.x) {
    const int n = min((int)blockDim.x, kk - c0);
    const int j = c0 + t;
    if (t < n) s_node[t] = base + idx[j];
    __syncthreads();
    if (t < n) {
      // last write wins inside the chunk; later chunks run after this one
      bool last = true;
      for (int o = t + 1; o < n; ++o)
        if (s_node[o] == s_node[t]) { last = false; break; }
      if (last) {
        double v = (mode == 0) ? pow(__dadd_rn(fabs(td[j]), eps), alpha) : td[j];
        nodes[s_node[t]] = v;
      }
    }
    tree_fix_ancestors(nodes, depth, s_node, n);
  }
  if (kk < k) {
    if (t == 0)
      raise_flag(flags, (idx[kk] < 0 || idx[kk] >= limit) ? DQN_FLAG_INDEX : DQN_FLAG_BAD_PRIORITY);
    return;                                   // reference raises: max_p untouched
  }
  if (mode == 0 && max_p != nullptr) {
    double m = -INFINITY;
    for (int j = t; j < k; j += blockDim.x) m = fmax(m, __dadd_rn(fabs(td[j]), eps));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((t & 31) == 0) s_red[t >> 5] = m;
    __syncthreads();
    if (t == 0) {
      double v = s_red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, s_red[w]);
      const double cur = *max_p;
      if (v > cur) *max_p = v;                // max(self.max_priority, p.max())
    }
  }
}

// update_priorities for learner-sized batches (k <= kSmallK): the same
// result as tree_update_kernel without a global-memory round trip per level.
// A node touched this step is (left + right) of children that are either
// touched too (their new value is published in shared memory) or untouched
// (their old value can be loaded up front, all levels in parallel).
constexpr int kSmallK = 256;
constexpr int kMaxDepth = 32;

__global__ void __launch_bounds__(kSmallK)
tree_update_small_kernel(double *__restrict__ nodes, int depth, const int64_t *__restrict__ limit_p,
                         const int64_t *__restrict__ idx, const double *__restrict__ td, int k,
                         double alpha, double eps, double *__restrict__ max_p, int32_t *flags,
                         const int32_t *__restrict__ k_dev) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  if (k_dev) k = min(k, *k_dev);               // device-side batch length (data-parallel owners)
  __shared__ int64_t s_node[kSmallK];
  __shared__ double s_val[kSmallK];
  __shared__ int s_first_bad;
  __shared__ double s_red[kSmallK / 32];
  const int t = threadIdx.x;
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) return;
  const int64_t limit = *limit_p;
  if (t == 0) s_first_bad = k;
  __syncthreads();
  int64_t leaf = 0;
  double v = 0.0, p = -INFINITY;
  if (t < k) {
    leaf = idx[t];
    p = __dadd_rn(fabs(td[t]), eps);                    // |td| + eps
    bool bad = leaf < 0 || leaf >= limit;
    if (!bad) {
      v = pow(p, alpha);                                 // raw ** alpha
      bad = !(v >= 0.0) || isinf(v);
    }
    if (bad) atomicMin(&s_first_bad, t);
  }
  __syncthreads();
  const int kk = s_first_bad;
  const int64_t node = (int64_t(1) << depth) + leaf;
  s_node[t] = t < kk ? node : -1;
  __syncthreads();
  bool act = t < kk;
  for (int o = t + 1; act && o < kk; ++o)                // last write wins
    if (s_node[o] == node) act = false;
  double sib[kMaxDepth];
#pragma unroll
  for (int l = 0; l < kMaxDepth; ++l)
    if (l < depth) sib[l] = act ? nodes[(node >> l) ^ 1] : 0.0;
  if (act) nodes[node] = v;
  double cur = v;
#pragma unroll
  for (int l = 0; l < kMaxDepth; ++l) {
    if (l >= depth) break;
    __syncthreads();
    s_node[t] = act ? (node >> l) : -1;
    s_val[t] = cur;
    __syncthreads();
    if (act) {
      const int64_t me = node >> l, other = me ^ 1;
      double sv = sib[l];
      for (int o = 0; o < kk; ++o)
        if (s_node[o] == other) sv = s_val[o];
      cur = (me & 1) ? __dadd_rn(sv, cur) : __dadd_rn(cur, sv);   // left + right
      nodes[me >> 1] = cur;
    }
  }
  if (kk < k) {
    if (t == kk)
      raise_flag(flags, (leaf < 0 || leaf >= limit) ? DQN_FLAG_INDEX : DQN_FLAG_BAD_PRIORITY);
    return;
  }
  if (max_p != nullptr) {
    double m = p;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((t & 31) == 0) s_red[t >> 5] = m;
    __syncthreads();
    if (t == 0) {
      double mx = s_red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, s_red[w]);
      if (mx > *max_p) *max_p = mx;
    }
  }
}

// update_priorities for k <= 32 (the learner's batch): one warp, no shared
// memory or barriers.  Lanes whose paths meet are found with
// __match_any_sync; a node's untouched child comes from the up-front sibling
// loads, a touched one from the lane that owns it (__shfl_sync).
__global__ void __launch_bounds__(32)
tree_update_warp_kernel(double *__restrict__ nodes, int depth, const int64_t *__restrict__ limit_p,
                        const int64_t *__restrict__ idx, const double *__restrict__ td, int k,
                        double alpha, double eps, double *__restrict__ max_p, int32_t *flags,
                        const int32_t *__restrict__ k_dev) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  if (k_dev) k = min(k, *k_dev);               // device-side batch length (data-parallel owners)
  constexpr unsigned FULL = 0xffffffffu;
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) return;
  const int t = threadIdx.x;
  const int64_t limit = *limit_p;
  int64_t leaf = 0;
  double v = 0.0, p = -INFINITY;
  bool bad = false;
  if (t < k) {
    leaf = idx[t];
    p = __dadd_rn(fabs(td[t]), eps);                     // |td| + eps
    bad = leaf < 0 || leaf >= limit;
    if (!bad) {
      v = pow(p, alpha);                                  // raw ** alpha
      bad = !(v >= 0.0) || isinf(v);
    }
  }
  const unsigned badmask = __ballot_sync(FULL, bad);
  const int kk = badmask ? __ffs(badmask) - 1 : k;       // first failing position
  const bool valid = t < kk;
  const int64_t node = (int64_t(1) << depth) + leaf;
  const long long uniq = -1 - (long long)t;               // never equal to a node id
  const unsigned same_leaf = __match_any_sync(FULL, valid ? (long long)node : uniq);
  const bool act = valid && (31 - __clz(same_leaf)) == t;  // last write wins
  double sib[kMaxDepth];
#pragma unroll
  for (int l = 0; l < kMaxDepth; ++l)
    if (l < depth) sib[l] = act ? nodes[(node >> l) ^ 1] : 0.0;
  if (act) nodes[node] = v;
  double cur = v;
#pragma unroll
  for (int l = 0; l < kMaxDepth; ++l) {
    if (l >= depth) break;
    const int64_t me = node >> l;
    const unsigned fam = __match_any_sync(FULL, act ? (long long)(me >> 1) : uniq);
    const unsigned self = __match_any_sync(FULL, act ? (long long)me : uniq);
    const unsigned other = fam & ~self;                   // lanes holding the sibling
    const double shared = __shfl_sync(FULL, cur, other ? __ffs(other) - 1 : t);
    const double sv = other ? shared : sib[l];
    cur = (me & 1) ? __dadd_rn(sv, cur) : __dadd_rn(cur, sv);   // left + right
    if (act) nodes[me >> 1] = cur;
  }
  if (kk < k) {
    if (t == kk)
      raise_flag(flags, (leaf < 0 || leaf >= limit) ? DQN_FLAG_INDEX : DQN_FLAG_BAD_PRIORITY);
    return;
  }
  if (max_p != nullptr) {
    double m = p;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    if (t == 0 && m > *max_p) *max_p = m;
  }
}

// store (replay.py:207-210): n consecutive slots get max_p^alpha.
__global__ void __launch_bounds__(kTreeThreads)
tree_store_kernel(double *__restrict__ nodes, int depth, int64_t capacity, int64_t slot,
                  int64_t n, const double *__restrict__ max_p, double alpha) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ int64_t s_node[kTreeThreads];
  const int t = threadIdx.x;
  const double v = pow(*max_p, alpha);
  const int64_t base = int64_t(1) << depth;
  const int64_t m = n < capacity ? n : capacity;   // later wraps overwrite the same slot value
  for (int64_t c0 = 0; c0 < m; c0 += blockDim.x) {
    const int cn = (int)min((int64_t)blockDim.x, m - c0);
    if (t < cn) {
      s_node[t] = base + (slot + c0 + t) % capacity;
      nodes[s_node[t]] = v;
    }
    tree_fix_ancestors(nodes, depth, s_node, cn);
  }
}

__global__ void tree_level_kernel(double *__restrict__ nodes, int64_t lo, int64_t hi) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  for (int64_t a = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < hi;
       a += (int64_t)gridDim.x * blockDim.x)
    nodes[a] = __dadd_rn(nodes[2 * a], nodes[2 * a + 1]);
}

// ---- bulk priority update (k >= kBulkK): many CTAs, bit-exact with the
// sequential reference.  The reference recomputes every ancestor as the sum
// of its current children, so the final tree equals: final leaf values (last
// write in batch order wins) + every internal level rebuilt bottom-up.
constexpr int kBulkK = 4096;

__device__ __forceinline__ bool bulk_value(const int64_t *idx, const double *td, int j,
                                           int64_t limit, double alpha, double eps, double &v) {
  const int64_t i = idx[j];
  if (i < 0 || i >= limit) return false;
  v = pow(__dadd_rn(fabs(td[j]), eps), alpha);
  return v >= 0.0 && !isinf(v);
}

// first invalid position in batch order (index range, then value)
__global__ void tree_bulk_check_kernel(const int64_t *__restrict__ idx, const double *__restrict__ td,
                                       int k, const int64_t *__restrict__ limit_p, double alpha,
                                       double eps, int *__restrict__ first_bad,
                                       const int32_t *__restrict__ flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int64_t limit = *limit_p;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    double v;
    if (!bulk_value(idx, td, j, limit, alpha, eps, v)) atomicMin(first_bad, j);
  }
}

// winner[leaf] = last batch position writing it (positions before first_bad)
__global__ void tree_bulk_winner_kernel(const int64_t *__restrict__ idx, int k,
                                        const int *__restrict__ first_bad, int *__restrict__ winner,
                                        const int32_t *__restrict__ flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) return;
  const int kk = min(*first_bad, k);           // INT_MAX at rest: no invalid position
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < kk; j += gridDim.x * blockDim.x)
    atomicMax(winner + idx[j], j);
}

// the winning position writes its leaf and clears the winner slot
__global__ void tree_bulk_scatter_kernel(double *__restrict__ nodes, int depth,
                                         const int64_t *__restrict__ idx,
                                         const double *__restrict__ td, int k, double alpha,
                                         double eps, const int *__restrict__ first_bad,
                                         int *__restrict__ winner,
                                         const int32_t *__restrict__ flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) return;
  const int kk = min(*first_bad, k);
  const int64_t base = int64_t(1) << depth;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < kk; j += gridDim.x * blockDim.x) {
    const int64_t i = idx[j];
    if (winner[i] == j) {
      nodes[base + i] = pow(__dadd_rn(fabs(td[j]), eps), alpha);
      winner[i] = -1;
    }
  }
}

// flags (first invalid position) or max_priority = max(max_priority, max |td| + eps)
__global__ void tree_bulk_finish_kernel(const int64_t *__restrict__ idx,
                                        const double *__restrict__ td, int k,
                                        const int64_t *__restrict__ limit_p, double eps,
                                        int *__restrict__ first_bad, double *__restrict__ max_p,
                                        int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ double red[32];
  if (flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT))) {
    if (threadIdx.x == 0) *first_bad = 0x7fffffff;
    return;
  }
  const int kk = *first_bad;
  const int t = threadIdx.x;
  if (kk < k) {
    if (t == 0) {
      const int64_t i = idx[kk];
      raise_flag(flags, (i < 0 || i >= *limit_p) ? DQN_FLAG_INDEX : DQN_FLAG_BAD_PRIORITY);
      *first_bad = 0x7fffffff;               // reset for the next call
    }
    return;                                   // reference raises: max_p untouched
  }
  double m = -INFINITY;
  for (int j = t; j < k; j += blockDim.x) m = fmax(m, __dadd_rn(fabs(td[j]), eps));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((t & 31) == 0) red[t >> 5] = m;
  __syncthreads();
  if (t == 0) {
    double v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    if (max_p && v > *max_p) *max_p = v;       // max(self.max_priority, p.max())
    *first_bad = 0x7fffffff;
  }
}

inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace
}  // namespace dqn

using namespace dqn;

extern "C" int dqn_ring_store(void *stream, uint8_t *states, uint8_t *next_states,
                              int64_t slot_bytes, int64_t *actions, double *rewards,
                              uint8_t *terminals, int64_t capacity, int64_t cursor, int32_t n,
                              const uint8_t *src_states, const uint8_t *src_next_states,
                              const int64_t *src_actions, const double *src_rewards,
                              const uint8_t *src_terminals, int64_t *size_dev,
                              int64_t new_size) {
  DQN_CHECK_ARG(states && next_states && actions && rewards && terminals && slot_bytes > 0 &&
                    capacity >= 1 && cursor >= 0 && cursor < capacity && n >= 0 &&
                    n <= capacity && (n == 0 || (src_states && src_next_states && src_actions &&
                                                  src_rewards && src_terminals)),
                "ring_store: bad args");
  if (n == 0) return DQN_OK;
  launch_k(ring_store_kernel, dim3((unsigned)n, 2), 256, 0, as_stream(stream), states,
           next_states, slot_bytes, actions, rewards, terminals, capacity, cursor, src_states,
           src_next_states, src_actions, src_rewards, src_terminals, size_dev, new_size);
  DQN_LAUNCH_CHECK("ring_store");
  return DQN_OK;
}


extern "C" int dqn_ring_fill_hash(void *stream, uint8_t *frames, int64_t slot0, int64_t nslots,
                                  int64_t slot_bytes, uint64_t counter_base) {
  DQN_CHECK_ARG(frames && slot_bytes % 8 == 0 && nslots >= 0, "ring_fill_hash: bad args");
  const int64_t words = slot_bytes / 8;
  const int64_t total = nslots * words;
  if (total == 0) return DQN_OK;
  launch_k(ring_fill_hash_kernel, grid_for(total, 256, 148 * 64), 256, 0, as_stream(stream), 
      reinterpret_cast<uint64_t *>(frames + slot0 * slot_bytes), total, slot0 * words,
      counter_base);
  DQN_LAUNCH_CHECK("ring_fill_hash");
  return DQN_OK;
}

extern "C" int dqn_ring_gather(void *stream, const uint8_t *states, const uint8_t *next_states,
                               int64_t slot_bytes, const int64_t *actions, const double *rewards,
                               const uint8_t *terminals, const int64_t *idx, int32_t k,
                               uint8_t *out_states, uint8_t *out_next_states,
                               int64_t *out_actions, double *out_rewards,
                               uint8_t *out_terminals) {
  DQN_CHECK_ARG(idx && k >= 0 && slot_bytes > 0, "ring_gather: bad args");
  if (k == 0) return DQN_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = (out_states || out_next_states) && slot_bytes % 16 == 0 &&
                   ((uintptr_t)states % 16 == 0) && ((uintptr_t)next_states % 16 == 0) &&
                   ((uintptr_t)out_states % 16 == 0) && ((uintptr_t)out_next_states % 16 == 0);
  if (vec && out_states && out_next_states && slot_bytes <= 48 * 1024 && tma_gather_enabled()) {
    launch_k(ring_gather_tma_kernel, dim3((unsigned)k, 2), 32, (size_t)slot_bytes, st, states,
             next_states, slot_bytes, idx, out_states, out_next_states, actions, rewards,
             terminals, out_actions, out_rewards, out_terminals);
    DQN_LAUNCH_CHECK("ring_gather_tma");
    return DQN_OK;
  }
  if (vec) {   // frames + metadata in one launch
    const int64_t vecs = slot_bytes / 16;
    dim3 grid((unsigned)((vecs + kGatherChunk - 1) / kGatherChunk * k), 2);
    launch_k(ring_gather_vec_kernel, grid, kGatherThreads, 0, st, 
        reinterpret_cast<const int4 *>(states), reinterpret_cast<const int4 *>(next_states), vecs,
        idx, reinterpret_cast<int4 *>(out_states), reinterpret_cast<int4 *>(out_next_states),
        actions, rewards, terminals, out_actions, out_rewards, out_terminals);
    DQN_LAUNCH_CHECK("ring_gather");
    return DQN_OK;
  }
  if (out_states || out_next_states) {
    {
      dim3 grid((unsigned)k, 2);
      launch_k(ring_gather_bytes_kernel, grid, 256, 0, st, states, next_states, slot_bytes, idx,
                                                     out_states, out_next_states);
    }
    DQN_LAUNCH_CHECK("ring_gather");
  }
  if (out_actions || out_rewards || out_terminals) {
    launch_k(ring_gather_meta_kernel, (k + 255) / 256, 256, 0, st, actions, rewards, terminals, idx, k,
                                                            out_actions, out_rewards,
                                                            out_terminals);
    DQN_LAUNCH_CHECK("ring_gather_meta");
  }
  return DQN_OK;
}

extern "C" int dqn_tree_sample(void *stream, const double *nodes, int32_t depth, const int64_t *size,
                               const double *u, int32_t k, const double *beta, int64_t *idx,
                               double *prob, double *weight, int32_t *flags) {
  DQN_CHECK_ARG(nodes && size && u && beta && idx && prob && weight && k >= 1 && depth >= 1 &&
                    depth < 40,
                "tree_sample: bad args");
  cudaStream_t st = as_stream(stream);
  if (k <= 1024) {
    int threads = ((k + 31) / 32) * 32;
    launch_k(tree_sample_kernel, 1, threads, 0, st, nodes, depth, size, u, k, beta, idx, prob, weight,
                                              flags);
    DQN_LAUNCH_CHECK("tree_sample");
    return DQN_OK;
  }
  // Large batches (sampler microbenchmarks; the learner uses k <= 1024): the
  // normaliser needs a grid-wide max, so two passes; the per-CTA maxima, the
  // batch max and the pass-1 ticket live in a process-wide scratch allocated
  // (zeroed) outside any graph capture.
  static std::mutex mu;
  static double *scratch = nullptr;
  const int top = depth < kTopLevels ? depth : kTopLevels;
  const int smem = (int)sizeof(double) << top;
  const int blocks = 2 * kNumSMs;                   // persistent: 2 CTAs of 512 per SM
  std::lock_guard<std::mutex> lock(mu);
  if (!scratch) {
    int st_ = cuda_status(cudaMalloc(&scratch, sizeof(double) * (blocks + 2)), "tree_sample scratch");
    if (st_) return st_;
    st_ = cuda_status(cudaMemset(scratch, 0, sizeof(double) * (blocks + 2)), "tree_sample scratch");
    if (st_) return st_;
    st_ = cuda_status(cudaFuncSetAttribute(tree_sample_raw_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(double) << kTopLevels),
                      "tree_sample smem");
    if (st_) return st_;
  }
  double *gmax = scratch + blocks;
  unsigned int *ticket = reinterpret_cast<unsigned int *>(scratch + blocks + 1);
  launch_k(tree_sample_raw_kernel, blocks, kSampleThreads, (size_t)smem, st, nodes, depth, size, u, k,
           beta, idx, prob, weight, scratch, gmax, ticket, flags);
  DQN_LAUNCH_CHECK("tree_sample_raw");
  launch_k(tree_sample_norm_kernel, grid_for(k, 256), 256, 0, st, weight, k, (const double *)gmax);
  DQN_LAUNCH_CHECK("tree_sample_norm");
  return DQN_OK;
}

extern "C" int dqn_sample_gather(void *stream, const double *nodes, int32_t depth,
                                 const int64_t *size, const double *u, int32_t k,
                                 const double *beta, int64_t *idx, double *prob, double *weight,
                                 int32_t *flags, const uint8_t *states,
                                 const uint8_t *next_states, int64_t slot_bytes,
                                 const int64_t *actions, const double *rewards,
                                 const uint8_t *terminals, uint8_t *out_states,
                                 uint8_t *out_next_states, int64_t *out_actions,
                                 double *out_rewards, uint8_t *out_terminals) {
  DQN_CHECK_ARG(nodes && size && u && beta && idx && (prob == nullptr) == (weight == nullptr) &&
                    k >= 1 && depth >= 1 &&
                    depth < 40 && states && next_states && out_states && out_next_states &&
                    slot_bytes > 0 && slot_bytes % 16 == 0 && (uintptr_t)states % 16 == 0 &&
                    (uintptr_t)next_states % 16 == 0 && (uintptr_t)out_states % 16 == 0 &&
                    (uintptr_t)out_next_states % 16 == 0 && k < 65535,
                "sample_gather: bad args (16-byte aligned frames)");
  const int64_t vecs = slot_bytes / 16;
  const unsigned rows = (unsigned)k + (weight ? 1u : 0u);   // + the weights CTA row
  if (slot_bytes <= 48 * 1024 && tma_gather_enabled()) {
    launch_k(sample_gather_kernel<true>, dim3(1, rows, 2), 32, (size_t)slot_bytes,
             as_stream(stream), nodes, depth, size, u, k, beta, idx, prob, weight, flags,
             reinterpret_cast<const int4 *>(states), reinterpret_cast<const int4 *>(next_states),
             vecs, reinterpret_cast<int4 *>(out_states), reinterpret_cast<int4 *>(out_next_states),
             actions, rewards, terminals, out_actions, out_rewards, out_terminals);
    DQN_LAUNCH_CHECK("sample_gather_tma");
    return DQN_OK;
  }
  dim3 grid((unsigned)((vecs + kGatherChunk - 1) / kGatherChunk), rows, 2);
  launch_k(sample_gather_kernel<false>, grid, kGatherThreads, 0, as_stream(stream), nodes, depth, size,
           u, k, beta, idx, prob, weight, flags, reinterpret_cast<const int4 *>(states),
           reinterpret_cast<const int4 *>(next_states), vecs,
           reinterpret_cast<int4 *>(out_states), reinterpret_cast<int4 *>(out_next_states),
           actions, rewards, terminals, out_actions, out_rewards, out_terminals);
  DQN_LAUNCH_CHECK("sample_gather");
  return DQN_OK;
}

extern "C" int dqn_tree_find(void *stream, const double *nodes, int32_t depth,
                             const double *queries, int64_t n, int64_t *idx, int32_t *flags) {
  DQN_CHECK_ARG(nodes && queries && idx && n >= 0 && depth >= 1, "tree_find: bad args");
  if (n == 0) return DQN_OK;
  launch_k(tree_find_kernel, grid_for(n, 256), 256, 0, as_stream(stream), nodes, depth, queries, n, idx,
                                                                     flags);
  DQN_LAUNCH_CHECK("tree_find");
  return DQN_OK;
}

extern "C" int dqn_tree_update(void *stream, double *nodes, int32_t depth, const int64_t *size,
                               const int64_t *idx, const double *td, int32_t k, double alpha,
                               double eps, double *max_p, int32_t *flags) {
  DQN_CHECK_ARG(nodes && size && idx && td && k >= 0 && depth >= 1, "tree_update: bad args");
  if (k == 0) return DQN_OK;
  if (k <= 32 && depth <= kMaxDepth) {
    launch_k(tree_update_warp_kernel, 1, 32, 0, as_stream(stream), nodes, depth, size, idx, td, k, alpha,
                                                             eps, max_p, flags, (const int32_t *)nullptr);
    DQN_LAUNCH_CHECK("tree_update_warp");
    return DQN_OK;
  }
  if (k <= kSmallK && depth <= kMaxDepth) {
    launch_k(tree_update_small_kernel, 1, ((k + 31) / 32) * 32, 0, as_stream(stream), 
        nodes, depth, size, idx, td, k, alpha, eps, max_p, flags, (const int32_t *)nullptr);
    DQN_LAUNCH_CHECK("tree_update_small");
    return DQN_OK;
  }
  // bulk path: process-wide scratch (first_bad + a winner slot per leaf,
  // allocated outside graph capture and kept at rest: first_bad = INT_MAX,
  // winner = -1)
  static int *bulk = nullptr;
  static int64_t bulk_leaves = 0;
  cudaStream_t st = as_stream(stream);
  const int64_t leaves = int64_t(1) << depth;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (k >= kBulkK && (bulk_leaves >= leaves || cap == cudaStreamCaptureStatusNone)) {
    if (bulk_leaves < leaves) {
      if (bulk) cudaFree(bulk);
      int stc = cuda_status(cudaMalloc(&bulk, sizeof(int) * (leaves + 1)), "tree_update scratch");
      if (stc) { bulk = nullptr; bulk_leaves = 0; return stc; }
      cudaMemsetAsync(bulk + 1, 0xFF, sizeof(int) * leaves, st);       // winner = -1
      const int big = 0x7fffffff;
      cudaMemcpyAsync(bulk, &big, sizeof(int), cudaMemcpyHostToDevice, st);
      cudaStreamSynchronize(st);
      bulk_leaves = leaves;
    }
    int *first_bad = bulk, *winner = bulk + 1;
    const int g = grid_for(k, 256);
    launch_k(tree_bulk_check_kernel, g, 256, 0, st, idx, td, k, size, alpha, eps, first_bad,
             (const int32_t *)flags);
    DQN_LAUNCH_CHECK("tree_update_bulk_check");
    launch_k(tree_bulk_winner_kernel, g, 256, 0, st, idx, k, first_bad, winner,
             (const int32_t *)flags);
    DQN_LAUNCH_CHECK("tree_update_bulk_winner");
    launch_k(tree_bulk_scatter_kernel, g, 256, 0, st, nodes, depth, idx, td, k, alpha, eps,
             first_bad, winner, (const int32_t *)flags);
    DQN_LAUNCH_CHECK("tree_update_bulk_scatter");
    for (int l = depth - 1; l >= 0; --l) {
      const int64_t lo = int64_t(1) << l, hi = int64_t(1) << (l + 1);
      launch_k(tree_level_kernel, grid_for(hi - lo, 256), 256, 0, st, nodes, lo, hi);
      DQN_LAUNCH_CHECK("tree_update_bulk_level");
    }
    launch_k(tree_bulk_finish_kernel, 1, 1024, 0, st, idx, td, k, size, eps, first_bad, max_p,
             flags);
    DQN_LAUNCH_CHECK("tree_update_bulk_finish");
    return DQN_OK;
  }
  launch_k(tree_update_kernel, 1, kTreeThreads, 0, as_stream(stream), nodes, depth, size, 0, idx, td, k,
                                                                alpha, eps, max_p, flags, 0);
  DQN_LAUNCH_CHECK("tree_update");
  return DQN_OK;
}

extern "C" int dqn_tree_update_n(void *stream, double *nodes, int32_t depth, const int64_t *size,
                                 const int64_t *idx, const double *td, int32_t k_max,
                                 const int32_t *k_dev, double alpha, double eps, double *max_p,
                                 int32_t *flags) {
  DQN_CHECK_ARG(nodes && size && idx && td && k_dev && k_max >= 0 && k_max <= kSmallK &&
                    depth >= 1 && depth <= kMaxDepth,
                "tree_update_n: bad args (k_max <= 256)");
  if (k_max == 0) return DQN_OK;
  cudaStream_t st = as_stream(stream);
  if (k_max <= 32)
    launch_k(tree_update_warp_kernel, 1, 32, 0, st, nodes, depth, size, idx, td, k_max, alpha, eps,
             max_p, flags, k_dev);
  else
    launch_k(tree_update_small_kernel, 1, ((k_max + 31) / 32) * 32, 0, st, nodes, depth, size, idx,
             td, k_max, alpha, eps, max_p, flags, k_dev);
  DQN_LAUNCH_CHECK("tree_update_n");
  return DQN_OK;
}

extern "C" int dqn_tree_set(void *stream, double *nodes, int32_t depth, int64_t capacity,
                            const int64_t *idx, const double *values, int32_t k, int32_t *flags) {
  DQN_CHECK_ARG(nodes && idx && values && k >= 0 && depth >= 1, "tree_set: bad args");
  if (k == 0) return DQN_OK;
  launch_k(tree_update_kernel, 1, kTreeThreads, 0, as_stream(stream), nodes, depth, nullptr, capacity, idx,
                                                                values, k, 0.0, 0.0, nullptr,
                                                                flags, 1);
  DQN_LAUNCH_CHECK("tree_set");
  return DQN_OK;
}

extern "C" int dqn_tree_store(void *stream, double *nodes, int32_t depth, int64_t capacity,
                              int64_t slot, int64_t n, const double *max_p, double alpha) {
  DQN_CHECK_ARG(nodes && max_p && capacity >= 1 && slot >= 0 && slot < capacity && n >= 0,
                "tree_store: bad args");
  if (n == 0) return DQN_OK;
  launch_k(tree_store_kernel, 1, kTreeThreads, 0, as_stream(stream), nodes, depth, capacity, slot, n,
                                                               max_p, alpha);
  DQN_LAUNCH_CHECK("tree_store");
  return DQN_OK;
}

extern "C" int dqn_tree_rebuild(void *stream, double *nodes, int32_t depth) {
  DQN_CHECK_ARG(nodes && depth >= 1 && depth < 40, "tree_rebuild: bad args");
  for (int l = depth - 1; l >= 0; --l) {
    const int64_t lo = int64_t(1) << l, hi = int64_t(1) << (l + 1);
    launch_k(tree_level_kernel, grid_for(hi - lo, 256), 256, 0, as_stream(stream), nodes, lo, hi);
    DQN_LAUNCH_CHECK("tree_rebuild");
  }
  return DQN_OK;
}
