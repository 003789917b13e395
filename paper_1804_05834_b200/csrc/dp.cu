// Data-parallel prioritized-replay learner, device side (SURVEY.md §8(e),
// BASELINE cfg5; the algorithm and its host restatement are in dp.py).
//
// N ranks, one per GPU; rank r owns replay shard r (global transition g at
// rank g % N, slot g / N) with its own fp64 sum tree.  Per global update of
// K = k * N strata, every step below is a fixed-size device kernel or NCCL
// collective, so the whole update is one CUDA graph per rank:
//
//   dqn_dp_shard_info   [total, size, max_p] of this shard      -> all_gather (N x 3)
//   dqn_dp_route        T = sum of totals in rank order, prefix masses,
//                       q_j = clip((j + u_j) * T / K), owner_j, local mass
//   dqn_dp_descend      owners descend their own queries      -> (idx, leaf) table,
//                       zero elsewhere                         -> all_reduce SUM
//   dqn_dp_weights      P_j = leaf_j / T, w_j = (size_total * P_j)^-beta / max w
//   dqn_dp_gather       rank r's strata [r k, (r+1) k): frames and metadata read
//                       straight from the owners' rings through CUDA IPC peer
//                       mappings (NVLink), no frame collective
//   (learner update on the local batch; gradients all_reduce SUM; TD all_gather)
//   dqn_dp_owned        owned strata in global batch order -> dqn_tree_update_n,
//                       max_p over all K TD errors (identical on every rank)
#include "common.cuh"
#include "tree_descend.cuh"

#include <math.h>
#include <string.h>

namespace dqn {
namespace {

constexpr int kMaxRanks = 64;

__global__ void dp_info_kernel(const double *__restrict__ nodes, const int64_t *__restrict__ size,
                               const double *__restrict__ max_p, double *__restrict__ out) {
  pdl_begin();
  if (threadIdx.x == 0) {
    out[0] = nodes[1];
    out[1] = (double)*size;
    out[2] = *max_p;
  }
}

// dp.py stratified_queries, one thread per stratum (K <= 1024).
__global__ void dp_route_kernel(const double *__restrict__ info, int world,
                                const double *__restrict__ u, int K, int64_t *__restrict__ owner,
                                double *__restrict__ q_local, double *__restrict__ sums,
                                int32_t *flags, const double *__restrict__ nodes, int depth,
                                int rank, double *__restrict__ table) {
  pdl_begin();
  __shared__ double prefix[kMaxRanks + 1];
  __shared__ double tot[kMaxRanks];
  if (threadIdx.x == 0) {
    double acc = 0.0, mx = 0.0;
    int64_t n = 0;
    prefix[0] = 0.0;
    for (int r = 0; r < world; ++r) {
      tot[r] = info[3 * r];
      acc = __dadd_rn(acc, tot[r]);              // T = t_0 + t_1 + ... in rank order
      prefix[r + 1] = acc;
      n += (int64_t)info[3 * r + 1];
      mx = r == 0 ? info[2] : fmax(mx, info[3 * r + 2]);
    }
    sums[0] = acc;
    sums[1] = (double)n;
    sums[2] = mx;
    if (!(acc > 0.0)) raise_flag(flags, DQN_FLAG_ZERO_TOTAL);
  }
  __syncthreads();
  const double T = prefix[world];
  const int j = threadIdx.x;
  if (j >= K) return;
  if (!(T > 0.0)) {
    owner[j] = 0;
    q_local[j] = 0.0;
    if (table) table[2 * j] = table[2 * j + 1] = 0.0;
    return;
  }
  const double seg = __ddiv_rn(T, (double)K);
  double q = __dmul_rn(__dadd_rn((double)j, u[j]), seg);
  q = fmin(fmax(q, 1e-300), nextafter(T, 0.0));
  int o = 0;                                      // first shard with prefix[o + 1] >= q
  while (o < world - 1 && prefix[o + 1] < q) ++o;
  while (o < world - 1 && tot[o] <= 0.0) ++o;     // skip empty shards (boundary rounding)
  owner[j] = o;
  const double ql = __dsub_rn(q, prefix[o]);
  q_local[j] = ql;
  if (table) {                                    // fused owner descent (dp_descend_kernel)
    double idx = 0.0, leaf = 0.0;
    const double total = nodes[1];
    if (o == rank && total > 0.0) {
      double lv;
      idx = (double)tree_descend(nodes, depth, ql, nextafter(total, 0.0), &lv);
      leaf = lv;
    }
    table[2 * j] = idx;
    table[2 * j + 1] = leaf;
  }
}

__global__ void dp_descend_kernel(const double *__restrict__ nodes, int depth,
                                  const int64_t *__restrict__ owner,
                                  const double *__restrict__ q_local, int K, int rank,
                                  double *__restrict__ table) {
  pdl_begin();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  double idx = 0.0, leaf = 0.0;
  const double total = nodes[1];
  if (owner[j] == rank && total > 0.0) {
    double lv;
    const int64_t i = tree_descend(nodes, depth, q_local[j], nextafter(total, 0.0), &lv);
    idx = (double)i;
    leaf = lv;
  }
  table[2 * j] = idx;
  table[2 * j + 1] = leaf;
}

// IS weights over the global batch by one CTA (any size): raw weights, max,
// normalise; this rank's strata get their weight, every stratum its slot.
__device__ void dp_weights_cta(const double *__restrict__ table, const double *__restrict__ sums,
                               const double *__restrict__ beta_p, int K, int k, int rank,
                               int64_t *__restrict__ local_idx, double *__restrict__ w_all,
                               double *__restrict__ w_mine) {
  __shared__ double red[32];
  const double T = sums[0], size_total = sums[1], beta = *beta_p;
  double m = 0.0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    double w = 0.0;
    if (T > 0.0) w = pow(__dmul_rn(size_total, __ddiv_rn(table[2 * j + 1], T)), -beta);
    w_all[j] = w;
    local_idx[j] = (int64_t)table[2 * j];
    m = fmax(m, w);
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int i = 1; i < (int)((blockDim.x + 31) >> 5); ++i) v = fmax(v, red[i]);
    red[0] = v;
  }
  __syncthreads();
  const double mx = red[0];
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double wn = mx > 0.0 ? __ddiv_rn(w_all[j], mx) : 0.0;
    w_all[j] = wn;
    if (j >= rank * k && j < (rank + 1) * k) w_mine[j - rank * k] = wn;
  }
}

// IS weights over the global batch (replay.py:227-229 with P over the union
// of shards); this rank's strata get their weight and local slot.
__global__ void dp_weights_kernel(const double *__restrict__ table, const double *__restrict__ sums,
                                  const double *__restrict__ beta_p, int K, int k, int rank,
                                  int64_t *__restrict__ local_idx, double *__restrict__ w_all,
                                  double *__restrict__ w_mine) {
  pdl_begin();
  __shared__ double red[32];
  const int j = threadIdx.x;
  const double T = sums[0], size_total = sums[1], beta = *beta_p;
  double w = 0.0;
  if (j < K && T > 0.0) {
    const double p = __ddiv_rn(table[2 * j + 1], T);
    w = pow(__dmul_rn(size_total, p), -beta);
  }
  if (j < K) local_idx[j] = (int64_t)table[2 * j];
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
  if (j < K) {
    const double wn = red[0] > 0.0 ? __ddiv_rn(w, red[0]) : 0.0;
    w_all[j] = wn;
    if (j >= rank * k && j < (rank + 1) * k) w_mine[j - rank * k] = wn;
  }
}

// One CTA per (stratum of this rank, which frame): 16-byte copies of the
// state / next state from the owner's ring; CTA (b, 0) also copies the
// metadata.  Frames land in x[b] (states) and x[k + b] (next states).
__global__ void __launch_bounds__(256)
dp_gather_kernel(const dqn_peer_ring *__restrict__ rings, const int64_t *__restrict__ owner,
                 const double *__restrict__ table, int k, int rank, int64_t slot_bytes,
                 uint8_t *__restrict__ x, int64_t *__restrict__ actions, double *__restrict__ rewards,
                 uint8_t *__restrict__ terminals, const double *__restrict__ sums,
                 const double *__restrict__ beta_p, int K, int64_t *__restrict__ local_idx,
                 double *__restrict__ w_all, double *__restrict__ w_mine) {
  pdl_begin();
  const int b = blockIdx.x, which = blockIdx.y;
  if (which == 2) {                 // CTA (0, 2): the IS weights beside the frame copies
    if (b == 0) dp_weights_cta(table, sums, beta_p, K, k, rank, local_idx, w_all, w_mine);
    return;
  }
  const int j = rank * k + b;
  const int o = (int)owner[j];
  const int64_t slot = (int64_t)table[2 * j];
  const dqn_peer_ring R = rings[o];
  const uint8_t *src = (which ? R.next_states : R.states) + slot * slot_bytes;
  uint8_t *dst = x + ((int64_t)which * k + b) * slot_bytes;
  const int64_t n16 = slot_bytes / 16;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  uint4 *d4 = reinterpret_cast<uint4 *>(dst);
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) d4[i] = s4[i];
  for (int64_t i = n16 * 16 + threadIdx.x; i < slot_bytes; i += blockDim.x) dst[i] = src[i];
  if (which == 0 && threadIdx.x == 0) {
    actions[b] = R.actions[slot];
    rewards[b] = R.rewards[slot];
    terminals[b] = R.terminals[slot];
  }
}

// Owned strata in global batch order (the owner's update_priorities call,
// replay.py:232-241) and max_priority over ALL K errors (same on every rank).
__global__ void dp_owned_kernel(const int64_t *__restrict__ owner,
                                const int64_t *__restrict__ local_idx,
                                const double *__restrict__ td_all, int K, int rank, double eps,
                                int64_t *__restrict__ idx_c, double *__restrict__ td_c,
                                int32_t *__restrict__ n_c, double *__restrict__ max_p,
                                const int32_t *flags, const double *__restrict__ sums) {
  pdl_begin();
  __shared__ int s_pos[1025];
  __shared__ double red[32];
  __shared__ int bad;
  const int j = threadIdx.x;
  if (j == 0) bad = 0;
  const bool mine = j < K && owner[j] == rank;
  s_pos[j + 1] = mine ? 1 : 0;
  if (j == 0) s_pos[0] = 0;
  __syncthreads();
  if (j == 0) {                                    // K <= 1024: serial scan is enough
    for (int i = 1; i <= K; ++i) s_pos[i] += s_pos[i - 1];
    *n_c = s_pos[K];
  }
  __syncthreads();
  if (mine) {
    idx_c[s_pos[j]] = local_idx[j];
    td_c[s_pos[j]] = td_all[j];
  }
  double m = -INFINITY;
  if (j < K) {
    const double p = __dadd_rn(fabs(td_all[j]), eps);
    if (!(p >= 0.0) || isinf(p)) atomicExch(&bad, 1);
    m = p;
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((j & 31) == 0) red[j >> 5] = m;
  __syncthreads();
  if (j == 0 && !bad && !(flags && (*flags & (DQN_FLAG_ZERO_TOTAL | DQN_FLAG_NONFINITE_OUT)))) {
    double v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    if (sums) v = fmax(v, sums[2]);      // the global running max over the shards
    if (v > *max_p) *max_p = v;
  }
}

// Results of a global update for the host, written into pinned host memory
// by the device (zero-copy): [td | w | owner | local idx] as doubles, then
// the status word last (fenced), which the host polls.
__global__ void dp_report_kernel(const double *__restrict__ td_all,
                                 const double *__restrict__ w_all,
                                 const int64_t *__restrict__ owner,
                                 const int64_t *__restrict__ local_idx, int K,
                                 const int32_t *__restrict__ flags, double *host_out,
                                 int32_t *host_flag) {
  pdl_begin();
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    host_out[j] = td_all[j];
    host_out[K + j] = w_all[j];
    host_out[2 * K + j] = (double)owner[j];
    host_out[3 * K + j] = (double)local_idx[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *(volatile int32_t *)host_flag = *flags;
  }
}

}  // namespace
}  // namespace dqn

using namespace dqn;

static int threads_for(int K) { return ((K + 31) / 32) * 32; }

extern "C" int dqn_dp_shard_info(void *stream, const double *nodes, const int64_t *size,
                                 const double *max_p, double *out3) {
  DQN_CHECK_ARG(nodes && size && max_p && out3, "dp_shard_info: null pointer");
  launch_k(dp_info_kernel, 1, 32, 0, as_stream(stream), nodes, size, max_p, out3);
  DQN_LAUNCH_CHECK("dp_shard_info");
  return DQN_OK;
}

extern "C" int dqn_dp_route(void *stream, const double *info, int32_t world, const double *u,
                            int32_t K, int64_t *owner, double *q_local, double *sums,
                            int32_t *flags, const double *nodes, int32_t depth, int32_t rank,
                            double *table) {
  DQN_CHECK_ARG(info && u && owner && q_local && sums && world >= 1 && world <= kMaxRanks &&
                    K >= 1 && K <= 1024 && (!table || (nodes && depth >= 1 && depth < 40)),
                "dp_route: bad args (world <= 64, K <= 1024)");
  launch_k(dp_route_kernel, 1, threads_for(K), 0, as_stream(stream), info, world, u, K, owner,
           q_local, sums, flags, nodes, depth, rank, table);
  DQN_LAUNCH_CHECK("dp_route");
  return DQN_OK;
}

extern "C" int dqn_dp_descend(void *stream, const double *nodes, int32_t depth,
                              const int64_t *owner, const double *q_local, int32_t K, int32_t rank,
                              double *table) {
  DQN_CHECK_ARG(nodes && owner && q_local && table && K >= 1 && depth >= 1 && depth < 40,
                "dp_descend: bad args");
  launch_k(dp_descend_kernel, (K + 127) / 128, 128, 0, as_stream(stream), nodes, depth, owner,
           q_local, K, rank, table);
  DQN_LAUNCH_CHECK("dp_descend");
  return DQN_OK;
}

extern "C" int dqn_dp_weights(void *stream, const double *table, const double *sums,
                              const double *beta, int32_t K, int32_t k, int32_t rank,
                              int64_t *local_idx, double *w_all, double *w_mine) {
  DQN_CHECK_ARG(table && sums && beta && local_idx && w_all && w_mine && K >= 1 && K <= 1024 &&
                    k >= 1 && (rank + 1) * k <= K,
                "dp_weights: bad args");
  launch_k(dp_weights_kernel, 1, threads_for(K), 0, as_stream(stream), table, sums, beta, K, k,
           rank, local_idx, w_all, w_mine);
  DQN_LAUNCH_CHECK("dp_weights");
  return DQN_OK;
}

extern "C" int dqn_dp_gather(void *stream, const dqn_peer_ring *rings, const int64_t *owner,
                             const double *table, int32_t k, int32_t rank, int64_t slot_bytes,
                             uint8_t *x, int64_t *actions, double *rewards, uint8_t *terminals,
                             const double *sums, const double *beta, int32_t K,
                             int64_t *local_idx, double *w_all, double *w_mine) {
  DQN_CHECK_ARG(rings && owner && table && x && actions && rewards && terminals && k >= 1 &&
                    slot_bytes > 0 && slot_bytes % 16 == 0 &&
                    (!sums || (beta && local_idx && w_all && w_mine && K >= (rank + 1) * k)),
                "dp_gather: bad args");
  launch_k(dp_gather_kernel, dim3(k, sums ? 3 : 2), 256, 0, as_stream(stream), rings, owner,
           table, k, rank, slot_bytes, x, actions, rewards, terminals, sums, beta, K, local_idx,
           w_all, w_mine);
  DQN_LAUNCH_CHECK("dp_gather");
  return DQN_OK;
}

extern "C" int dqn_dp_owned(void *stream, const int64_t *owner, const int64_t *local_idx,
                            const double *td_all, int32_t K, int32_t rank, double eps,
                            int64_t *idx_c, double *td_c, int32_t *n_c, double *max_p,
                            const int32_t *flags, const double *sums) {
  DQN_CHECK_ARG(owner && local_idx && td_all && idx_c && td_c && n_c && max_p && K >= 1 &&
                    K <= 1024,
                "dp_owned: bad args");
  launch_k(dp_owned_kernel, 1, threads_for(K), 0, as_stream(stream), owner, local_idx, td_all, K,
           rank, eps, idx_c, td_c, n_c, max_p, flags, sums);
  DQN_LAUNCH_CHECK("dp_owned");
  return DQN_OK;
}

// --- device memory shareable across processes (CUDA IPC) -------------------
// Replay shards of the data-parallel learner are plain cudaMalloc allocations
// so that their IPC handles cover exactly the buffer; peers map them with
// cudaIpcOpenMemHandle (lazy peer access: NVLink loads from the gather kernel).
extern "C" int dqn_dev_alloc(int64_t bytes, void **ptr) {
  DQN_CHECK_ARG(ptr && bytes > 0, "dev_alloc: bad args");
  return cuda_status(cudaMalloc(ptr, (size_t)bytes), "dev_alloc");
}

extern "C" int dqn_dev_free(void *ptr) {
  if (!ptr) return DQN_OK;
  return cuda_status(cudaFree(ptr), "dev_free");
}

extern "C" int dqn_ipc_handle(void *ptr, uint8_t *handle64) {
  DQN_CHECK_ARG(ptr && handle64, "ipc_handle: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  const int rc = cuda_status(cudaIpcGetMemHandle(&h, ptr), "ipc_handle");
  if (rc) return rc;
  memcpy(handle64, &h, 64);
  return DQN_OK;
}

extern "C" int dqn_ipc_open(const uint8_t *handle64, void **ptr) {
  DQN_CHECK_ARG(ptr && handle64, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc_open");
}

extern "C" int dqn_ipc_close(void *ptr) {
  if (!ptr) return DQN_OK;
  return cuda_status(cudaIpcCloseMemHandle(ptr), "ipc_close");
}

extern "C" int dqn_dp_report(void *stream, const double *td_all, const double *w_all,
                             const int64_t *owner, const int64_t *local_idx, int32_t K,
                             const int32_t *flags, double *host_out, int32_t *host_flag) {
  DQN_CHECK_ARG(td_all && w_all && owner && local_idx && flags && host_out && host_flag && K >= 1,
                "dp_report: bad args");
  launch_k(dp_report_kernel, 1, 256, 0, as_stream(stream), td_all, w_all, owner, local_idx, K,
           flags, host_out, host_flag);
  DQN_LAUNCH_CHECK("dp_report");
  return DQN_OK;
}
