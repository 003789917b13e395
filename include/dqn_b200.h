/*
 * dqn_b200.h -- C ABI of libdqn_b200.so, the B200 (sm_100a) implementation of
 * the CytonRL / deepq learner hot path.
 *
 * The reference (/root/reference/pkg/src/deepq) has no FFI: its boundary is
 * the duck-typed Python API that ``learn_step`` consumes.  Every entry point
 * below replaces one reference method and names it (file:line).  The Python
 * mirror in paper_1804_05834_b200/ binds these with ctypes (INTEGRATION.md
 * shows the binding a deepq maintainer would add).
 *
 * Conventions
 *  - All pointers are DEVICE pointers on the current device unless the name
 *    says ``host``.  Scalars are passed by value.  The caller owns every
 *    buffer; the library never allocates or frees caller memory.
 *  - ``stream`` is a cudaStream_t; all work is asynchronous on it, nothing
 *    synchronises the device, and every call is legal inside CUDA-graph
 *    capture.
 *  - Return value: 0 (DQN_OK) or a dqn_status; ``dqn_last_error()`` holds a
 *    thread-local message.  Faults only detectable on the device (an index out
 *    of range, zero total priority, a non-finite gradient) are OR-ed into a
 *    caller-provided int32 ``flags`` word (DQN_FLAG_*); the host reads it
 *    lazily and raises the reference's exception (errors.py:4-41).
 */
#ifndef DQN_B200_H
#define DQN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DQN_OK = 0,
  DQN_ERR_INVALID_ARG = 1,   /* ValueError */
  DQN_ERR_GEOMETRY = 2,      /* GeometryError (layers.py:182-190) */
  DQN_ERR_INDEX = 3,         /* IndexError (replay.py:157,239) */
  DQN_ERR_EMPTY = 4,         /* ValueError: empty replay (replay.py:120,219) */
  DQN_ERR_ZERO_TOTAL = 5,    /* ValueError: zero total (replay.py:171,222) */
  DQN_ERR_NONFINITE = 6,     /* NonFiniteError (network.py:102, optim.py:40) */
  DQN_ERR_CUDA = 7,
  DQN_ERR_UNSUPPORTED = 8    /* ConfigError */
} dqn_status;

/* device flag bits (int32 word written by kernels, read lazily by the host) */
#define DQN_FLAG_INDEX          0x1  /* update_priorities index out of range */
#define DQN_FLAG_ZERO_TOTAL     0x2  /* sample from a zero-mass tree */
#define DQN_FLAG_NONFINITE_GRAD 0x4  /* RmsProp.step finite scan failed: no update applied */
#define DQN_FLAG_NONFINITE_OUT  0x8  /* network output non-finite */
#define DQN_FLAG_BAD_PRIORITY   0x10 /* SumTree.set with negative / non-finite value */

const char *dqn_last_error(void);
int dqn_abi_version(void);             /* 5 */
/* 1 if this library was built with the tcgen05 (sm_100a UMMA) conv trunk */
int dqn_has_tcgen05(void);
/* kernels launched (or captured) through this library so far, all threads */
int64_t dqn_launch_count(void);

/* ------------------------------------------------------------------ replay */

/* Synthetic frames: bytes = splitmix64(counter_base | (slot*words + w)),
 * little-endian, for slots [slot0, slot0+nslots).  Test / bench input
 * generator (no reference counterpart; mirrors synth.frames on the host). */
int dqn_ring_fill_hash(void *stream, uint8_t *frames, int64_t slot0, int64_t nslots,
                       int64_t slot_bytes, uint64_t counter_base);

/* ReplayMemory._gather (replay.py:104-115): fancy-index gather of k slots.
 * states/next_states are [capacity][slot_bytes] byte rings (u8 frames or raw
 * float32 states).  Any output pointer may be NULL to skip it. */
int dqn_ring_gather(void *stream, const uint8_t *states, const uint8_t *next_states,
                    int64_t slot_bytes, const int64_t *actions, const double *rewards,
                    const uint8_t *terminals, const int64_t *idx, int32_t k,
                    uint8_t *out_states, uint8_t *out_next_states, int64_t *out_actions,
                    double *out_rewards, uint8_t *out_terminals);

/* PrioritizedReplay.sample (replay.py:215-229) + SumTree.find (167-181):
 * stratified queries q_j = (j + u_j) * (total / k), clipped descent, P = leaf
 * / total, w = (size * P)^-beta / max w.  ``beta`` and ``size`` (the ring's
 * fill count) are device scalars so a captured graph follows them.  Bit-exact with the reference given u. */
int dqn_tree_sample(void *stream, const double *nodes, int32_t depth, const int64_t *size,
                    const double *u, int32_t k, const double *beta, int64_t *idx,
                    double *prob, double *weight, int32_t *flags);

/* SumTree.find alone (replay.py:167-181) for arbitrary query masses. */
int dqn_tree_find(void *stream, const double *nodes, int32_t depth, const double *queries,
                  int64_t n, int64_t *idx, int32_t *flags);

/* PrioritizedReplay.update_priorities (replay.py:232-241): in batch order,
 * leaf_i = (|td_i| + eps)^alpha (last write wins), ancestors recomputed from
 * children; *max_p = max(*max_p, max(|td|+eps)).  An index outside [0,*size)
 * stops the update at that position (leaves before it stay written, as in the
 * reference), sets DQN_FLAG_INDEX and leaves max_p untouched. */
int dqn_tree_update(void *stream, double *nodes, int32_t depth, const int64_t *size,
                    const int64_t *idx, const double *td, int32_t k, double alpha,
                    double eps, double *max_p, int32_t *flags);

/* PrioritizedReplay.store's tree half (replay.py:207-210) for n consecutive
 * ring slots starting at ``slot`` (wrapping at capacity): leaf = max_p^alpha. */
int dqn_tree_store(void *stream, double *nodes, int32_t depth, int64_t capacity,
                   int64_t slot, int64_t n, const double *max_p, double alpha);

/* SumTree.set for k leaves (replay.py:155-165), batch order, last wins. */
int dqn_tree_set(void *stream, double *nodes, int32_t depth, int64_t capacity,
                 const int64_t *idx, const double *values, int32_t k, int32_t *flags);

/* Recompute every internal node bottom-up (bulk load). */
int dqn_tree_rebuild(void *stream, double *nodes, int32_t depth);

/* ----------------------------------------------------------------- network */

#define DQN_MAX_LAYERS 8

typedef enum { DQN_LAYER_CONV = 0, DQN_LAYER_LINEAR = 1, DQN_LAYER_DUELING = 2 } dqn_layer_kind;

/* One parameterised layer (layers.py:115-330) with an optional fused ReLU
 * (layers.py:99-112).  Linear layers use in_h = in_w = 1, in_c = features.
 * Offsets are in floats into the flat parameter (and gradient) buffers, laid
 * out in the reference registry order (network.py:74-84). */
typedef struct {
  int32_t kind, relu;
  int32_t in_h, in_w, in_c;
  int32_t out_h, out_w, out_c;
  int32_t fh, fw, sh, sw;
  int64_t w_off, b_off;    /* conv/linear weight+bias; dueling: value branch */
  int64_t w2_off, b2_off;  /* dueling: advantage branch */
} dqn_layer_desc;

/* dqn_net_desc.hints: this network's forward runs beside another one that is
 * on the critical path (the learner's target trunk beside its online trunk):
 * its launches take fewer SMs (smaller K splits / clusters).  Results differ
 * from the unhinted forward only by fp32 summation order. */
#define DQN_NET_HINT_SIDE 1

typedef struct {
  int32_t n_layers;
  int32_t input_u8;        /* 1: input bytes x = f32(u8)/255 (envs.py:300-311); 0: float32 */
  int32_t algo;            /* 0: auto (tcgen05 trunk when the geometry has a kernel), 1: SIMT only */
  int32_t hints;           /* DQN_NET_HINT_*: launch shapes only, never the formulas */
  dqn_layer_desc layer[DQN_MAX_LAYERS];
} dqn_net_desc;

/* Activations for one batch extent (layers.py:65-77 bindings).  act[l] is
 * layer l's output after its fused ReLU; dact[l] is the gradient w.r.t. layer
 * l's pre-activation output.  ``scratch`` holds split-K partial sums; size it
 * with dqn_net_scratch_floats. */
typedef struct {
  int32_t batch, pad_;
  const void *x;
  float *act[DQN_MAX_LAYERS];
  float *dact[DQN_MAX_LAYERS];
  float *dx;               /* input gradient (NULL = skip, as the learner does) */
  float *scratch;
  int64_t scratch_floats;
} dqn_binding;

int64_t dqn_net_scratch_floats(const dqn_net_desc *net, int32_t batch);

/* Network.forward (network.py:90-104): all layers front to back. */
int dqn_net_forward(void *stream, const dqn_net_desc *net, const float *params,
                    const dqn_binding *bind, int32_t *flags);

/* Network.backward (network.py:106-117): dq is the [batch][n_actions] output
 * gradient; fills dact[] (and dx when non-NULL). */
int dqn_net_backward(void *stream, const dqn_net_desc *net, const float *params,
                     const dqn_binding *bind, const float *dq);

/* Network.calculate_gradient (network.py:119-126): grads += dW, db for every
 * layer (deterministic fixed-order reductions, no float atomics). */
int dqn_net_wgrad(void *stream, const dqn_net_desc *net, float *grads,
                  const dqn_binding *bind);

/* One phase of one layer (0 forward, 1 backward to the layer's input,
 * 2 wgrad) -- the unit the bench times for its roofline line. */
int dqn_net_layer(void *stream, const dqn_net_desc *net, const float *params, float *grads,
                  const dqn_binding *bind, int32_t layer, int32_t phase, int32_t *flags);

/* ---------------------------------------------------------- loss / optim */

/* Work bytes dqn_head_td needs for `batch` rows and `n_actions` actions
 * (zero-initialised once by the caller; left zeroed between calls). */
int64_t dqn_head_td_work_bytes(int32_t batch, int32_t n_actions);

/* The learner's head block in two launches (replaces head forward x2,
 * dqn_td_loss, the head's dgrad and wgrad of learn_step, agent.py:91-132):
 * Q heads of the online net (on_bind: [s; s'] rows for Double DQN) and the
 * target net (tg_bind: s' rows) from their hidden features, then the TD block
 * exactly as dqn_td_loss (targets/td/losses/stats, dq into on_view->dact[L-1]),
 * the head backward into on_view->dact[L-2] (masked by the hidden ReLU) and
 * the head weight gradient added to on_grads.  Linear or dueling heads with
 * at most 18 actions and batch <= 1024; DQN_ERR_UNSUPPORTED otherwise.
 * host_out (optional, pinned host memory mapped for the device): also gets
 * [targets | td | losses | stats] (3 batch + 2 doubles), written by the
 * kernel itself -- no device-to-host copy in the learner's graph. */
int dqn_head_td(void *stream, const dqn_net_desc *on_net, const float *on_params,
                float *on_grads, const dqn_binding *on_bind, const dqn_binding *on_view,
                const dqn_net_desc *tg_net, const float *tg_params, const dqn_binding *tg_bind,
                const int64_t *actions, const double *rewards, const uint8_t *terminals,
                const double *weights, double gamma, int32_t td_flags, double *targets,
                double *td, double *losses, double *stats, void *work, int32_t *flags,
                double *host_out);

#define DQN_TD_DOUBLE 0x1
#define DQN_TD_HUBER 0x2
#define DQN_TD_REWARD_CLIP 0x4
/* dqn_head_td only: the last-CTA head form instead of the two-phase form */
#define DQN_TD_HEAD_LAST_CTA 0x8

/* compute_target_double / compute_target_dqn (agent.py:58-73) and the loss
 * block of learn_step (agent.py:110-124): argmax (first max), y = r + (t ? 0 :
 * gamma * Q_tg), delta = y - f64(Q_on(s,a)) in fp64, squared or Huber loss,
 * dq = f32(-w * delta) at (j, a_j) and 0 elsewhere.  q_next_online may be NULL
 * when !(flags & DQN_TD_DOUBLE).  stats[0] = sum|delta|, stats[1] = sum loss. */
int dqn_td_loss(void *stream, const float *q_online, const float *q_next_online,
                const float *q_next_target, const int64_t *actions, const double *rewards,
                const uint8_t *terminals, const double *weights, int32_t batch,
                int32_t n_actions, double gamma, int32_t flags, double *targets,
                double *td, double *losses, float *dq, double *stats);

/* Frame-deduplicated ring gather (replaces ReplayMemory._gather,
 * replay.py:104-115, for rings that keep each H x W frame once; the
 * reference itself stores full stacks).  frames: pool of
 * frame_bytes-byte planes; ids: per ring slot 2*stack int64 pool ids (state
 * planes, then next-state planes).  Writes the k sampled transitions'
 * channel-last stacks (frame_bytes * stack bytes each, byte-identical to a
 * full-stack ring holding the same transitions) and, where given, their
 * action / reward / terminal.  Indices must be valid slots. */
int dqn_frame_gather(void *stream, const uint8_t *frames, int64_t frame_bytes,
                     const int64_t *ids, int stack, const int64_t *indices, int k,
                     const int64_t *actions, const double *rewards, const bool *terminals,
                     uint8_t *out_states, uint8_t *out_next_states, int64_t *out_actions,
                     double *out_rewards, bool *out_terminals);

/* PrioritizedReplay.sample + _gather on the frame-deduplicated ring in ONE
 * launch (replay.py:104-115, 215-230): as dqn_sample_gather (stratified
 * descent per gather CTA, IS-weight CTA row), the stacks assembled from the
 * frame pool as dqn_frame_gather does.  Identical to dqn_tree_sample
 * followed by dqn_frame_gather.  prob == weight == NULL: no weights row, as
 * for dqn_sample_gather. */
int dqn_frame_sample_gather(void *stream, const double *nodes, int32_t depth, const int64_t *size,
                            const double *u, int32_t k, const double *beta, int64_t *idx,
                            double *prob, double *weight, int32_t *flags, const uint8_t *frames,
                            int64_t frame_bytes, const int64_t *ids, int stack,
                            const int64_t *actions, const double *rewards, const bool *terminals,
                            uint8_t *out_states, uint8_t *out_next_states, int64_t *out_actions,
                            double *out_rewards, bool *out_terminals);

/* RmsProp.step (optim.py:36-47) over a flat buffer: finite scan of all grads,
 * then (only if all finite) acc = acc*rho; acc += (1-rho)*g*g;
 * w -= (lr*g)/(sqrt(acc)+eps); g = 0 -- fp32, no FMA, bit-exact given g.
 * A non-finite gradient sets DQN_FLAG_NONFINITE_GRAD and applies nothing. */
int dqn_rmsprop_step(void *stream, float *w, float *g, float *acc, int64_t n,
                     float lr, float rho, float one_minus_rho, float eps, int32_t *flags);

/* The update of dqn_rmsprop_step without the finiteness scan, for gradients
 * whose producers raised DQN_FLAG_NONFINITE_GRAD as they wrote them
 * (dqn_net_layer phase 2 with a flag word, dqn_head_td): skipped on any error
 * flag, exactly as dqn_rmsprop_step.  flag_out (optional, pinned host memory):
 * receives the step's flag word once every earlier kernel of the stream has
 * completed (the learner's completion signal, polled by the host). */
int dqn_rmsprop_apply(void *stream, float *w, float *g, float *acc, int64_t n, float lr,
                      float rho, float one_minus_rho, float eps, int32_t *flags,
                      int32_t *flag_out);

/* clip_gradients (optim.py:61-75): fp64 global L2 norm into *norm_out; if
 * norm > max_norm, g *= f32(max_norm / norm). */
int dqn_clip_gradients(void *stream, float *g, int64_t n, double max_norm, double *norm_out);

/* sync_target (optim.py:78-89): bitwise copy of the flat parameter buffer. */
int dqn_sync_target(void *stream, float *dst, const float *src, int64_t n);

/* ---- data-parallel learner (algorithm in dp.py) --------
 * N ranks (one per GPU), rank r owns replay shard r (global transition g at
 * rank g % N, slot g / N) with its own sum tree; K = k * N strata per global
 * update.  The reference has no distributed mode: each entry restates one
 * step of a global learn_step (agent.py:91-132, replay.py:215-241) over the
 * union of the shards. */
typedef struct dqn_peer_ring {    /* a rank's ring, mapped into this process */
  const uint8_t *states;
  const uint8_t *next_states;
  const int64_t *actions;
  const double *rewards;
  const uint8_t *terminals;
} dqn_peer_ring;

/* out3 = [tree total, ring size, max_priority] of this shard (all_gathered). */
int dqn_dp_shard_info(void *stream, const double *nodes, const int64_t *size,
                      const double *max_p, double *out3);
/* info = N x 3 gathered shard infos; u = K uniforms (same on every rank).
 * T = totals summed in rank order; q_j = clip((j + u_j) * T / K) as
 * SumTree.find clips; owner_j = first shard whose prefix mass reaches q_j;
 * q_local = q_j - prefix[owner_j]; sums = [T, total size, max of max_p].
 * With table != NULL the owner descent of dqn_dp_descend is fused in (this
 * rank's tree = nodes/depth). */
int dqn_dp_route(void *stream, const double *info, int32_t world, const double *u, int32_t K,
                 int64_t *owner, double *q_local, double *sums, int32_t *flags,
                 const double *nodes, int32_t depth, int32_t rank, double *table);
/* table[j] = (leaf index, leaf value) for the strata this rank owns, zeros
 * elsewhere (all_reduce SUM gives every rank the full table). */
int dqn_dp_descend(void *stream, const double *nodes, int32_t depth, const int64_t *owner,
                   const double *q_local, int32_t K, int32_t rank, double *table);
/* P_j = leaf_j / T, w_j = (size_total * P_j)^-beta / max_j w_j (replay.py:227-229
 * over the global batch); local_idx[j] = table index; w_mine = this rank's k. */
int dqn_dp_weights(void *stream, const double *table, const double *sums, const double *beta,
                   int32_t K, int32_t k, int32_t rank, int64_t *local_idx, double *w_all,
                   double *w_mine);
/* This rank's strata [rank k, (rank+1) k) read from the owners' rings
 * (rings[N], peer mappings; slot = table[j].index): states to x[0..k), next
 * states to x[k..2k).  With sums != NULL one extra CTA computes the IS
 * weights of dqn_dp_weights in the same launch. */
int dqn_dp_gather(void *stream, const dqn_peer_ring *rings, const int64_t *owner,
                  const double *table, int32_t k, int32_t rank, int64_t slot_bytes, uint8_t *x,
                  int64_t *actions, double *rewards, uint8_t *terminals, const double *sums,
                  const double *beta, int32_t K, int64_t *local_idx, double *w_all,
                  double *w_mine);
/* The owned strata in global batch order -> idx_c/td_c/*n_c (for
 * dqn_tree_update_n); max_p = max(max_p, sums[2], max_j |td_j| + eps) over
 * all K, so every shard keeps the global running max priority (sums from
 * dqn_dp_route; NULL = this shard's only). */
int dqn_dp_owned(void *stream, const int64_t *owner, const int64_t *local_idx,
                 const double *td_all, int32_t K, int32_t rank, double eps, int64_t *idx_c,
                 double *td_c, int32_t *n_c, double *max_p, const int32_t *flags,
                 const double *sums);
/* The update's results for the host, written by the device into pinned host
 * memory: host_out = [td | w | owner | local idx] (4 K doubles), then
 * *host_flag = *flags (fenced; the host's completion signal). */
int dqn_dp_report(void *stream, const double *td_all, const double *w_all, const int64_t *owner,
                  const int64_t *local_idx, int32_t K, const int32_t *flags, double *host_out,
                  int32_t *host_flag);
/* dqn_tree_update with the batch length read from device memory (*k_dev <= k_max <= 256). */
int dqn_tree_update_n(void *stream, double *nodes, int32_t depth, const int64_t *size,
                      const int64_t *idx, const double *td, int32_t k_max, const int32_t *k_dev,
                      double alpha, double eps, double *max_p, int32_t *flags);
/* Process-shareable device memory for replay shards (CUDA IPC). */
int dqn_dev_alloc(int64_t bytes, void **ptr);
int dqn_dev_free(void *ptr);
int dqn_ipc_handle(void *ptr, uint8_t *handle64);
int dqn_ipc_open(const uint8_t *handle64, void **ptr);
int dqn_ipc_close(void *ptr);

/* ReplayMemory.store_many (replay.py:91-102): n staged transitions into slots
 * (cursor + i) % capacity (raw state bytes, any ring dtype; n <= capacity);
 * the sources may be pinned host memory, read in place.  *size_dev (optional)
 * = new_size.  The PER tree half is dqn_tree_store. */
int dqn_ring_store(void *stream, uint8_t *states, uint8_t *next_states, int64_t slot_bytes,
                   int64_t *actions, double *rewards, uint8_t *terminals, int64_t capacity,
                   int64_t cursor, int32_t n, const uint8_t *src_states,
                   const uint8_t *src_next_states, const int64_t *src_actions,
                   const double *src_rewards, const uint8_t *src_terminals, int64_t *size_dev,
                   int64_t new_size);

/* dqn_tree_sample followed by dqn_ring_gather of the sampled slots (states,
 * next states, metadata) in ONE launch: each gather CTA descends its own
 * query, one extra CTA row computes the batch-normalised IS weights.  Same
 * results as the two calls (replay.py:104-115, 215-230); 16-byte aligned
 * frames (slot_bytes % 16 == 0).  prob == weight == NULL: no weights row --
 * the gather CTAs write idx, and the caller computes prob / weight with
 * dqn_tree_sample (same indices), e.g. on another stream beside the trunk. */
int dqn_sample_gather(void *stream, const double *nodes, int32_t depth, const int64_t *size,
                      const double *u, int32_t k, const double *beta, int64_t *idx,
                      double *prob, double *weight, int32_t *flags, const uint8_t *states,
                      const uint8_t *next_states, int64_t slot_bytes, const int64_t *actions,
                      const double *rewards, const uint8_t *terminals, uint8_t *out_states,
                      uint8_t *out_next_states, int64_t *out_actions, double *out_rewards,
                      uint8_t *out_terminals);

/* CUDA-graph plumbing for the learner (no reference counterpart: the
 * reference runs eagerly).  Instantiate a captured cudaGraph_t, optionally
 * honouring per-kernel-node priorities (every launch of this library carries
 * its stream's priority), launch it, destroy it. */
int dqn_graph_instantiate(void *graph, int use_node_priority, void **exec_out);
int dqn_graph_launch(void *exec, void *stream);
int dqn_graph_destroy(void *exec);

/* preprocess_frame (envs.py:289-311) for n raw uint8 frames [n][h][w][c]
 * (c = 1 gray or 3 RGB): /255, BT.601 luma, half-pixel bilinear resize to
 * out_h x out_w, all in fp64 in the reference's operation order, then f32 --
 * bit-exact.  Output pixel (i, j) of frame f goes to
 * out[f * frame_stride + (i * out_w + j) * pix_stride] (pix_stride = stack
 * depth writes one channel of an HWC frame stack). */
int dqn_preprocess_frames(void *stream, const uint8_t *frames, int64_t n, int h, int w, int c,
                          int out_h, int out_w, float *out, int64_t frame_stride,
                          int64_t pix_stride);

#ifdef __cplusplus
}
#endif
#endif /* DQN_B200_H */
