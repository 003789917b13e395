// Frame-deduplicated replay ring: stack assembly for the gather.
//
// The reference stores every transition's full state and next-state stacks
// (replay.py:83-84; SPEC.md:294 says so explicitly), 2 x 28,224 B per slot at
// Atari shapes.  Consecutive transitions of an episode share all but one of
// their frames, so the deduplicated ring keeps each H x W frame once in a
// frame pool and, per transition, the 2S pool ids of its state / next-state
// stack planes (host bookkeeping: frame_ring.py).  This kernel rebuilds the
// channel-last stacks of sampled transitions -- byte-identical to what
// ReplayMemory._gather (replay.py:104-115) returns for the same transitions
// -- plus the action / reward / terminal metadata.
//
// Bound: HBM.  Algorithmic bytes per sampled transition: 2S frame reads +
// 2 stack writes (2 x 28,224 B at Atari shapes) + ids and metadata.
#include "common.cuh"
#include "tree_descend.cuh"
#include "bulk_copy.cuh"

namespace dqn {
namespace {

constexpr int kFgThreads = 256;

// One channel-last stack from its S pool planes (row[0..S)) into dst.
// Threads [t0, t0 + nt) of the CTA (whole warps) assemble the stack; for
// the 4-plane, 16-byte path splanes (4 x frame_bytes of shared memory) and
// bar (an initialised single-use mbarrier) stage the planes.
__device__ __forceinline__ void gather_stack(const uint8_t *frames, int64_t frame_bytes,
                                             const int64_t *row, int S, uint8_t *dst, int tid,
                                             int nt, uint4 *splanes, uint64_t *bar) {
  if (S == 4 && frame_bytes % 16 == 0) {
    // 16 pixels of each plane per lane and pass: one 16-byte load per plane
    // (a warp reads 512 contiguous bytes of each plane), the 64 interleaved
    // output bytes staged through shared memory so that each store
    // instruction of the warp writes 512 contiguous bytes (slot s of lane L
    // at 4 L + ((s + L / 2) & 3): conflict-free both ways)
    __shared__ uint4 stg[kFgThreads / 32][128];
    uint4 *sw = stg[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    // the four planes arrive in shared memory by TMA bulk copies (one
    // issuing thread, no register staging), then are interleaved from there
    uint4 *p0 = splanes, *p1 = splanes + frame_bytes / 16, *p2 = p1 + frame_bytes / 16,
          *p3 = p2 + frame_bytes / 16;
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bc_smem(bar)),
                   "r"((uint32_t)(4 * frame_bytes))
                   : "memory");
      for (int s = 0; s < 4; ++s)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(bc_smem(splanes + s * (frame_bytes / 16))),
            "l"(frames + row[s] * frame_bytes), "r"((uint32_t)frame_bytes), "r"(bc_smem(bar))
            : "memory");
    }
    bc_mbar_wait(bar, 0);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    const int64_t nq = frame_bytes / 16;
    // warp-uniform trip count: lanes past nq store nothing but join the syncs
    for (int64_t q0 = tid - lane; q0 < nq; q0 += nt) {
      const int64_t q = q0 + lane;
      const bool ok = q < nq;
      uint4 A = make_uint4(0, 0, 0, 0), B = A, C = A, D = A;
      if (ok) { A = p0[q]; B = p1[q]; C = p2[q]; D = p3[q]; }
      const uint32_t a[4] = {A.x, A.y, A.z, A.w}, b[4] = {B.x, B.y, B.z, B.w},
                     c[4] = {C.x, C.y, C.z, C.w}, d[4] = {D.x, D.y, D.z, D.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int u = (t + (lane >> 1)) & 3;          // output sub-slot written this round
        uint32_t au = a[0], bu = b[0], cu = c[0], du = d[0];
#pragma unroll
        for (int v = 1; v < 4; ++v)
          if (u == v) { au = a[v]; bu = b[v]; cu = c[v]; du = d[v]; }
        const uint32_t ab_lo = __byte_perm(au, bu, 0x5140), cd_lo = __byte_perm(cu, du, 0x5140);
        const uint32_t ab_hi = __byte_perm(au, bu, 0x7362), cd_hi = __byte_perm(cu, du, 0x7362);
        sw[4 * lane + u] = make_uint4(__byte_perm(ab_lo, cd_lo, 0x5410), __byte_perm(ab_lo, cd_lo, 0x7632),
                                      __byte_perm(ab_hi, cd_hi, 0x5410), __byte_perm(ab_hi, cd_hi, 0x7632));
      }
      __syncwarp();
      const int64_t nvalid = (nq - q0 < 32 ? nq - q0 : 32) * 4;   // output uint4s of this warp pass
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int m = 32 * t + lane;
        if (m < nvalid) o[4 * q0 + m] = sw[m];
      }
      __syncwarp();
    }
  } else if (S == 4 && frame_bytes % 4 == 0) {
    // 4 pixels of each plane per thread: one u32 per plane in, the four
    // interleaved pixels (a_i b_i c_i d_i) as one 16-byte store out
    const uint32_t *p0 = reinterpret_cast<const uint32_t *>(frames + row[0] * frame_bytes);
    const uint32_t *p1 = reinterpret_cast<const uint32_t *>(frames + row[1] * frame_bytes);
    const uint32_t *p2 = reinterpret_cast<const uint32_t *>(frames + row[2] * frame_bytes);
    const uint32_t *p3 = reinterpret_cast<const uint32_t *>(frames + row[3] * frame_bytes);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    for (int64_t q = tid; q < frame_bytes / 4; q += nt) {
      const uint32_t a = __ldg(p0 + q), b = __ldg(p1 + q), c = __ldg(p2 + q), d = __ldg(p3 + q);
      const uint32_t ab_lo = __byte_perm(a, b, 0x5140), cd_lo = __byte_perm(c, d, 0x5140);
      const uint32_t ab_hi = __byte_perm(a, b, 0x7362), cd_hi = __byte_perm(c, d, 0x7362);
      o[q] = make_uint4(__byte_perm(ab_lo, cd_lo, 0x5410), __byte_perm(ab_lo, cd_lo, 0x7632),
                        __byte_perm(ab_hi, cd_hi, 0x5410), __byte_perm(ab_hi, cd_hi, 0x7632));
    }
  } else {
    for (int64_t p = tid; p < frame_bytes; p += nt)
      for (int s = 0; s < S; ++s) dst[p * S + s] = frames[row[s] * frame_bytes + p];
  }
}

// grid (k): CTA j assembles both stacks of transition j (threads [0, 128):
// state, [128, 256): next state), so the idx -> ids -> frames chain of
// dependent loads is paid once per transition
__global__ void __launch_bounds__(kFgThreads)
frame_gather_kernel(const uint8_t *__restrict__ frames, int64_t frame_bytes,
                    const int64_t *ids, int S, const int64_t *idx, const int64_t *actions,
                    const double *rewards, const bool *terms, uint8_t *__restrict__ out_s,
                    uint8_t *__restrict__ out_n, int64_t *__restrict__ out_a,
                    double *__restrict__ out_r, bool *__restrict__ out_t) {
  // no __restrict__ on idx / ids / metadata: with it the compiler may hoist
  // their loads above the PDL wait (tools/pdl_hoist_scan.py) and read
  // indices the previous kernel is still writing
  extern __shared__ __align__(128) uint4 fg_smem[];
  __shared__ uint64_t fg_bar[2];
  if (threadIdx.x == 0) {
    bc_mbar_init(&fg_bar[0]);
    bc_mbar_init(&fg_bar[1]);
  }
  __syncthreads();
  pdl_begin();
  const int j = blockIdx.x, half = kFgThreads / 2, which = threadIdx.x / half;
  const int64_t slot = idx[j];
  const int64_t *row = ids + slot * 2 * S + which * S;
  uint8_t *dst = (which ? out_n : out_s) + (int64_t)j * frame_bytes * S;
  if (threadIdx.x == 0) {
    if (out_a) out_a[j] = actions[slot];
    if (out_r) out_r[j] = rewards[slot];
    if (out_t) out_t[j] = terms[slot];
  }
  gather_stack(frames, frame_bytes, row, S, dst, threadIdx.x - which * half, half,
               fg_smem + which * (4 * frame_bytes / 16), &fg_bar[which]);
}

// Stratified sum-tree descent + stack assembly in one launch (the learner's
// PER batch from the deduplicated ring; replay.py:104-115, 215-230): CTA
// j descends query j with one warp (eight levels per round trip) and
// assembles both stacks of that slot and its metadata; the extra CTA j = k
// computes idx / P / normalised IS weights (prob == weight == nullptr: no
// extra CTA, the gather CTAs write idx; the caller runs dqn_tree_sample).
// Same results as dqn_tree_sample followed by dqn_frame_gather.
__global__ void __launch_bounds__(kFgThreads)
frame_sample_gather_kernel(const double *nodes, int depth, const int64_t *size_p, const double *u,
                           int k, const double *beta_p, int64_t *idx, double *prob,
                           double *weight, int32_t *flags, const uint8_t *frames,
                           int64_t frame_bytes, const int64_t *ids, int S,
                           const int64_t *actions, const double *rewards, const bool *terms,
                           uint8_t *out_s, uint8_t *out_n, int64_t *out_a, double *out_r,
                           bool *out_t) {
  extern __shared__ __align__(128) uint4 fg_smem[];
  __shared__ uint64_t fg_bar[2];
  if (threadIdx.x == 0) {
    bc_mbar_init(&fg_bar[0]);
    bc_mbar_init(&fg_bar[1]);
  }
  __syncthreads();
  pdl_begin();
  const int j = blockIdx.x, half = kFgThreads / 2, which = threadIdx.x / half;
  if (j == k) {
    __shared__ double red[kFgThreads / 32];
    sample_is_weights_block(nodes, depth, size_p, u, k, beta_p, idx, prob, weight, flags, red);
    return;
  }
  __shared__ int64_t s_slot;
  const double total = nodes[1];
  if (threadIdx.x < 32) {
    int64_t i = 0;
    if (total > 0.0)
      i = warp_tree_descend(nodes, depth,
                            __dmul_rn(__dadd_rn((double)j, u[j]), __ddiv_rn(total, (double)k)),
                            nextafter(total, 0.0));
    if (threadIdx.x == 0) {
      s_slot = i;
      if (weight == nullptr) idx[j] = i;   // no weights CTA: the caller's dqn_tree_sample has them
      if (out_a) out_a[j] = actions[i];
      if (out_r) out_r[j] = rewards[i];
      if (out_t) out_t[j] = terms[i];
    }
  }
  __syncthreads();
  const int64_t slot = s_slot;
  gather_stack(frames, frame_bytes, ids + slot * 2 * S + which * S, S,
               (which ? out_n : out_s) + (int64_t)j * frame_bytes * S, threadIdx.x - which * half,
               half, fg_smem + which * (4 * frame_bytes / 16), &fg_bar[which]);
}

// staged planes of both stacks (the 4-plane 16-byte path only)
inline size_t fg_smem_bytes(int64_t frame_bytes, int stack) {
  return (stack == 4 && frame_bytes % 16 == 0) ? (size_t)(2 * 4 * frame_bytes) : 0;
}
inline bool fg_configure(const void *kern, size_t smem) {
  if (smem > 200 * 1024) {
    set_error("frame gather: %zu B of staged planes per CTA", smem);
    return false;
  }
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
         cudaSuccess;
}

}  // namespace
}  // namespace dqn

using namespace dqn;

extern "C" int dqn_frame_gather(void *stream, const uint8_t *frames, int64_t frame_bytes,
                                const int64_t *ids, int stack, const int64_t *indices, int k,
                                const int64_t *actions, const double *rewards,
                                const bool *terminals, uint8_t *out_states,
                                uint8_t *out_next_states, int64_t *out_actions,
                                double *out_rewards, bool *out_terminals) {
  DQN_CHECK_ARG(frames && ids && indices && out_states && out_next_states && k >= 0 &&
                    frame_bytes > 0 && stack >= 1 && stack <= 16,
                "frame_gather: bad args");
  if (k == 0) return DQN_OK;
  if (stack == 4 && frame_bytes % 16 == 0)
    DQN_CHECK_ARG(((uintptr_t)frames % 16 == 0) && ((uintptr_t)out_states % 16 == 0) &&
                      ((uintptr_t)out_next_states % 16 == 0),
                  "frame_gather: misaligned buffers");
  else if (stack == 4 && frame_bytes % 4 == 0)
    DQN_CHECK_ARG(((uintptr_t)frames % 4 == 0) && ((uintptr_t)out_states % 16 == 0) &&
                      ((uintptr_t)out_next_states % 16 == 0),
                  "frame_gather: misaligned buffers");
  const size_t smem = fg_smem_bytes(frame_bytes, stack);
  if (smem > 48 * 1024 && !fg_configure((const void *)frame_gather_kernel, smem))
    return DQN_ERR_CUDA;
  launch_k(frame_gather_kernel, dim3(k), kFgThreads, smem, as_stream(stream), frames,
           frame_bytes, ids, stack, indices, actions, rewards, terminals, out_states,
           out_next_states, out_actions, out_rewards, out_terminals);
  DQN_LAUNCH_CHECK("frame_gather");
  return DQN_OK;
}

extern "C" int dqn_frame_sample_gather(void *stream, const double *nodes, int32_t depth,
                                       const int64_t *size, const double *u, int32_t k,
                                       const double *beta, int64_t *idx, double *prob,
                                       double *weight, int32_t *flags, const uint8_t *frames,
                                       int64_t frame_bytes, const int64_t *ids, int stack,
                                       const int64_t *actions, const double *rewards,
                                       const bool *terminals, uint8_t *out_states,
                                       uint8_t *out_next_states, int64_t *out_actions,
                                       double *out_rewards, bool *out_terminals) {
  DQN_CHECK_ARG(nodes && size && u && beta && idx && (prob == nullptr) == (weight == nullptr) &&
                    frames && ids &&
                    out_states && out_next_states && k >= 1 && k < 65535 && depth >= 1 &&
                    frame_bytes > 0 && stack >= 1 && stack <= 16,
                "frame_sample_gather: bad args");
  if (stack == 4 && frame_bytes % 16 == 0)
    DQN_CHECK_ARG(((uintptr_t)frames % 16 == 0) && ((uintptr_t)out_states % 16 == 0) &&
                      ((uintptr_t)out_next_states % 16 == 0),
                  "frame_sample_gather: misaligned buffers");
  const size_t smem = fg_smem_bytes(frame_bytes, stack);
  if (smem > 48 * 1024 && !fg_configure((const void *)frame_sample_gather_kernel, smem))
    return DQN_ERR_CUDA;
  launch_k(frame_sample_gather_kernel, dim3(k + (weight ? 1 : 0)), kFgThreads, smem, as_stream(stream), nodes,
           depth, size, u, k, beta, idx, prob, weight, flags, frames, frame_bytes, ids, stack,
           actions, rewards, terminals, out_states, out_next_states, out_actions, out_rewards,
           out_terminals);
  DQN_LAUNCH_CHECK("frame_sample_gather");
  return DQN_OK;
}
