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

namespace dqn {
namespace {

constexpr int kFgThreads = 256;

// grid (k, 2): blockIdx.y 0 = state stack, 1 = next-state stack
__global__ void __launch_bounds__(kFgThreads)
frame_gather_kernel(const uint8_t *__restrict__ frames, int64_t frame_bytes,
                    const int64_t *ids, int S, const int64_t *idx, const int64_t *actions,
                    const double *rewards, const bool *terms, uint8_t *__restrict__ out_s,
                    uint8_t *__restrict__ out_n, int64_t *__restrict__ out_a,
                    double *__restrict__ out_r, bool *__restrict__ out_t) {
  // no __restrict__ on idx / ids / metadata: with it the compiler may hoist
  // their loads above the PDL wait (tools/pdl_hoist_scan.py) and read
  // indices the previous kernel is still writing
  pdl_begin();
  const int j = blockIdx.x, which = blockIdx.y;
  const int64_t slot = idx[j];
  const int64_t *row = ids + slot * 2 * S + which * S;
  uint8_t *dst = (which ? out_n : out_s) + (int64_t)j * frame_bytes * S;
  if (which == 0 && threadIdx.x == 0) {
    if (out_a) out_a[j] = actions[slot];
    if (out_r) out_r[j] = rewards[slot];
    if (out_t) out_t[j] = terms[slot];
  }
  if (S == 4 && frame_bytes % 16 == 0) {
    // 16 pixels of each plane per thread: one 16-byte load per plane, four
    // 16-byte stores of interleaved pixels (4x the bytes in flight of the
    // u32 path below)
    const uint4 *p0 = reinterpret_cast<const uint4 *>(frames + row[0] * frame_bytes);
    const uint4 *p1 = reinterpret_cast<const uint4 *>(frames + row[1] * frame_bytes);
    const uint4 *p2 = reinterpret_cast<const uint4 *>(frames + row[2] * frame_bytes);
    const uint4 *p3 = reinterpret_cast<const uint4 *>(frames + row[3] * frame_bytes);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    for (int64_t q = threadIdx.x; q < frame_bytes / 16; q += blockDim.x) {
      const uint4 A = __ldg(p0 + q), B = __ldg(p1 + q), C = __ldg(p2 + q), D = __ldg(p3 + q);
      const uint32_t a[4] = {A.x, A.y, A.z, A.w}, b[4] = {B.x, B.y, B.z, B.w},
                     c[4] = {C.x, C.y, C.z, C.w}, d[4] = {D.x, D.y, D.z, D.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t ab_lo = __byte_perm(a[u], b[u], 0x5140), cd_lo = __byte_perm(c[u], d[u], 0x5140);
        const uint32_t ab_hi = __byte_perm(a[u], b[u], 0x7362), cd_hi = __byte_perm(c[u], d[u], 0x7362);
        o[4 * q + u] = make_uint4(__byte_perm(ab_lo, cd_lo, 0x5410), __byte_perm(ab_lo, cd_lo, 0x7632),
                                  __byte_perm(ab_hi, cd_hi, 0x5410), __byte_perm(ab_hi, cd_hi, 0x7632));
      }
    }
  } else if (S == 4 && frame_bytes % 4 == 0) {
    // 4 pixels of each plane per thread: one u32 per plane in, the four
    // interleaved pixels (a_i b_i c_i d_i) as one 16-byte store out
    const uint32_t *p0 = reinterpret_cast<const uint32_t *>(frames + row[0] * frame_bytes);
    const uint32_t *p1 = reinterpret_cast<const uint32_t *>(frames + row[1] * frame_bytes);
    const uint32_t *p2 = reinterpret_cast<const uint32_t *>(frames + row[2] * frame_bytes);
    const uint32_t *p3 = reinterpret_cast<const uint32_t *>(frames + row[3] * frame_bytes);
    uint4 *o = reinterpret_cast<uint4 *>(dst);
    for (int64_t q = threadIdx.x; q < frame_bytes / 4; q += blockDim.x) {
      const uint32_t a = __ldg(p0 + q), b = __ldg(p1 + q), c = __ldg(p2 + q), d = __ldg(p3 + q);
      const uint32_t ab_lo = __byte_perm(a, b, 0x5140), cd_lo = __byte_perm(c, d, 0x5140);
      const uint32_t ab_hi = __byte_perm(a, b, 0x7362), cd_hi = __byte_perm(c, d, 0x7362);
      o[q] = make_uint4(__byte_perm(ab_lo, cd_lo, 0x5410), __byte_perm(ab_lo, cd_lo, 0x7632),
                        __byte_perm(ab_hi, cd_hi, 0x5410), __byte_perm(ab_hi, cd_hi, 0x7632));
    }
  } else {
    for (int64_t p = threadIdx.x; p < frame_bytes; p += blockDim.x)
      for (int s = 0; s < S; ++s) dst[p * S + s] = frames[row[s] * frame_bytes + p];
  }
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
  launch_k(frame_gather_kernel, dim3(k, 2), kFgThreads, 0, as_stream(stream), frames,
           frame_bytes, ids, stack, indices, actions, rewards, terminals, out_states,
           out_next_states, out_actions, out_rewards, out_terminals);
  DQN_LAUNCH_CHECK("frame_gather");
  return DQN_OK;
}
