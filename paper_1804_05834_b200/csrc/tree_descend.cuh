// SumTree.find descent shared by the replay and data-parallel kernels.
#pragma once
#include "common.cuh"

namespace dqn {

static __device__ __forceinline__ double sel2(double a, double b, int i) { return i ? b : a; }
static __device__ __forceinline__ double sel4(const double (&v)[4], int i) {
  return (i & 2) ? sel2(v[2], v[3], i & 1) : sel2(v[0], v[1], i & 1);
}
static __device__ __forceinline__ double sel8(const double (&v)[8], int i) {
  return (i & 4) ? ((i & 2) ? sel2(v[6], v[7], i & 1) : sel2(v[4], v[5], i & 1))
                 : ((i & 2) ? sel2(v[2], v[3], i & 1) : sel2(v[0], v[1], i & 1));
}

// SumTree.find descent for one query mass (replay.py:172-181).  Returns the
// leaf index; *leaf_value (optional) receives nodes[leaf].
//
// Four levels per dependent round trip: the left-child sums of the next four
// levels below node n are nodes[2n], nodes[4n + {0,2}], nodes[8n + {0,2,4,6}]
// and nodes[16n + {0,2,..,14}] -- four short contiguous runs -- so all 15 are
// loaded together and the four compare/subtract steps then run exactly as the
// reference's per-level loop (same operations, same order).  The last group
// also loads the right children, which yields the leaf value for free.
// tree_descend_from: the same from node n at level l with remaining mass q
// (already clipped) -- the tail of a descent whose top levels ran elsewhere
// (the shared-memory staged sampler).
static __device__ __forceinline__ int64_t tree_descend_from(const double *__restrict__ nodes,
                                                            int depth, int64_t n, int l, double q,
                                                            double *leaf_value = nullptr) {
  double leaf = -1.0;
  for (; l + 4 <= depth; l += 4) {
    const bool last = l + 4 == depth;
    const double c1 = __ldg(nodes + 2 * n);
    double c2[2], c3[4], c4[8], c4r[8];
#pragma unroll
    for (int i = 0; i < 2; ++i) c2[i] = __ldg(nodes + 4 * n + 2 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i) c3[i] = __ldg(nodes + 8 * n + 2 * i);
#pragma unroll
    for (int i = 0; i < 8; ++i) c4[i] = __ldg(nodes + 16 * n + 2 * i);
    if (last && leaf_value) {
#pragma unroll
      for (int i = 0; i < 8; ++i) c4r[i] = __ldg(nodes + 16 * n + 2 * i + 1);
    }
    const bool r1 = q > c1;
    if (r1) q = __dsub_rn(q, c1);                 // q -= left_sum * go_right
    const int i1 = r1 ? 1 : 0;
    const double l2 = sel2(c2[0], c2[1], i1);
    const bool r2 = q > l2;
    if (r2) q = __dsub_rn(q, l2);
    const int i2 = 2 * i1 + (r2 ? 1 : 0);
    const double l3 = sel4(c3, i2);
    const bool r3 = q > l3;
    if (r3) q = __dsub_rn(q, l3);
    const int i3 = 2 * i2 + (r3 ? 1 : 0);
    const double l4 = sel8(c4, i3);
    const bool r4 = q > l4;
    if (r4) q = __dsub_rn(q, l4);
    n = 16 * n + 2 * i3 + (r4 ? 1 : 0);
    if (last && leaf_value) leaf = r4 ? sel8(c4r, i3) : l4;
  }
  // remaining levels: two per round trip, then one
  for (; l + 2 <= depth; l += 2) {
    const double ls = __ldg(nodes + 2 * n);               // nodes[2n]
    const double lls = __ldg(nodes + 4 * n);              // nodes[4n]   (left-left)
    const double rls = __ldg(nodes + 4 * n + 2);          // nodes[4n+2] (right-left)
    const bool r1 = q > ls;
    if (r1) q = __dsub_rn(q, ls);
    const int64_t c = 2 * n + (r1 ? 1 : 0);
    const double ls2 = r1 ? rls : lls;
    const bool r2 = q > ls2;
    if (r2) q = __dsub_rn(q, ls2);
    n = 2 * c + (r2 ? 1 : 0);
  }
  for (; l < depth; ++l) {
    const int64_t left = n << 1;
    const double ls = __ldg(nodes + left);
    const bool right = q > ls;
    if (right) q = __dsub_rn(q, ls);          // q -= left_sum * go_right
    n = left + (right ? 1 : 0);
  }
  if (leaf_value) *leaf_value = leaf >= 0.0 ? leaf : __ldg(nodes + n);
  return n - (int64_t(1) << depth);
}

static __device__ __forceinline__ int64_t tree_descend(const double *__restrict__ nodes, int depth,
                                                double q, double hi,
                                                double *leaf_value = nullptr) {
  q = fmin(fmax(q, 1e-300), hi);            // np.clip(q, 1e-300, nextafter(total, 0))
  return tree_descend_from(nodes, depth, 1, 0, q, leaf_value);
}


// The same descent by one full warp, eight levels per dependent round trip:
// the 2 + 4 + ... + 256 nodes of the eight levels below the current node are
// loaded by the 32 lanes at once (level l's node o sits in lane o % 32, slot
// o / 32), then the eight compare / subtract steps run exactly as above with
// each left-child sum taken from its lane by a shuffle.  Every lane returns
// the leaf index; *leaf_value gets nodes[leaf].
static __device__ __forceinline__ double wsel(const double *r, int slot) {
  double v = r[0];
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (slot == i) v = r[i];
  return v;
}

static __device__ __forceinline__ int64_t warp_tree_descend(const double *__restrict__ nodes,
                                                            int depth, double q, double hi,
                                                            double *leaf_value = nullptr) {
  const int lane = threadIdx.x & 31;
  q = fmin(fmax(q, 1e-300), hi);
  int64_t n = 1;
  int l = 0;
  double leaf = 0.0;
  while (l < depth) {
    const int G = depth - l < 8 ? depth - l : 8;
    // r[g][s]: node (n << (g + 1)) + 32 s + lane of level g + 1 below n
    double r[8][8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
#pragma unroll
      for (int sl = 0; sl < 8; ++sl) {
        const int cnt = 2 << g;                       // nodes at this level
        const int o = 32 * sl + lane;
        r[g][sl] = (g < G && o < cnt) ? __ldg(nodes + (n << (g + 1)) + o) : 0.0;
      }
    }
    int64_t p = 0;                                    // offset inside the level
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (g >= G) break;
      const int o = (int)(2 * p);                     // left child of the path node
      const double mine = wsel(r[g], o >> 5);
      const double ls = __shfl_sync(0xffffffffu, mine, o & 31);
      const bool right = q > ls;
      if (right) q = __dsub_rn(q, ls);
      p = 2 * p + (right ? 1 : 0);
      if (g == G - 1 && leaf_value) {
        const int ol = (int)p;
        leaf = __shfl_sync(0xffffffffu, wsel(r[g], ol >> 5), ol & 31);
      }
    }
    n = (n << G) + p;
    l += G;
  }
  if (leaf_value) *leaf_value = leaf;
  return n - (int64_t(1) << depth);
}

// The IS-weights CTA of the fused sample+gather kernels (replay.py:215-230):
// descends all k stratified queries, writes idx / P / w and normalises w by
// the batch max (block-wide reduce; red holds blockDim.x / 32 doubles).
static __device__ __forceinline__ void sample_is_weights_block(
    const double *nodes, int depth, const int64_t *size_p, const double *u, int k,
    const double *beta_p, int64_t *idx, double *prob, double *weight, int32_t *flags,
    double *red) {
  const double total = nodes[1];
  const bool ok = total > 0.0;
  double mx = 0.0;
  const double beta = *beta_p, size = (double)*size_p, seg = __ddiv_rn(total, (double)k);
  const double hi = nextafter(total, 0.0);
  for (int q = threadIdx.x; q < k; q += blockDim.x) {
    if (!ok) {
      idx[q] = 0; prob[q] = 0.0; weight[q] = 0.0;
      continue;
    }
    double leaf;
    const int64_t i = tree_descend(nodes, depth, __dmul_rn(__dadd_rn((double)q, u[q]), seg), hi,
                                   &leaf);
    const double p = __ddiv_rn(leaf, total);
    const double w = pow(__dmul_rn(size, p), -beta);
    idx[q] = i;
    prob[q] = p;
    weight[q] = w;
    mx = fmax(mx, w);
  }
  if (!ok) {
    if (threadIdx.x == 0) raise_flag(flags, DQN_FLAG_ZERO_TOTAL);
    return;
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    red[0] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < k; q += blockDim.x) weight[q] = __ddiv_rn(weight[q], red[0]);
}

}  // namespace dqn
