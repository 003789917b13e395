// Weight gradient of the first (uint8-input) convolution on the tcgen05
// tensor cores, straight from the uint8 frames (layers.py:250-255; the
// pixel rule x = u8 / 255 of envs.py:300-311 applied once to the sums):
//
//   dW[r][co] = (sum_pix X_u8[pix][r] * dY[pix][co]) / 255,   r = (fy, fx, c)
//   db[co]    =  sum_pix dY[pix][co]
//
// One CTA per image, no im2col in HBM:
//   * the image (28,224 B for Atari) arrives in shared memory by one TMA bulk
//     copy (cp.async.bulk);
//   * dY of the image (400 x 32 fp32) is read once with coalesced float4
//     loads, transposed in registers and stored K-major (k = pixel) in the
//     canonical no-swizzle layout as two tf32 pieces stacked along N:
//     [dY_hi ; dY_lo] (hi = the value, which a kind::tf32 MMA truncates to 19
//     bits; lo = value - trunc(value)), with the bias sums taken on the way;
//   * A (the patch matrix, M = r, K = pixel) is built in TENSOR memory from
//     the image in shared memory: each thread owns one r (TMEM lane) and
//     writes 16 pixels per tcgen05.st -- uint8 values are exact in tf32, so
//     A is one piece and one MMA  A * [B_hi ; B_lo]  (N = 2 Cout) per 8-pixel
//     step gives hi and lo products side by side; 64-pixel blocks alternate
//     between two TMEM stages and two accumulator pairs (shorter accumulation
//     chains, summed in a fixed order in the epilogue);
//   * images are reduced deterministically: a thread-block cluster of up to 8
//     images sums its partials through distributed shared memory (rank j owns
//     rows j*R/8..), the cluster partials go to global scratch, and the last
//     cluster to finish a row slice (atomic ticket per slice) adds the
//     clusters in cluster order, divides by 255, accumulates into the
//     gradient and flags non-finite values (optim.py:38-40 semantics).
//
// Algorithmic traffic per launch (Atari, batch 32): frames 32 x 28,224 B +
// dY 32 x 51,200 B + dW/db read-modify-write 2 x 32.9 KB = 2.60 MB; the
// former path wrote and re-read a 3.28 MB transposed im2col (im2col_t).
#include "bulk_copy.cuh"
#include "tc_gemm.cuh"

namespace dqn {
namespace {

constexpr int kW1Threads = 512;

#ifdef DQN_TC_TRACE
// per-CTA %globaltimer marks (trace build only): entry, after pdl_wait, B
// built, image landed, MMAs done, epilogue staged, cluster reduced, exit
__device__ unsigned long long g_w1_trace[256 * 8];
__device__ int g_w1_skip;     // 1: no MMAs, 2: no A values (zeros), 4: no tcgen05.st
#define W1_SKIP(b) (g_w1_skip & (b))
#define W1_MARK(i)                                                          \
  if (threadIdx.x == 0 && blockIdx.x < 256) {                               \
    unsigned long long _t;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                  \
    g_w1_trace[blockIdx.x * 8 + (i)] = _t;                                  \
  }
#else
#define W1_MARK(i)
#define W1_SKIP(b) false
#endif

struct W1Args {
  const uint8_t *x;
  const float *dy;
  float *grad, *bias_grad;     // dW [R][N], db [N]
  float *gpart;                // [nclusters][R * N + N] cluster partials
  int *counters;               // [cl] slice tickets (zero between launches)
  int32_t *flags;
  int H, W, C, OH, OW, fw, sh, sw;
  int P, PS, PP, PP8, R, img_bytes, img_smem, cl, nclusters;   // PS units per image, PP pixels each
  int units;                   // batch * PS (image, pixel-range) units over the grid
};

__device__ __forceinline__ uint32_t w1_chunk(int RB, int row, int k) {
  return (uint32_t)((k >> 2) * (RB * 16) + (row >> 3) * 128 + (row & 7) * 16);
}

template <int N, int MT, int SWC>
__global__ void __launch_bounds__(kW1Threads, 1) conv1_wgrad_u8_kernel(const __grid_constant__ W1Args a) {
  constexpr int RB = 2 * N;                  // stacked B rows [hi ; lo]
  constexpr int ACC_COLS = 2 * MT * RB;      // two accumulator pairs per M-tile
  constexpr int A_COLS = 64;                 // pixels per block (8 MMA k-steps)
  constexpr uint32_t IDESC = tc::make_idesc_tf32(RB);
  constexpr int NQ = N / 4;                  // channel quads
  static_assert(ACC_COLS + 2 * MT * A_COLS <= 512, "TMEM budget");
  static_assert(kW1Threads % NQ == 0, "a thread keeps one channel quad");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t empty[2], done, imgbar;
  __shared__ uint32_t tmem_slot;
  __shared__ float bias_red[kW1Threads / NQ][N];
  __shared__ float bias_cta[N];
  __shared__ int gbase[128];                 // image byte offset of each 4-pixel group

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  W1_MARK(0)
  uint8_t *simg = smem;
  const uint32_t bbase = tc::smem_u32(smem + a.img_smem);
  float *stage = reinterpret_cast<float *>(smem + a.img_smem);   // aliases B after the MMAs

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 32) {
    tc::mbar_init(&empty[0], 1);
    tc::mbar_init(&empty[1], 1);
    tc::mbar_init(&done, 1);
    tc::mbar_init(&imgbar, 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_trigger();
  pdl_wait();                                // x and dY come from earlier kernels
  const uint32_t tmem = tmem_slot;
  W1_MARK(1)

  // warp w: TMEM lane quarter w % 4; its 4 sub-groups (w / 4) cover the MT x 4
  // 16-pixel slices of a 64-pixel block
  const int quarter = warp & 3, sub = warp >> 2;
  const int nkb = (a.PP8 + A_COLS - 1) / A_COLS;
  const int rowlen = a.fw * a.C;
  const int mw = (sub * MT) >> 2;            // this warp's M-tile (the same for its slices)
  const int r = mw * 128 + quarter * 32 + lane;
  const int fy = r / rowlen;
  const int roff = fy * a.W * a.C + (r - fy * rowlen);   // (fx, c) is r - fy * rowlen
  const int ngroups = a.PP / 4;
  const int q = t % NQ;
  float bs[4] = {0.f, 0.f, 0.f, 0.f};
  int g = 0;                                 // k-blocks issued by this CTA so far

  // units (image, pixel half) blockIdx.x, + gridDim.x, ...: every unit's
  // products accumulate into the same TMEM pairs (one partial per CTA)
  int it = 0;
  for (int unit = blockIdx.x; unit < a.units; unit += gridDim.x, ++it) {
    const int img = unit / a.PS, pbase = (unit % a.PS) * a.PP;
    if (it > 0) tc::mbar_wait(&done, (it - 1) & 1);     // the last unit's MMAs read B / A
    // pixels come in groups of 4 consecutive output columns (OW % 4 == 0):
    // group gg starts at output pixel pbase + 4 gg, its pixels SWC bytes apart
    for (int gg = t; gg < ngroups; gg += kW1Threads) {
      const int p = pbase + 4 * gg, oy = p / a.OW, ox = p - oy * a.OW;
      gbase[gg] = (oy * a.sh * a.W + ox * a.sw) * a.C;
    }
    if (t == 0) {
      tc::mbar_expect_tx(&imgbar, (uint32_t)a.img_bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(tc::smem_u32(simg)),
          "l"(a.x + (int64_t)img * a.img_bytes), "r"((uint32_t)a.img_bytes),
          "r"(tc::smem_u32(&imgbar))
          : "memory");
    }

    // ---- B = [dY_hi ; dY_lo], K-major over the unit's pixels (+ bias sums)
    {
      const float *dyi = a.dy + ((int64_t)img * a.P + pbase) * N + 4 * q;
      const int nu = (a.PP8 / 4) * NQ;
      for (int u = t; u < nu; u += kW1Threads) {
        const int pq = u / NQ, p0 = 4 * pq;
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (p0 + j < a.PP) {
            const float *src = dyi + (int64_t)(p0 + j) * N;
            asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v[j].x), "=f"(v[j].y), "=f"(v[j].z), "=f"(v[j].w)
                         : "l"(src));
          } else {
            v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        // channel 4q + i over pixels p0..p0+3; lanes rotate i so one store
        // instruction of the warp covers all 8 rows of a core matrix
        const int rot = pq & 3;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int i = (s + rot) & 3;
          const float4 c = i == 0 ? make_float4(v[0].x, v[1].x, v[2].x, v[3].x)
                           : i == 1 ? make_float4(v[0].y, v[1].y, v[2].y, v[3].y)
                           : i == 2 ? make_float4(v[0].z, v[1].z, v[2].z, v[3].z)
                                    : make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
          const int row = 4 * q + i;
          tc::st_shared_v4(bbase + w1_chunk(RB, row, p0), c);
          tc::st_shared_v4(bbase + w1_chunk(RB, N + row, p0),
                           make_float4(tc::tf32_lo(c.x), tc::tf32_lo(c.y), tc::tf32_lo(c.z),
                                       tc::tf32_lo(c.w)));
          bs[i] = __fadd_rn(bs[i], __fadd_rn(__fadd_rn(c.x, c.y), __fadd_rn(c.z, c.w)));
        }
      }
    }
    tc::fence_proxy_async();                 // B (generic stores) -> tensor-core reads
    __syncthreads();                         // gbase of this unit visible to every thread
    W1_MARK(2)
    tc::mbar_wait(&imgbar, it & 1);
    W1_MARK(3)

    // ---- A blocks in TMEM, MMAs
    for (int kb = 0; kb < nkb; ++kb, ++g) {
      const int s = g & 1;
      if (g >= 2) tc::mbar_wait(&empty[s], ((g - 2) >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const int slice = sub * MT + j, cs = slice & 3;
        const int g0 = (kb * A_COLS + cs * 16) / 4;
        float v[16];
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          if (!W1_SKIP(2) && g0 + gi < ngroups) {          // warp-uniform
            const uint8_t *src = simg + roff + gbase[g0 + gi];
#pragma unroll
            for (int i = 0; i < 4; ++i)    // exact uint8 -> fp32: (2^23 | b) - 2^23
              v[4 * gi + i] = __fsub_rn(__uint_as_float(0x4B000000u | src[i * SWC]), 8388608.f);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[4 * gi + i] = 0.f;
          }
        }
        if (!W1_SKIP(4))
          tc::tmem_st16(tmem + ((uint32_t)(quarter * 32) << 16) +
                            (uint32_t)(ACC_COLS + (s * MT + mw) * A_COLS + cs * 16), v);
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      __syncthreads();
      if (t == 0) {
        tc::tc_fence_after();
        const int nks = min(8, (a.PP8 - kb * A_COLS) / 8);
#pragma unroll 1
        for (int kq = 0; kq < (W1_SKIP(1) ? 0 : nks); ++kq) {
          const uint64_t bd = tc::make_sdesc(bbase + (uint32_t)((kb * 8 + kq) * 2 * RB * 16),
                                             RB * 16, 128);
#pragma unroll
          for (int m = 0; m < MT; ++m)
            tc::mma_ts(tmem + (uint32_t)(((g & 1) * MT + m) * RB),
                       tmem + (uint32_t)(ACC_COLS + (s * MT + m) * A_COLS + 8 * kq), bd, IDESC,
                       (g >= 2 || kq > 0) ? 1u : 0u);
        }
        tc::mma_commit(&empty[s]);
        if (kb == nkb - 1) tc::mma_commit(&done);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) bias_red[t / NQ][4 * q + i] = bs[i];
  tc::mbar_wait(&done, (it - 1) & 1);
  tc::tc_fence_after();
  W1_MARK(4)

  // ---- epilogue: this image's partial [R][N] into smem (B is dead)
  const int npair = g < 2 ? 1 : 2;
  constexpr int SLICES = MT * (N / 16);            // (M-tile, 16-channel group)
  for (int sl = sub; sl < SLICES; sl += 4) {
    const int m = sl / (N / 16), c0 = (sl % (N / 16)) * 16;
    const int r = m * 128 + quarter * 32 + lane;
    float lo[16], hi[16], tmp[16];
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    tc::tmem_ld16(lane_base + (uint32_t)(m * RB + N + c0), lo);
    tc::tmem_ld16(lane_base + (uint32_t)(m * RB + c0), hi);
    if (npair > 1) {
      tc::tmem_ld16(lane_base + (uint32_t)((MT + m) * RB + N + c0), tmp);
#pragma unroll
      for (int i = 0; i < 16; ++i) lo[i] = __fadd_rn(lo[i], tmp[i]);
      tc::tmem_ld16(lane_base + (uint32_t)((MT + m) * RB + c0), tmp);
#pragma unroll
      for (int i = 0; i < 16; ++i) hi[i] = __fadd_rn(hi[i], tmp[i]);
    }
    if (r < a.R) {
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4 *>(&stage[r * N + c0 + i]) =
            make_float4(__fadd_rn(lo[i], hi[i]), __fadd_rn(lo[i + 1], hi[i + 1]),
                        __fadd_rn(lo[i + 2], hi[i + 2]), __fadd_rn(lo[i + 3], hi[i + 3]));
    }
  }
  __syncthreads();
  if (t < N) {
    float s = bias_red[0][t];
    for (int g = 1; g < kW1Threads / NQ; ++g) s = __fadd_rn(s, bias_red[g][t]);
    bias_cta[t] = s;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");

  // ---- cluster reduction: rank j sums rows [j R / cl, ...) over the ranks in order
  const int cl = a.cl, rank = blockIdx.x % cl, cid = blockIdx.x / cl;
  const int rows = a.R / cl, r0 = rank * rows;
  float *gp = a.gpart + (int64_t)cid * (a.R * N + N);
  W1_MARK(5)
  if (cl > 1) tc::cluster_sync();
  for (int idx = t; idx < rows * NQ; idx += kW1Threads) {
    const int rr = r0 + idx / NQ, c4 = (idx % NQ) * 4;
    float4 acc;
    if (cl > 1) {
      const uint32_t la = tc::smem_u32(&stage[rr * N + c4]);
      float4 v[8];
#pragma unroll
      for (int qq = 0; qq < 8; ++qq)         // all loads in flight, then the ordered sum
        if (qq < cl) v[qq] = tc::ld_dsmem4(tc::dsmem_addr(la, qq));
      acc = v[0];
#pragma unroll
      for (int qq = 1; qq < 8; ++qq)
        if (qq < cl) {
          acc.x = __fadd_rn(acc.x, v[qq].x); acc.y = __fadd_rn(acc.y, v[qq].y);
          acc.z = __fadd_rn(acc.z, v[qq].z); acc.w = __fadd_rn(acc.w, v[qq].w);
        }
    } else {
      acc = *reinterpret_cast<const float4 *>(&stage[rr * N + c4]);
    }
    *reinterpret_cast<float4 *>(gp + rr * N + c4) = acc;
  }
  if (rank == 0 && t < N) {
    float s = bias_cta[t];
    if (cl > 1) {
      const uint32_t la = tc::smem_u32(&bias_cta[t]);
      s = tc::ld_dsmem(tc::dsmem_addr(la, 0));
      for (int qq = 1; qq < cl; ++qq) s = __fadd_rn(s, tc::ld_dsmem(tc::dsmem_addr(la, qq)));
    }
    gp[a.R * N + t] = s;
  }
  if (cl > 1) tc::cluster_sync();            // peers' smem no longer read
  W1_MARK(6)

  // ---- across clusters: the last cluster to finish slice `rank` adds them in order
  __shared__ int s_ticket;
  __threadfence();
  __syncthreads();
  if (t == 0) s_ticket = atomicAdd(&a.counters[rank], 1);
  __syncthreads();
  W1_MARK(7)
  if (s_ticket != a.nclusters - 1) return;
  __threadfence();
  const int64_t cstride = (int64_t)a.R * N + N;
  for (int idx = t; idx < rows * NQ; idx += kW1Threads) {
    const int rr = r0 + idx / NQ, c4 = (idx % NQ) * 4;
    const float *src = a.gpart + rr * N + c4;
    float4 acc = __ldcg(reinterpret_cast<const float4 *>(src));
    for (int c0 = 1; c0 < a.nclusters; c0 += 8) {
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)            // 8 loads in flight, summed in cluster order
        if (c0 + j < a.nclusters) v[j] = __ldcg(reinterpret_cast<const float4 *>(src + (c0 + j) * cstride));
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + j < a.nclusters) {
          acc.x = __fadd_rn(acc.x, v[j].x); acc.y = __fadd_rn(acc.y, v[j].y);
          acc.z = __fadd_rn(acc.z, v[j].z); acc.w = __fadd_rn(acc.w, v[j].w);
        }
    }
    float *g = a.grad + rr * N + c4;
    float4 o = *reinterpret_cast<float4 *>(g);
    o.x = __fadd_rn(o.x, __fdiv_rn(acc.x, 255.0f));
    o.y = __fadd_rn(o.y, __fdiv_rn(acc.y, 255.0f));
    o.z = __fadd_rn(o.z, __fdiv_rn(acc.z, 255.0f));
    o.w = __fadd_rn(o.w, __fdiv_rn(acc.w, 255.0f));
    *reinterpret_cast<float4 *>(g) = o;
    note_grad4(a.flags, o);
  }
  if (rank == 0 && t < N) {
    float s = __ldcg(a.gpart + a.R * N + t);
    for (int c = 1; c < a.nclusters; ++c) s = __fadd_rn(s, __ldcg(a.gpart + c * cstride + a.R * N + t));
    acc_grad(a.bias_grad + t, s, a.flags);
  }
  if (t == 0) a.counters[rank] = 0;          // next launch (graph replay) starts from zero
}

template <int N, int MT, int SWC>
int launch_w1(cudaStream_t st, const W1Args &a, int smem) {
  auto kern = conv1_wgrad_u8_kernel<N, MT, SWC>;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "conv1_wgrad_u8");
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.cl * a.nclusters);
  cfg.blockDim = dim3(kW1Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  attr[2].id = cudaLaunchAttributeClusterDimension;
  attr[2].val.clusterDim.x = a.cl;
  attr[2].val.clusterDim.y = 1;
  attr[2].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 3;
  cudaLaunchKernelEx(&cfg, kern, a);
  DQN_LAUNCH_CHECK("conv1_wgrad_u8");
  return DQN_OK;
}

inline int w1_smem(const dqn_layer_desc &L, int P8, int &img_smem) {
  const int img = L.in_h * L.in_w * L.in_c;
  img_smem = (img + 127) / 128 * 128;
  const int b = 2 * L.out_c * P8 * 4;
  const int stage = L.fh * L.fw * L.in_c * L.out_c * 4;
  return img_smem + (b > stage ? b : stage);
}

}  // namespace

// CTAs per image: two half-images when the halves are whole 8-pixel MMA steps
// (measured in the learner's graph, Atari batch 32: 1 / 2 / 4 CTAs per image
// -> 2 best; 4 doubles the cross-cluster partials)
inline int w1_splits(int P) { return P % 16 == 0 && P / 2 <= 512 ? 2 : 1; }

// Is layer 0 a uint8 convolution this kernel takes (Atari: 8x8x4 -> 32,
// 16-byte pixel step, 20 output columns)?
bool conv1_wgrad_u8_ok(const dqn_net_desc *net) {
  if (!net->input_u8 || net->n_layers < 1 || net->algo == 1) return false;
  const dqn_layer_desc &L = net->layer[0];
  if (L.kind != DQN_LAYER_CONV) return false;
  const int R = L.fh * L.fw * L.in_c, P = L.out_h * L.out_w;
  if (R % 128 || R > 256 || !(L.out_c == 16 || L.out_c == 32)) return false;
  if ((L.in_h * L.in_w * L.in_c) % 16 || L.out_w % 4 || L.sw * L.in_c != 16) return false;
  const int PP = P / w1_splits(P);
  if (PP > 512) return false;
  int img_smem;
  return w1_smem(L, (PP + 7) / 8 * 8, img_smem) <= 200 * 1024;
}

#ifdef DQN_TC_TRACE
int g_w1_cl_max = 8;   // diagnostic: largest cluster
#else
constexpr int g_w1_cl_max = 8;
#endif

int64_t conv1_wgrad_u8_scratch(const dqn_net_desc *net, int batch) {
  const dqn_layer_desc &L = net->layer[0];
  const int R = L.fh * L.fw * L.in_c;
  // at most one partial per CTA
  return (int64_t)batch * w1_splits(L.out_h * L.out_w) * (R * L.out_c + L.out_c);
}

int conv1_wgrad_u8_tc(cudaStream_t st, const dqn_net_desc *net, const uint8_t *x,
                      const float *dy, float *grads, float *scratch, int *counters, int batch,
                      int32_t *flags) {
  if (!conv1_wgrad_u8_ok(net) || batch < 1 || ((uintptr_t)x % 16) || ((uintptr_t)dy % 16))
    return DQN_ERR_UNSUPPORTED;
  const dqn_layer_desc &L = net->layer[0];
  W1Args a{};
  a.x = x;
  a.dy = dy;
  a.grad = grads + L.w_off;
  a.bias_grad = grads + L.b_off;
  a.gpart = scratch;
  a.counters = counters;
  a.flags = flags;
  a.H = L.in_h; a.W = L.in_w; a.C = L.in_c;
  a.OH = L.out_h; a.OW = L.out_w; a.fw = L.fw; a.sh = L.sh; a.sw = L.sw;
  a.P = L.out_h * L.out_w;
  a.PS = w1_splits(a.P);
  a.PP = a.P / a.PS;
  a.PP8 = (a.PP + 7) / 8 * 8;
  a.R = L.fh * L.fw * L.in_c;
  a.img_bytes = L.in_h * L.in_w * L.in_c;
  a.units = batch * a.PS;
  // one CTA per unit up to 128 CTAs (learner batches); larger batches loop
  // over units inside the CTA, so the cross-CTA reduction stays <= 128 partials
  const int ctas = a.units <= 128 ? a.units : 128;
  a.cl = 1;
  for (int c : {8, 4, 2})                   // 8-CTA clusters measured best (vs 1, 2, 4)
    if (c <= g_w1_cl_max && ctas % c == 0 && a.R % c == 0) { a.cl = c; break; }
  a.nclusters = ctas / a.cl;
  const int smem = w1_smem(L, a.PP8, a.img_smem);
  const int MT = a.R / 128;
  if (L.out_c == 32)
    return MT == 2 ? launch_w1<32, 2, 16>(st, a, smem) : launch_w1<32, 1, 16>(st, a, smem);
  return MT == 2 ? launch_w1<16, 2, 16>(st, a, smem) : launch_w1<16, 1, 16>(st, a, smem);
}

}  // namespace dqn

#ifdef DQN_TC_TRACE
extern "C" void dqn_w1_skip(int m) { cudaMemcpyToSymbol(dqn::g_w1_skip, &m, sizeof(m)); }
extern "C" void dqn_w1_set_cluster_max(int c) { dqn::g_w1_cl_max = c; }
extern "C" int dqn_w1_trace(unsigned long long *host) {
  return (int)cudaMemcpyFromSymbol(host, dqn::g_w1_trace, sizeof(dqn::g_w1_trace));
}
#endif
