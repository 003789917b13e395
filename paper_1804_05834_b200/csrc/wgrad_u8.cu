// Weight gradient of the first (uint8-input) convolution on the tcgen05
// tensor cores, straight from the uint8 frames (layers.py:250-255; the
// pixel rule x = u8 / 255 of envs.py:300-311 applied once to the sums):
//
//   dW[r][co] = (sum_pix X_u8[pix][r] * dY[pix][co]) / 255,   r = (fy, fx, c)
//   db[co]    =  sum_pix dY[pix][co]
//
// One CTA per unit (image or pixel range of one: Atari, half an image = 200
// output pixels), 512 threads per 128-row M-tile of r (Atari R = 256: 1024
// threads), no im2col in HBM:
//   * the image (28,224 B for Atari) arrives in shared memory by one TMA bulk
//     copy (cp.async.bulk);
//   * dY of the unit (200 x 32 fp32) is read once with coalesced float4
//     loads, transposed in registers and stored K-major (k = pixel) in the
//     canonical no-swizzle layout as two tf32 pieces stacked along N:
//     [dY_hi ; dY_lo] (hi = the value, which a kind::tf32 MMA truncates to 19
//     bits; lo = value - trunc(value)), with the bias sums taken on the way;
//   * A (the patch matrix, M = 128 values of r per M-tile, K = pixel) is built
//     whole from the image before any MMA -- its first 192 pixels in TENSOR
//     memory beside the M-tile's accumulator (64 + 192 = 256 columns per
//     M-tile), the rest (Atari: 8 pixels) as K-major chunks in shared memory
//     -- so nothing waits on the tensor core and no TMEM slot is recycled.
//     uint8 values are exact in tf32, so A is one piece and one MMA
//     A * [B_hi ; B_lo] (N = 2 Cout) per 8-pixel step gives hi and lo
//     products side by side; one thread issues both M-tiles' MMAs with every
//     address in registers (the issue loop, ~100 cycles per MMA, is the
//     kernel's longest phase);
//   * partials are reduced deterministically: each CTA sends the rows of its
//     partial that rank k of its (4-CTA) cluster owns straight from TMEM
//     registers into that rank's shared memory (st.async, counted on the
//     owner's mbarrier: no cluster barrier around the exchange); the owner
//     adds them in rank order and writes the cluster partial to global
//     scratch; the last cluster to finish a row slice (atomic ticket per
//     slice) adds the clusters in a fixed order, divides by 255, accumulates
//     into the gradient and flags non-finite values (optim.py:38-40
//     semantics).
//
// 64 CTAs at Atari batch 32 (2 units per image): the kernel runs beside the
// conv2 wgrad, whose cluster split-K needs whole free SMs in a GPC; 96 or 192
// CTAs of a finer split were faster alone but starved it.
//
// Algorithmic traffic per launch (Atari, batch 32): frames 32 x 28,224 B +
// dY 32 x 51,200 B + dW/db read-modify-write 2 x 32.9 KB = 2.60 MB; the
// former path wrote and re-read a 3.28 MB transposed im2col (im2col_t).
#include "bulk_copy.cuh"
#include "tc_gemm.cuh"

namespace dqn {
namespace {

#ifdef DQN_TC_TRACE
// per-CTA %globaltimer marks (trace build only): entry, after pdl_wait, B
// built, image landed, MMAs done, partial sent, cluster partial written,
// ticket, cross-cluster sum done (last cluster only), MMA issue start / end
__device__ unsigned long long g_w1_trace[256 * 12];
__device__ int g_w1_skip;     // 1: no MMAs, 2: no A values (zeros), 4: no tcgen05.st
#define W1_SKIP(b) (w1_skip & (b))   // w1_skip: g_w1_skip read once per CTA
#define W1_SKIP_LOAD const int w1_skip = g_w1_skip;
#define W1_MARK(i)                                                          \
  if (threadIdx.x == 0 && blockIdx.x < 256) {                               \
    unsigned long long _t;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                  \
    g_w1_trace[blockIdx.x * 12 + (i)] = _t;                                  \
  }
#else
#define W1_MARK(i)
#define W1_SKIP(b) false
#define W1_SKIP_LOAD
#endif

struct W1Args {
  const uint8_t *x;
  const float *dy;
  float *grad, *bias_grad;     // dW [R][N], db [N]
  float *gpart;                // [ncl][R * N + N] cluster partials
  int *counters;               // [cl] slice tickets (zero between launches)
  int32_t *flags;
  int H, W, C, OH, OW, fw, sh, sw;
  int P, PS, PP, R, img_bytes, img_smem, cl, ncl;   // PS units per image, PP pixels each (the last: the rest)
  int units;                   // batch * PS (image, pixel-range) units
  int recv_off;                // smem byte offset of the receive slots [cl][R / cl][N] + bias [cl][N]
  int tail_off, tail_bytes;    // A past kW1TmemPix pixels: [MT][128 x (PP - kW1TmemPix)] fp32
  int cpm;                     // CTAs (= cl * ncl)
};

// 16-byte chunk (row, 4 consecutive k) of the K-major no-swizzle B operand
// with RB rows: core matrices of 8 rows x 16 B, k-chunks RB * 16 B apart
__device__ __forceinline__ uint32_t w1_chunk(int RB, int row, int k) {
  return (uint32_t)((k >> 2) * (RB * 16) + (row >> 3) * 128 + (row & 7) * 16);
}

// A pixels per M-tile held in TMEM (beside the 64-column accumulator, 256
// columns per M-tile); a unit's further pixels (<= 64) are read from smem
constexpr int kW1TmemPix = 192;
constexpr int kW1MaxPix = kW1TmemPix + 64;

__device__ __forceinline__ void w1_mma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// split cluster barrier: arrive early (after the receive barrier's init),
// wait just before the first store into a peer
__device__ __forceinline__ void cluster_arrive_() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16 / 4 bytes into a (possibly remote) CTA's shared memory, counted on its mbarrier
__device__ __forceinline__ void st_async4(uint32_t addr, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async1(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];"
               ::"r"(addr), "f"(v), "r"(bar)
               : "memory");
}

template <int N, int MT, int SWC>
__global__ void __launch_bounds__(512 * MT, 1) conv1_wgrad_u8_kernel(const __grid_constant__ W1Args a) {
  constexpr int T = 512 * MT;                // 16 warps per 128-row M-tile of r
  constexpr int R = 128 * MT;
  constexpr int RB = 2 * N;                  // stacked B rows [hi ; lo]; accumulator columns
  constexpr int A_COL = RB;                  // A (K = the unit's pixels) after the accumulator
  constexpr uint32_t IDESC = tc::make_idesc_tf32(RB);
  constexpr int NQ = N / 4;                  // channel quads
  static_assert(T % NQ == 0, "a thread keeps one channel quad");
  static_assert((T / NQ) % 8 == 0 && 8 * N <= T, "bias sums in 8 parts");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done, imgbar, recv;
  __shared__ uint32_t tmem_slot;
  __shared__ float bias_red[T / NQ][N];
  __shared__ int gbase[128];                 // image byte offset of each 4-pixel group

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  W1_MARK(0)
  W1_SKIP_LOAD
  const int cl = a.cl, rank = blockIdx.x % cl, cid = blockIdx.x / cl;
  const int rows = R / cl, r0 = rank * rows;   // rows of dW this rank reduces
  uint8_t *simg = smem;
  const uint32_t bbase = tc::smem_u32(smem + a.img_smem);
  const uint32_t rbase = tc::smem_u32(smem + a.recv_off);
  const uint32_t tbase = tc::smem_u32(smem + a.tail_off);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(256 * MT)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 32) {
    tc::mbar_init(&done, 1);
    tc::mbar_init(&imgbar, 1);
    tc::mbar_init(&recv, 1);
    // every rank sends this CTA its rows (rows x N floats each); rank 0 also
    // receives the ranks' bias sums
    tc::mbar_expect_tx(&recv, (uint32_t)((R * N + (rank == 0 ? cl * N : 0)) * 4));
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (cl > 1) cluster_arrive_();
  pdl_trigger();
  pdl_wait();                                // x and dY come from earlier kernels
  W1_MARK(1)

  // warp w: M-tile h = w / 16 (its own 256 TMEM columns), TMEM lane quarter
  // w % 4 (A rows = 32 values of r), 16-pixel column chunks (w % 16) / 4 + 4 i
  const int h = warp >> 4, quarter = warp & 3, sub = (warp >> 2) & 3;
  const int rowlen = a.fw * a.C;
  const int r = h * 128 + quarter * 32 + lane;
  const int fy = r / rowlen;
  const int roff = fy * a.W * a.C + (r - fy * rowlen);   // (fx, c) is r - fy * rowlen
  const int q = t % NQ;
  const uint32_t tmem0 = tmem_slot;
  const uint32_t tmem = tmem0 + (uint32_t)(h * 256);
  const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
  float bs[4] = {0.f, 0.f, 0.f, 0.f};

  // units (image, pixel range) blockIdx.x, + gridDim.x, ...: every unit's
  // products accumulate into the same TMEM accumulators (one partial per CTA)
  int it = 0;
  for (int unit = blockIdx.x; unit < a.units; unit += gridDim.x, ++it) {
    const int img = unit / a.PS, pbase = (unit % a.PS) * a.PP;
    const int len = min(a.PP, a.P - pbase), len8 = (len + 7) & ~7, ngroups = len / 4;
    // (the last unit's A build is done -- its CTA barrier -- so gbase and the
    // image buffer are free; its MMAs may still read B and A: waited for
    // below, after this unit's dY loads are in flight)
    // pixels come in groups of 4 consecutive output columns (OW % 4 == 0):
    // group gg starts at output pixel pbase + 4 gg, its pixels SWC bytes apart
    for (int gg = t; gg < ngroups; gg += T) {
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
      const int nu = (len8 / 4) * NQ;
      for (int u = t; u < nu; u += T) {
        const int pq = u / NQ, p0 = 4 * pq;
        float4 v[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          if (p0 + jj < len) {
            const float *src = dyi + (int64_t)(p0 + jj) * N;
            asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v[jj].x), "=f"(v[jj].y), "=f"(v[jj].z), "=f"(v[jj].w)
                         : "l"(src));
          } else {
            v[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        if (it > 0 && u == t) tc::mbar_wait(&done, (it - 1) & 1);   // the last unit's MMAs
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
      if (it > 0 && t >= nu) tc::mbar_wait(&done, (it - 1) & 1);
    }
    tc::fence_proxy_async();                 // B (generic stores) -> tensor-core reads
    __syncthreads();                         // gbase of this unit visible to every thread
    W1_MARK(2)
    tc::mbar_wait(&imgbar, it & 1);
    W1_MARK(3)

    // ---- the whole unit's A: its first kW1TmemPix pixels in TMEM, the rest
    // (Atari: the last 8) in shared memory; nothing waits on the tensor core
    tc::tc_fence_after();
    const int tlen = min(len8, kW1TmemPix);
    for (int ch = sub; ch * 16 < tlen; ch += 4) {
      float v[16];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        const int gg = ch * 4 + gi;
        if (!W1_SKIP(2) && gg < ngroups) {                 // warp-uniform
          const uint8_t *src = simg + roff + gbase[gg];
#pragma unroll
          for (int i = 0; i < 4; ++i)    // exact uint8 -> fp32: (2^23 | b) - 2^23
            v[4 * gi + i] = __fsub_rn(__uint_as_float(0x4B000000u | src[i * SWC]), 8388608.f);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) v[4 * gi + i] = 0.f;
        }
      }
      if (!W1_SKIP(4)) tc::tmem_st16(lane_base + (uint32_t)(A_COL + ch * 16), v);
    }
    if (len8 > kW1TmemPix) {
      // tail chunk (M-tile hh, row, pixels 4 ck..4 ck + 3 past kW1TmemPix), K-major
      const int nck = (len8 - kW1TmemPix) / 4;
      for (int idx = t; idx < MT * 128 * nck; idx += T) {
        const int hh = idx / (128 * nck), rem = idx - hh * 128 * nck;
        const int row = rem & 127, ck = rem >> 7;
        const int rt = hh * 128 + row, fyt = rt / rowlen;
        const int gg = kW1TmemPix / 4 + ck;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gg < ngroups) {
          const uint8_t *src = simg + fyt * a.W * a.C + (rt - fyt * rowlen) + gbase[gg];
          v.x = __fsub_rn(__uint_as_float(0x4B000000u | src[0]), 8388608.f);
          v.y = __fsub_rn(__uint_as_float(0x4B000000u | src[SWC]), 8388608.f);
          v.z = __fsub_rn(__uint_as_float(0x4B000000u | src[2 * SWC]), 8388608.f);
          v.w = __fsub_rn(__uint_as_float(0x4B000000u | src[3 * SWC]), 8388608.f);
        }
        tc::st_shared_v4(tbase + (uint32_t)(hh * a.tail_bytes) + w1_chunk(128, row, 4 * ck), v);
      }
      tc::fence_proxy_async();
    }
    tc::tmem_wait_st();
    tc::tc_fence_before();
    __syncthreads();
    if (t == 0) {
      tc::tc_fence_after();
      W1_MARK(9)
      // addresses in registers: the issue loop is on the critical path (a
      // shared-memory reload of the TMEM base per MMA doubles its cost)
      const uint32_t d0 = tmem0, ts = min(len8, kW1TmemPix) / 8, ns = len8 / 8;
      const uint64_t bd0 = tc::make_sdesc(bbase, RB * 16, 128);
#pragma unroll 2
      for (uint32_t ks = 0; ks < (W1_SKIP(1) ? 0u : ts); ++ks) {
        const uint64_t bd = bd0 + (uint64_t)(ks * 2 * RB);        // start address field, 16-B units
        const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
#pragma unroll
        for (int m = 0; m < MT; ++m)
          tc::mma_ts(d0 + (uint32_t)(m * 256), d0 + (uint32_t)(m * 256 + A_COL) + 8 * ks, bd, IDESC, acc);
      }
      for (uint32_t ks = ts; ks < (W1_SKIP(1) ? 0u : ns); ++ks) {
        const uint64_t bd = bd0 + (uint64_t)(ks * 2 * RB);
#pragma unroll
        for (int m = 0; m < MT; ++m)
          w1_mma_ss(d0 + (uint32_t)(m * 256),
                    tc::make_sdesc(tbase + (uint32_t)(m * a.tail_bytes) + (ks - ts) * 2 * 128 * 16, 128 * 16, 128),
                    bd, IDESC, 1u);
      }
      W1_MARK(10)
      tc::mma_commit(&done);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) bias_red[t / NQ][4 * q + i] = bs[i];
  // one warp polls the MMAs' barrier, the rest sleep on the CTA barrier
  // (32 warps polling shared memory slow the tensor core's operand reads)
  if (warp == 0) tc::mbar_wait(&done, (it - 1) & 1);
  __syncthreads();
  tc::tc_fence_after();
  W1_MARK(4)

  // ---- epilogue: the partial [R][N] leaves TMEM straight for the rank that
  // owns its rows: st.async into that CTA's receive slot [this rank], counted
  // on its mbarrier (no cluster barrier around the exchange)
  if (cl > 1) cluster_wait_();               // every peer's receive barrier is initialised
  constexpr int SLICES = 4 * (N / 16);       // (lane quarter, 16-channel group) per M-tile
  if ((warp & 15) < SLICES) {
    const int c0 = sub * 16;
    float lo[16], hi[16];
    tc::tmem_ld16(lane_base + (uint32_t)(N + c0), lo);
    tc::tmem_ld16(lane_base + (uint32_t)c0, hi);
    const int owner = r / rows;
    const uint32_t dst = tc::dsmem_addr(
        rbase + (uint32_t)(((rank * rows + r - owner * rows) * N + c0) * 4), owner);
    const uint32_t bar = tc::dsmem_addr(tc::smem_u32(&recv), owner);
#pragma unroll
    for (int i = 0; i < 16; i += 4)
      st_async4(dst + 4 * i, make_float4(__fadd_rn(lo[i], hi[i]), __fadd_rn(lo[i + 1], hi[i + 1]),
                                         __fadd_rn(lo[i + 2], hi[i + 2]),
                                         __fadd_rn(lo[i + 3], hi[i + 3])),
                bar);
  }
  __syncthreads();                           // bias_red complete
  // bias: 8 partial sums of T / NQ / 8 thread rows each, then the 8 in order
  constexpr int BR = T / NQ / 8;
  if (t < 8 * N) {
    const int c = t % N, part = t / N;
    float s = bias_red[part * BR][c];
    for (int gg = 1; gg < BR; ++gg) s = __fadd_rn(s, bias_red[part * BR + gg][c]);
    bias_red[part * BR][c] = s;
  }
  __syncthreads();
  if (t < N) {
    float s = bias_red[0][t];
    for (int part = 1; part < 8; ++part) s = __fadd_rn(s, bias_red[part * BR][t]);
    st_async1(tc::dsmem_addr(rbase + (uint32_t)((R * N + rank * N + t) * 4), 0), s,
              tc::dsmem_addr(tc::smem_u32(&recv), 0));
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_slot),
                 "r"(256 * MT)
                 : "memory");
  W1_MARK(5)

  // ---- this rank's rows summed over the cluster in rank order -> cluster partial
  const int64_t cstride = R * N + N;
  float *gp = a.gpart + (int64_t)cid * cstride;
  const float *recvf = reinterpret_cast<const float *>(smem + a.recv_off);
  tc::mbar_wait(&recv, 0);
  for (int idx = t; idx < rows * NQ; idx += T) {
    const int rr = idx / NQ, c4 = (idx % NQ) * 4;
    float4 acc = *reinterpret_cast<const float4 *>(recvf + rr * N + c4);
    for (int qq = 1; qq < cl; ++qq) {
      const float4 v = *reinterpret_cast<const float4 *>(recvf + (qq * rows + rr) * N + c4);
      acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
    }
    *reinterpret_cast<float4 *>(gp + (r0 + rr) * N + c4) = acc;
  }
  if (rank == 0 && t < N) {
    const float *bsl = recvf + R * N;
    float s = bsl[t];
    for (int qq = 1; qq < cl; ++qq) s = __fadd_rn(s, bsl[qq * N + t]);
    gp[R * N + t] = s;
  }
  W1_MARK(6)

  // ---- across clusters: the last cluster to finish slice `rank` adds them in
  // a fixed order: thread group g sums clusters g, g + G, ... of an item (16
  // bytes), then the groups are added in order
  __shared__ int s_ticket;
  __threadfence();
  __syncthreads();
  if (t == 0) s_ticket = atomicAdd(&a.counters[rank], 1);
  __syncthreads();
  W1_MARK(7)
  if (s_ticket != a.ncl - 1) return;
  __threadfence();
  const int items = rows * NQ;
  const int G = items >= T ? 1 : min(4, T / items), TG = T / G;
  float4 *red = reinterpret_cast<float4 *>(smem + a.recv_off);   // the receive slots are read
  for (int base = 0; base < items; base += TG) {
    const int item = base + t % TG, grp = t / TG;
    const bool act = item < items;
    const int rr = r0 + item / NQ, c4 = (item % NQ) * 4;
    float *gr = a.grad + rr * N + c4;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f), acc = o;
    if (act) {
      if (grp == 0) o = *reinterpret_cast<const float4 *>(gr);      // in flight with the partials
      const float *src = a.gpart + rr * N + c4;
      float4 v[3] = {o, o, o};
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (grp + k * G < a.ncl) v[k] = __ldcg(reinterpret_cast<const float4 *>(src + (grp + k * G) * cstride));
      acc = v[0];
#pragma unroll
      for (int k = 1; k < 3; ++k)
        if (grp + k * G < a.ncl) {
          acc.x = __fadd_rn(acc.x, v[k].x); acc.y = __fadd_rn(acc.y, v[k].y);
          acc.z = __fadd_rn(acc.z, v[k].z); acc.w = __fadd_rn(acc.w, v[k].w);
        }
      for (int c = grp + 3 * G; c < a.ncl; c += G) {
        const float4 w = __ldcg(reinterpret_cast<const float4 *>(src + c * cstride));
        acc.x = __fadd_rn(acc.x, w.x); acc.y = __fadd_rn(acc.y, w.y);
        acc.z = __fadd_rn(acc.z, w.z); acc.w = __fadd_rn(acc.w, w.w);
      }
      if (grp > 0) red[(grp - 1) * TG + t % TG] = acc;
    }
    __syncthreads();
    if (act && grp == 0) {
      for (int k = 1; k < G && k < a.ncl; ++k) {
        const float4 w = red[(k - 1) * TG + t];
        acc.x = __fadd_rn(acc.x, w.x); acc.y = __fadd_rn(acc.y, w.y);
        acc.z = __fadd_rn(acc.z, w.z); acc.w = __fadd_rn(acc.w, w.w);
      }
      o.x = __fadd_rn(o.x, __fdiv_rn(acc.x, 255.0f));
      o.y = __fadd_rn(o.y, __fdiv_rn(acc.y, 255.0f));
      o.z = __fadd_rn(o.z, __fdiv_rn(acc.z, 255.0f));
      o.w = __fadd_rn(o.w, __fdiv_rn(acc.w, 255.0f));
      *reinterpret_cast<float4 *>(gr) = o;
      note_grad4(a.flags, o);
    }
    __syncthreads();
  }
  if (rank == 0 && t < N) {
    float v[8];
    float s = 0.f;
    for (int c0 = 0; c0 < a.ncl; c0 += 8) {  // 8 loads in flight, summed in cluster order
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < a.ncl) v[k] = __ldcg(a.gpart + (c0 + k) * cstride + R * N + t);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < a.ncl) s = c0 + k == 0 ? v[0] : __fadd_rn(s, v[k]);
    }
    acc_grad(a.bias_grad + t, s, a.flags);
  }
  W1_MARK(8)
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
  cfg.gridDim = dim3(a.cpm);
  cfg.blockDim = dim3(512 * MT);
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

// image | B [hi ; lo] (2 Cout x P8) | A tail | receive slots (R x Cout + 8 x Cout floats)
inline int w1_smem(const dqn_layer_desc &L, int P8, int &img_smem, int &tail_off, int &tail_bytes,
                   int &recv_off) {
  const int img = L.in_h * L.in_w * L.in_c, R = L.fh * L.fw * L.in_c;
  img_smem = (img + 127) / 128 * 128;
  tail_off = img_smem + 2 * L.out_c * P8 * 4;
  tail_bytes = P8 > kW1TmemPix ? 128 * (P8 - kW1TmemPix) * 4 : 0;
  recv_off = tail_off + R / 128 * tail_bytes;
  return recv_off + (R + 8) * L.out_c * 4;
}

}  // namespace

// Units per image: the fewest pixel ranges of whole 8-pixel MMA steps (the
// last one takes the rest) of at most kW1MaxPix pixels: Atari 400 -> 200 + 200
inline int w1_unit_pixels_for(int P, int ps) { return ((P + ps - 1) / ps + 7) / 8 * 8; }
inline int w1_splits(int P) {
  int ps = 1;
  while (w1_unit_pixels_for(P, ps) > kW1MaxPix) ++ps;
  return ps;
}
inline int w1_unit_pixels(int P) { return w1_unit_pixels_for(P, w1_splits(P)); }

// Is layer 0 a uint8 convolution this kernel takes (Atari: 8x8x4 -> 32,
// 16-byte pixel step, 20 output columns)?
bool conv1_wgrad_u8_ok(const dqn_net_desc *net) {
  if (!net->input_u8 || net->n_layers < 1 || net->algo == 1) return false;
  const dqn_layer_desc &L = net->layer[0];
  if (L.kind != DQN_LAYER_CONV) return false;
  const int R = L.fh * L.fw * L.in_c, P = L.out_h * L.out_w;
  if (R % 128 || R > 256 || !(L.out_c == 16 || L.out_c == 32)) return false;
  if ((L.in_h * L.in_w * L.in_c) % 16 || L.out_w % 4 || L.sw * L.in_c != 16) return false;
  const int PP = w1_unit_pixels(P);
  if (PP > kW1MaxPix || (w1_splits(P) - 1) * PP >= P) return false;   // no empty unit
  int img_smem, tail_off, tail_bytes, recv_off;
  return w1_smem(L, PP, img_smem, tail_off, tail_bytes, recv_off) <= 200 * 1024;
}

// largest cluster: 4 (product A/B in the learner, r02g kernel: 8,022 vs 7,987
// with 8, 7,826 with 2 -- four-CTA clusters leave the concurrent conv2 wgrad's
// clusters room in the GPCs)
#ifdef DQN_TC_TRACE
int g_w1_cl_max = 4;   // diagnostic: largest cluster
#else
constexpr int g_w1_cl_max = 4;
#endif

// one CTA per unit up to 64 units (Atari batch 32 in the learner: the rest of
// the SMs stay free for the concurrent wgrads); larger batches loop over units
// inside up to 144 CTAs (clusters of 8 on 148 SMs), so the reduction stays
// <= 144 partials
inline int w1_cpm(int units) { return units <= 64 ? units : std::min(units, 144); }

int64_t conv1_wgrad_u8_scratch(const dqn_net_desc *net, int batch) {
  const dqn_layer_desc &L = net->layer[0];
  // at most one partial per CTA
  return (int64_t)w1_cpm(batch * w1_splits(L.out_h * L.out_w)) *
         (L.fh * L.fw * L.in_c * L.out_c + L.out_c);
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
  a.PP = w1_unit_pixels(a.P);
  a.R = L.fh * L.fw * L.in_c;
  a.img_bytes = L.in_h * L.in_w * L.in_c;
  a.units = batch * a.PS;
  a.cpm = w1_cpm(a.units);
  a.cl = 1;
  for (int c : {8, 4, 2})                   // up to g_w1_cl_max
    if (c <= g_w1_cl_max && a.cpm % c == 0) { a.cl = c; break; }
  a.ncl = a.cpm / a.cl;
  int smem = w1_smem(L, a.PP, a.img_smem, a.tail_off, a.tail_bytes, a.recv_off);
#ifdef W1_EXCLUSIVE
  smem = std::max(smem, 200 * 1024);
#endif
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
