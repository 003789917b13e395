// The trunk's fp32-input convolutions (conv2, conv3 of the Atari net:
// layers.py:226-255 forward) as an implicit GEMM on tcgen05 with BOTH
// operands fed by TMA tensor loads -- no operand passes through registers on
// its way from global memory.
//
//   D[pixel][n] = sum_k A[pixel][k] W[k][n],  k = (r, s, c)  (patch_off order)
//
// A (the im2col rows) is never materialised.  A k-block of 32 is one filter
// tap (r, s) and 32 channels, so the A tile of a k-block is the input read at
// one fixed tap for every output pixel of the tile: a strided box of the
// NHWC activations.  For stride S the input is viewed as the 5-D tensor
//
//   {S*C, W/S, S, H/S, B}   (x = S*x2 + xs folded into the innermost dim)
//
// so that tap (r, s) is the box {32, OW, 1, OH, ipt} at
// {(s%S)*C + c0, s/S, r%S, r/S, img0}: OW x OH output pixels of ipt whole
// images, each row 32 channels = 128 B, written by the TMA straight into the
// 128-byte-swizzle K-major layout the MMA reads.  A tile holds whole images
// (ipt = floor(128 / (OH*OW)): conv2 1 image = 81 of 128 rows, conv3 2
// images = 98 rows); the rows past them are never stored.
//
// W [K][N] (N contiguous) arrives as raw [32 k][N] tiles that the converter
// warps transpose into the K-major B operand (tf32 MMAs take K-major operands
// only) together with its tf32 lo piece; they also derive A's lo piece in
// place.  3xTF32 as in lin_tc.cu / tc_gemm.cuh:
//   A_hi * [B_hi ; B_lo]  (N = 2 NB) -> [hi*hi | hi*lo],  A_lo * B_hi -> += lo*hi
// into two TMEM accumulator pairs alternating by k-block, summed in a fixed
// order.  K is split across a thread-block cluster; the cluster reduces the
// partial tiles through distributed shared memory in rank order
// (deterministic), adds the bias and applies the ReLU.
//
// The same kernel computes the input gradient (layers.py:235-248) of a conv
// whose filter tiles its stride, one GEMM per stride phase (py, px):
//
//   dX[S yq + py][S xq + px][c] = sum_{i, j, n} dY[yq - i][xq - j][n] W[py + S i][px + S j][c][n]
//
// rows = the phase's input pixels of whole images, K = its taps x dY channels.
// The dY box of tap (i, j) starts at (-j, -i): the TMA fills the rows that
// fall off the dY grid with zeros.  W's rows (r, s, c) with n contiguous are
// K-major for this product and arrive as 128B-swizzle boxes (only their lo
// pieces are computed); the epilogue applies the ReLU mask of the layer
// below.  Launch shapes: 2 stages, 2 CTAs per SM; K split sized for ~128 CTAs
// per forward launch (64 for a DQN_NET_HINT_SIDE trunk), ~256 per dgrad.
#include "tc_gemm.cuh"

#include <algorithm>

namespace dqn {
namespace {

constexpr int CT_BK = 32;                      // k per stage: one tap x 32 channels
constexpr int CT_BM = 128;                     // A tile rows (output pixels)
constexpr int CT_THREADS = 192;                // warps 0-3 convert + epilogue, 4 TMA, 5 MMA

struct ConvTcArgs {
  CUtensorMap amap;                            // fwd: activations, dgrad: dY (5-D views, SW128)
  CUtensorMap bmap;                            // fwd: W [K][N] raw [32 k][N]; dgrad: W rows (SW128)
  int K, C, fw, S;                             // GEMM depth (per stride phase), channels of the
                                               // k-blocks (fwd: in, dgrad: out), filter width, stride
  int P, ipt, npix;                            // rows per image, images per tile, B * P
  int klen;                                    // k per cluster rank (multiple of CT_BK)
  int a_bytes;                                 // one A piece: ipt*P rows rounded up to 8, x 128 B
  // dgrad: rows are the input pixels (S*yq + py, S*xq + px) of stride phase
  // (py, px) = blockIdx.z, QH x QW of them per image; taps (py + S i, px + S j)
  int QW, TW, H, W, cin;                       // phase grid width, taps per phase row, input dims
  const float *bias;                           // fwd
  int relu;                                    // fwd
  const float *mask;                           // dgrad: the layer below's ReLU output (or null)
  float *y;                                    // fwd: [B * P][N]; dgrad: dX [B][H][W][cin]
};

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void ct_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// K-major 128-byte-swizzle operand tile: 128 B rows, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t ct_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Stage: A_hi | A_lo (a_bytes each, runtime) | [B_hi ; B_lo] | raw W tile.
// Two stages of the Atari convs fit twice per SM (conv2 2 x 46 KB, conv3
// 2 x 50 KB), so the online and target networks' launches share the SMs.
template <int NB, bool DG>
struct CtPlan {
  static constexpr int B_BYTES = 2 * NB * CT_BK * 4;     // [B_hi ; B_lo]
  static constexpr int RAW = DG ? 0 : CT_BK * NB * 4;    // fwd: W tile as loaded
  static constexpr int LD = NB + 4;                      // staged partial row stride (floats)
  static constexpr int EPI = CT_BM * LD * 4;
  static int stage(int a_bytes) { return 2 * a_bytes + B_BYTES + RAW; }
  static int bytes(int st, int a_bytes) { return std::max(st * stage(a_bytes), EPI) + 1024; }
  static constexpr int TMEM = 4 * NB <= 128 ? 128 : 256;
};

// TS: A's lo pieces go to tensor memory (tcgen05.st, one row
// per converter thread) and the lo * hi MMA reads them there (TS form), one
// accumulator pair: a stage is A_hi | [B_hi ; B_lo] | raw W, one A piece
// smaller, so three stages fit twice per SM.
template <int NB, int CT_ST, bool DG, bool TS = false>
__global__ void __launch_bounds__(CT_THREADS, 2) conv_tc_kernel(const __grid_constant__ ConvTcArgs p) {
  using PL = CtPlan<NB, DG>;
  constexpr int A_PIECES = TS ? 1 : 2;
  constexpr int CT_EPI_LD = PL::LD;
  constexpr uint32_t ID_FULL = tc::make_idesc_tf32(2 * NB), ID_HALF = tc::make_idesc_tf32(NB);
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[CT_ST], conv[CT_ST], empty[CT_ST], done;
  __shared__ uint32_t tmem_slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t sbase = (tc::smem_u32(smem) + 1023u) & ~1023u;
  const int img0 = blockIdx.x * p.ipt;
  const int pix0 = img0 * p.P;
  const int rows = min(p.ipt * p.P, p.npix - pix0);     // valid A rows of this tile
  const int cl = gridDim.y, rank = blockIdx.y;
  const int kbeg = rank * p.klen, kend = min(p.K, kbeg + p.klen);
  const int nkb = kend > kbeg ? (kend - kbeg) / CT_BK : 0;

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(TS ? 256 : PL::TMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 32 * 5) {
    for (int s = 0; s < CT_ST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_trigger();
  pdl_wait();                                 // activations come from the layer below
  const uint32_t tmem = tmem_slot;

  const uint32_t stage_b = (uint32_t)(A_PIECES * p.a_bytes + PL::B_BYTES + PL::RAW);
  auto a_hi = [&](int s) { return sbase + (uint32_t)s * stage_b; };
  auto a_lo = [&](int s) { return sbase + (uint32_t)s * stage_b + (uint32_t)p.a_bytes; };
  auto b_st = [&](int s) { return sbase + (uint32_t)s * stage_b + (uint32_t)(A_PIECES * p.a_bytes); };
  auto b_raw = [&](int s) {
    return sbase + (uint32_t)s * stage_b + (uint32_t)(A_PIECES * p.a_bytes + PL::B_BYTES);
  };

  if (warp == 4) {
    if (lane == 0) {                          // TMA producer
      const uint32_t a_box = (uint32_t)(p.ipt * p.P * CT_BK * 4);
      const int py = DG ? (int)blockIdx.z / p.S : 0, px = DG ? (int)blockIdx.z % p.S : 0;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % CT_ST, use = kb / CT_ST;
        if (use > 0) tc::mbar_wait(&empty[s], (use - 1) & 1);
        tc::mbar_expect_tx(&full[s], a_box + (uint32_t)(DG ? NB * CT_BK * 4 : PL::RAW));
        const int k0 = kbeg + kb * CT_BK;
        const int tap = k0 / p.C, c0 = k0 - tap * p.C;
        if constexpr (DG) {
          // tap (i, j) of this phase: filter (py + S i, px + S j) reads dY at
          // (yq - i, xq - j); rows off the dY grid come back as zeros
          const int i = tap / p.TW, j = tap - i * p.TW;
          const int r = py + p.S * i, q = px + p.S * j;
          tma_load_5d(a_hi(s), &p.amap, c0, -j, 0, -i, img0, &full[s]);
          tc::tma_load_2d(b_st(s), &p.bmap, c0, (r * p.fw + q) * NB, &full[s]);
        } else {
          const int r = tap / p.fw, q = tap - r * p.fw;
          tma_load_5d(a_hi(s), &p.amap, (q % p.S) * p.C + c0, q / p.S, r % p.S, r / p.S, img0,
                      &full[s]);
          tc::tma_load_2d(b_raw(s), &p.bmap, 0, k0, &full[s]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {                          // MMA issuer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % CT_ST, use = kb / CT_ST;
        tc::mbar_wait(&conv[s], use & 1);
        tc::tc_fence_after();
        const uint32_t dbig = tmem + (uint32_t)(TS ? 0 : (kb & 1) * 2 * NB);
#pragma unroll
        for (int kq = 0; kq < CT_BK / 8; ++kq) {
          const uint64_t da = ct_desc(a_hi(s) + 32 * kq);
          const uint64_t db = ct_desc(b_st(s) + 32 * kq);
          if constexpr (TS) {
            ct_mma(dbig, da, db, ID_FULL, (kb == 0 && kq == 0) ? 0u : 1u);
            tc::mma_ts(dbig + NB, tmem + 2 * NB + (uint32_t)(s * CT_BK + 8 * kq), db, ID_HALF, 1u);
          } else {
            const uint64_t dl = ct_desc(a_lo(s) + 32 * kq);
            ct_mma(dbig, da, db, ID_FULL, (kb < 2 && kq == 0) ? 0u : 1u);
            ct_mma(dbig + NB, dl, db, ID_HALF, 1u);
          }
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&done);
    }
  } else {                                    // warps 0-3: lo pieces, W transpose
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % CT_ST, use = kb / CT_ST;
      tc::mbar_wait(&full[s], use & 1);
      if constexpr (TS) {
        // A lo of row t into TMEM lane t, columns 2 NB + 32 s .. (k order)
        float lo[CT_BK];
#pragma unroll
        for (int c = 0; c < CT_BK / 4; ++c) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (t < rows)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(a_hi(s) + (uint32_t)(t * 128 + ((c ^ (t & 7)) << 4))));
          lo[4 * c] = tc::tf32_lo(v.x);
          lo[4 * c + 1] = tc::tf32_lo(v.y);
          lo[4 * c + 2] = tc::tf32_lo(v.z);
          lo[4 * c + 3] = tc::tf32_lo(v.w);
        }
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 2 * NB + (uint32_t)(s * CT_BK);
        tc::tmem_st16(ta, lo);
        tc::tmem_st16(ta + 16, lo + 16);
        tc::tmem_wait_st();
      } else {
        // A: the valid rows' 16-byte chunks, lo at the same (swizzled) offsets
        for (int i = t; i < rows * (CT_BK / 4); i += 128) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a_hi(s) + 16 * i));
          tc::st_shared_v4(a_lo(s) + 16 * i, make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y),
                                                         tc::tf32_lo(v.z), tc::tf32_lo(v.w)));
        }
      }
      if constexpr (DG) {
        // B arrived K-major (W rows (r, s, c), n contiguous): lo rows NB..2NB-1
        // are hi's bytes shifted by NB rows (the swizzle repeats every 8 rows)
        for (int i = t; i < NB * CT_BK / 4; i += 128) {
          const uint32_t src = b_st(s) + 16 * i;
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src));
          tc::st_shared_v4(src + NB * 128, make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y),
                                                       tc::tf32_lo(v.z), tc::tf32_lo(v.w)));
        }
      }
      // B: raw [32 k][NB n] -> row n (hi) and row NB + n (lo), 16-byte column
      // c ^ (n % 8) of the swizzled K-major tile (lanes = consecutive n)
      for (int u = t; u < (DG ? 0 : NB * (CT_BK / 4)); u += 128) {
        const int n = u % NB, c = u / NB;
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile("ld.shared.f32 %0, [%1];"
                       : "=f"(v[i]) : "r"(b_raw(s) + (uint32_t)(((4 * c + i) * NB + n) * 4)));
        const uint32_t off = (uint32_t)(n * 128 + ((c ^ (n & 7)) << 4));
        tc::st_shared_v4(b_st(s) + off, make_float4(v[0], v[1], v[2], v[3]));
        tc::st_shared_v4(b_st(s) + (uint32_t)(NB * 128) + off,
                         make_float4(tc::tf32_lo(v[0]), tc::tf32_lo(v[1]), tc::tf32_lo(v[2]),
                                     tc::tf32_lo(v[3])));
      }
      tc::fence_proxy_async();                // generic smem writes -> tensor-core reads
      if constexpr (TS) tc::tc_fence_before(); // TMEM stores -> the MMA thread
      tc::mbar_arrive(&conv[s]);
    }
  }

  // ---- epilogue: accumulators -> this CTA's partial tile, staged [128][CT_EPI_LD]
  __syncthreads();
  tc::mbar_wait(&done, 0);
  tc::tc_fence_after();
  float *stage = reinterpret_cast<float *>(smem + (sbase - tc::smem_u32(smem)));
  if (warp < 4) {
    const int row = warp * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    const bool two = !TS && nkb > 1;
#pragma unroll 1
    for (int c = 0; c < NB; c += 16) {
      float s0[16], s1[16], b0[16], b1[16];
      tc::tmem_ld16(lb + (uint32_t)(NB + c), s0);
      tc::tmem_ld16(lb + (uint32_t)c, b0);
      if (two) {
        tc::tmem_ld16(lb + (uint32_t)(3 * NB + c), s1);
        tc::tmem_ld16(lb + (uint32_t)(2 * NB + c), b1);
      }
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 v;
        float *e = &v.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float w = two ? __fadd_rn(__fadd_rn(s0[j + i], s1[j + i]),
                                          __fadd_rn(b0[j + i], b1[j + i]))
                              : __fadd_rn(s0[j + i], b0[j + i]);
          e[i] = nkb > 0 ? w : 0.f;
        }
        *reinterpret_cast<float4 *>(&stage[row * CT_EPI_LD + c + j]) = v;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TS ? 256 : PL::TMEM)
                 : "memory");
  // ---- cluster reduction: rank q owns a contiguous range of (row, 4 channels)
  // units and sums the ranks' partials in rank order; then bias and ReLU
  if (cl > 1) tc::cluster_sync();
  constexpr int U4 = NB / 4;
  const int units = rows * U4;
  const int ub = (int)((long long)units * rank / cl), ue = (int)((long long)units * (rank + 1) / cl);
  for (int u0 = ub + t; u0 < ue; u0 += 4 * CT_THREADS) {
    float4 acc[4];
    int uu[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uu[h] = u0 + h * CT_THREADS;
      acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (uu[h] >= ue) continue;
      const int row = uu[h] / U4, c4 = uu[h] - row * U4;
      const int sidx = row * CT_EPI_LD + 4 * c4;
      if (cl > 1) {
        const uint32_t la = tc::smem_u32(&stage[sidx]);
        float4 r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < cl) r[q] = tc::ld_dsmem4(tc::dsmem_addr(la, q));
        acc[h] = r[0];
#pragma unroll
        for (int q = 1; q < 8; ++q)
          if (q < cl) {
            acc[h].x = __fadd_rn(acc[h].x, r[q].x); acc[h].y = __fadd_rn(acc[h].y, r[q].y);
            acc[h].z = __fadd_rn(acc[h].z, r[q].z); acc[h].w = __fadd_rn(acc[h].w, r[q].w);
          }
      } else {
        acc[h] = *reinterpret_cast<const float4 *>(&stage[sidx]);
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (uu[h] >= ue) continue;
      const int row = uu[h] / U4, c4 = uu[h] - row * U4;
      float v[4] = {acc[h].x, acc[h].y, acc[h].z, acc[h].w};
      int64_t o;
      if constexpr (DG) {
        // row -> input pixel of this stride phase
        const int img = row / p.P, q = row - img * p.P;
        const int yq = q / p.QW, xq = q - yq * p.QW;
        const int y = p.S * yq + (int)blockIdx.z / p.S, x = p.S * xq + (int)blockIdx.z % p.S;
        if (y >= p.H || x >= p.W) continue;
        o = (((int64_t)(img0 + img) * p.H + y) * p.W + x) * p.cin + 4 * c4;
        if (p.mask) {
          const float4 m = *reinterpret_cast<const float4 *>(p.mask + o);
          if (!(m.x > 0.f)) v[0] = 0.f;
          if (!(m.y > 0.f)) v[1] = 0.f;
          if (!(m.z > 0.f)) v[2] = 0.f;
          if (!(m.w > 0.f)) v[3] = 0.f;
        }
      } else {
        const float4 b = *reinterpret_cast<const float4 *>(p.bias + 4 * c4);
        v[0] = __fadd_rn(v[0], b.x); v[1] = __fadd_rn(v[1], b.y);
        v[2] = __fadd_rn(v[2], b.z); v[3] = __fadd_rn(v[3], b.w);
        if (p.relu) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (v[e] < 0.f) v[e] = 0.f;
        }
        o = (int64_t)(pix0 + row) * NB + 4 * c4;
      }
      *reinterpret_cast<float4 *>(p.y + o) = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  if (cl > 1) tc::cluster_sync();             // peers' staged partials read
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn ct_encode() {
  static EncodeTiledFn fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// NHWC activations [B][H][W][C] as {S*C, W/S, S, H/S, B}; boxes of one tap
bool ct_act_map(CUtensorMap *m, const float *x, const dqn_layer_desc &L, int batch, int ipt) {
  const EncodeTiledFn fn = ct_encode();
  const int S = L.sw, C = L.in_c, W = L.in_w, H = L.in_h;
  if (!fn || ((uintptr_t)x % 16)) return false;
  const cuuint64_t dims[5] = {(cuuint64_t)S * C, (cuuint64_t)W / S, (cuuint64_t)S,
                              (cuuint64_t)H / S, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)S * C * 4, (cuuint64_t)W * C * 4,
                                 (cuuint64_t)S * W * C * 4, (cuuint64_t)H * W * C * 4};
  const cuuint32_t box[5] = {CT_BK, (cuuint32_t)L.out_w, 1, (cuuint32_t)L.out_h, (cuuint32_t)ipt};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float *>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// W [K][N] fp32 (N contiguous) as raw [32 k][N] tiles
bool ct_w_map(CUtensorMap *m, const float *w, int K, int N) {
  const EncodeTiledFn fn = ct_encode();
  if (!fn || ((uintptr_t)w % 16)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
  const cuuint64_t strides[1] = {(cuuint64_t)N * 4};
  const cuuint32_t box[2] = {(cuuint32_t)N, CT_BK};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// dgrad operands: dY [B][OH][OW][N] as {N, OW, 1, OH, B} with boxes of the
// phase grid {32, QW, 1, QH, ipt} (reads off the grid fill zeros), and W as
// rows (r, s, c) of N: boxes {32 n, cin rows}, K-major for the MMA as loaded
bool ct_dy_map(CUtensorMap *m, const float *dy, const dqn_layer_desc &L, int batch, int ipt,
               int QH, int QW) {
  const EncodeTiledFn fn = ct_encode();
  const int N = L.out_c;
  if (!fn || ((uintptr_t)dy % 16)) return false;
  const cuuint64_t dims[5] = {(cuuint64_t)N, (cuuint64_t)L.out_w, 1, (cuuint64_t)L.out_h,
                              (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)N * 4, (cuuint64_t)L.out_w * N * 4,
                                 (cuuint64_t)L.out_w * N * 4, (cuuint64_t)L.out_h * L.out_w * N * 4};
  const cuuint32_t box[5] = {CT_BK, (cuuint32_t)QW, 1, (cuuint32_t)QH, (cuuint32_t)ipt};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float *>(dy), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool ct_wrows_map(CUtensorMap *m, const float *w, int rows, int N, int box_rows) {
  const EncodeTiledFn fn = ct_encode();
  if (!fn || ((uintptr_t)w % 16)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)N * 4};
  const cuuint32_t box[2] = {CT_BK, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// CTAs one forward launch aims for: K split = ceil(fill / tiles).  128, and
// 64 for a side trunk (DQN_NET_HINT_SIDE: the learner's target trunk beside
// its online one).  Measured in the learner: one fill for both 64 /
// 96 / 128 / 160 / 256 -> 128 best; fixed splits per layer 6-10 % slower;
// with the online at 128, target fills 32 / 48 / 64 / 80 / 96 / 128 / 192 ->
// 6,579 / 7,094 / 7,103-7,118 / 7,074 / 7,005 / 7,050 / 7,018 updates/s.
#ifdef DQN_TC_TRACE
int g_ct_cluster = 0;   // diagnostic: 0 auto, > 0 cluster size, -1 engine, -2/-3 one layer only
int g_ct_stages = 2;    // diagnostic: pipeline stages (2 or 3; 3 measured slower)
int g_ct_fill = 128;
int g_ct_fill_small = 64;    // diagnostic: fill of a side trunk (DQN_NET_HINT_SIDE)
int g_ct_dgrad = 1;     // diagnostic: 0 = conv dgrad on the generic engine
int g_ct_dfill = 256;   // dgrad: CTAs one launch aims for
int g_ct_ts = 3;        // diagnostic: forward with A lo in TMEM, this many stages (0 = off)
int g_ct_dts = 3;       // diagnostic: the same for the input gradients
#else
constexpr int g_ct_cluster = 0, g_ct_stages = 2, g_ct_fill = 128, g_ct_dgrad = 1, g_ct_dfill = 256;
constexpr int g_ct_fill_small = 64;
#endif

template <int NB, int ST, bool DG, bool TS = false>
int ct_launch(cudaStream_t st, const ConvTcArgs &a, dim3 grid, const char *what) {
  using PL = CtPlan<NB, DG>;
  auto kern = conv_tc_kernel<NB, ST, DG, TS>;
  // TS: one A piece per stage (its lo pieces live in TMEM)
  auto bytes = [](int a_bytes) {
    return TS ? std::max(ST * (a_bytes + PL::B_BYTES + PL::RAW), PL::EPI) + 1024
              : PL::bytes(ST, a_bytes);
  };
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         bytes(CT_BM * 128));
    if (e != cudaSuccess) return cuda_status(e, what);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(CT_THREADS);
  cfg.dynamicSmemBytes = bytes(a.a_bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  attr[2].id = cudaLaunchAttributeClusterDimension;
  attr[2].val.clusterDim.x = 1;
  attr[2].val.clusterDim.y = grid.y;
  attr[2].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 3;
  cudaLaunchKernelEx(&cfg, kern, a);
  DQN_LAUNCH_CHECK(what);
  return DQN_OK;
}

// K split across a cluster: about g_ct_fill CTAs per launch, no empty ranks
int ct_split(ConvTcArgs &a, int tiles, int sw, int fill) {
  const int chunks = a.K / CT_BK;
  int cl = (fill + tiles - 1) / tiles;
  if (g_ct_cluster >= 16)                        // diagnostic: stride-2 layer | stride-1 layer
    cl = sw == 2 ? (g_ct_cluster >> 4) : (g_ct_cluster & 15);
  else if (g_ct_cluster > 0)
    cl = g_ct_cluster;
  cl = std::max(1, std::min({cl, 8, chunks}));
  const int per = (chunks + cl - 1) / cl;
  a.klen = per * CT_BK;
  return (chunks + per - 1) / per;
}

}  // namespace

// fp32-input convolution this kernel tiles: 64 output channels, 32-channel
// k-blocks, equal strides dividing the input, whole images within 128 rows
bool conv_tc_ok(const dqn_layer_desc &L) {
  const int P = L.out_h * L.out_w;
  return L.kind == DQN_LAYER_CONV && L.out_c == 64 && L.in_c % CT_BK == 0 && L.sh == L.sw &&
         L.sw >= 1 && L.in_w % L.sw == 0 && L.in_h % L.sh == 0 && P >= 1 && P <= CT_BM &&
         L.out_w <= 256 && L.out_h <= 256;
}

int conv_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const float *x, const float *params,
                    float *y, int batch, bool side) {
  if (g_ct_cluster == -1 || (g_ct_cluster == -2 && L.sw != 2) || (g_ct_cluster == -3 && L.sw != 1))
    return DQN_ERR_UNSUPPORTED;   // diagnostic: the generic engine (all / all but stride 2 / 1)
  const int P = L.out_h * L.out_w;
  const int ipt = std::max(1, std::min(CT_BM / P, std::min(batch, 256)));
  ConvTcArgs a{};
  const float *w = params + L.w_off;
  a.K = L.fh * L.fw * L.in_c;
  if (!ct_act_map(&a.amap, x, L, batch, ipt) || !ct_w_map(&a.bmap, w, a.K, 64))
    return DQN_ERR_UNSUPPORTED;
  a.C = L.in_c;
  a.fw = L.fw;
  a.S = L.sw;
  a.P = P;
  a.ipt = ipt;
  a.npix = batch * P;
  a.a_bytes = ((ipt * P + 7) / 8) * 8 * 128;
  a.bias = params + L.b_off;
  a.relu = L.relu;
  a.y = y;
  const int tiles = (batch + ipt - 1) / ipt;
  const int cl = ct_split(a, tiles, L.sw, side ? g_ct_fill_small : g_ct_fill);
#ifdef DQN_TC_TRACE
  if (g_ct_stages == 3) return ct_launch<64, 3, false>(st, a, dim3(tiles, cl, 1), "conv_tc_forward");
  if (g_ct_ts == 0) return ct_launch<64, 2, false>(st, a, dim3(tiles, cl, 1), "conv_tc_forward");
  if (g_ct_ts == 4) return ct_launch<64, 4, false, true>(st, a, dim3(tiles, cl, 1), "conv_tc_forward");
  if (g_ct_ts == 2) return ct_launch<64, 2, false, true>(st, a, dim3(tiles, cl, 1), "conv_tc_forward");
#endif
  // A's lo pieces in TMEM, three stages (measured: B = 64 conv2 / conv3 9.4-11.0 vs
  // 10.9-13.9 us with both pieces in smem and two stages; learner +2.7 %; B = 4096
  // 217 / 126 vs 298 / 171 us)
  return ct_launch<64, 3, false, true>(st, a, dim3(tiles, cl, 1), "conv_tc_forward");
}

// dX of a convolution whose filter tiles its stride (fh % S == 0), as one
// GEMM per stride phase (blockIdx.z): 32 or 64 input channels, 64-channel dY
bool conv_tc_dgrad_ok(const dqn_layer_desc &L) {
  const int S = L.sw;
  const int QH = (L.in_h + S - 1) / S, QW = (L.in_w + S - 1) / S;
  return g_ct_dgrad && L.kind == DQN_LAYER_CONV && L.sh == S && S >= 1 && L.fh % S == 0 &&
         L.fw % S == 0 && L.in_h % S == 0 && L.in_w % S == 0 && L.out_c % CT_BK == 0 &&
         (L.in_c == 32 || L.in_c == 64) && QH * QW <= CT_BM && QW <= 256 && QH <= 256;
}

int conv_tc_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
                  const float *mask, float *dx, int batch) {
  if (!conv_tc_dgrad_ok(L)) return DQN_ERR_UNSUPPORTED;
  const int S = L.sw;
  const int QH = L.in_h / S, QW = L.in_w / S;
  const int P = QH * QW;
  const int ipt = std::max(1, std::min(CT_BM / P, std::min(batch, 256)));
  ConvTcArgs a{};
  if (!ct_dy_map(&a.amap, dy, L, batch, ipt, QH, QW) ||
      !ct_wrows_map(&a.bmap, w, L.fh * L.fw * L.in_c, L.out_c, L.in_c))
    return DQN_ERR_UNSUPPORTED;
  a.TW = L.fw / S;
  a.K = (L.fh / S) * a.TW * L.out_c;            // taps of one phase x dY channels
  a.C = L.out_c;
  a.fw = L.fw;
  a.S = S;
  a.P = P;
  a.ipt = ipt;
  a.npix = batch * P;
  a.a_bytes = ((ipt * P + 7) / 8) * 8 * 128;
  a.QW = QW;
  a.H = L.in_h;
  a.W = L.in_w;
  a.cin = L.in_c;
  a.mask = mask;
  a.y = dx;
  const int tiles = (batch + ipt - 1) / ipt;
  const int cl = ct_split(a, tiles * S * S, S, g_ct_dfill);
  const dim3 grid(tiles, cl, S * S);
#ifdef DQN_TC_TRACE
  if (g_ct_dts == 0)
    return L.in_c == 32 ? ct_launch<32, 2, true>(st, a, grid, "conv_tc_dgrad")
                        : ct_launch<64, 2, true>(st, a, grid, "conv_tc_dgrad");
  if (g_ct_dts == 4)
    return L.in_c == 32 ? ct_launch<32, 4, true, true>(st, a, grid, "conv_tc_dgrad")
                        : ct_launch<64, 4, true, true>(st, a, grid, "conv_tc_dgrad");
#endif
  // A's lo pieces in TMEM, three stages (learner +1.2 %; B = 4096 conv2 / conv3
  // 432 / 289 vs 528 / 376 us)
  return L.in_c == 32 ? ct_launch<32, 3, true, true>(st, a, grid, "conv_tc_dgrad")
                      : ct_launch<64, 3, true, true>(st, a, grid, "conv_tc_dgrad");
}

}  // namespace dqn

#ifdef DQN_TC_TRACE
// diagnostic build only (tools/ct_bench.py, tools/learner_ab.py, ...)
extern "C" void dqn_ct_set_cluster(int cl) { dqn::g_ct_cluster = cl; }
extern "C" void dqn_ct_set_stages(int st) { dqn::g_ct_stages = st; }
extern "C" void dqn_ct_set_fill(int f) { dqn::g_ct_fill = f; }
extern "C" void dqn_ct_set_fill_small(int f) { dqn::g_ct_fill_small = f; }
extern "C" void dqn_ct_set_dgrad(int on) { dqn::g_ct_dgrad = on; }
extern "C" void dqn_ct_set_dfill(int f) { dqn::g_ct_dfill = f; }
extern "C" void dqn_ct_set_ts(int v) { dqn::g_ct_ts = v; }
extern "C" void dqn_ct_set_dts(int v) { dqn::g_ct_dts = v; }
#endif
