// The learner's hidden linear layer (fc1: 3136 -> 512) on tcgen05 with
// every operand fed by TMA tensor loads (layers.py:148-160; network.py:90-117).
//
// At learner batch sizes (<= 64 rows) the linear layer is a weight-streaming
// GEMM: 6.4 MB of weights against a 32- or 64-row batch.  The generic engine
// (tc_gemm.cuh) tiles it as 128 batch rows (half empty) x 64 weight columns
// and stages both operands through registers.  Here the layer is turned
// around so that the WEIGHT dimension fills the 128-row MMA tiles and the
// batch rows are the MMA's N:
//
//   forward  D[n][m] = sum_k W^T[n][k] X[m][k]     (y[m][n] = relu(D + bias[n]))
//
// (The kernel also has a dgrad form, D[f][m] = sum_n W[f][n] dY[m][n], with W
// K-major; measured slower than the generic engine's TMA-fed LinDgradTmaPol
// in the learner, it is not dispatched.)
//
// One warp issues 2-D TMA tensor loads of the raw fp32 operands, stages
// ahead: the batch operand and the dgrad's weights (W [F][N], K-major) as
// 32-k x rows boxes in the 128-byte-swizzle K-major layout the MMA reads;
// the forward's weights (W [K][N], N contiguous) as raw [32 k][128 n] tiles
// that the converter warps transpose into that layout (tf32 MMAs take
// K-major operands only).  The converters also derive the tf32 lo pieces
// (x - trunc19(x)); one thread issues the 3xTF32 MMAs from shared memory:
//   A_hi * [B_hi ; B_lo]  (N = 2 NB) -> [hi*hi | hi*lo],  A_lo * B_hi -> += lo*hi
// into two TMEM accumulator pairs alternating by k-block, summed in a fixed
// order in the epilogue (the accuracy scheme of tc_gemm.cuh).
// K is split across a thread-block cluster (<= 16 CTAs); the cluster reduces
// its partial tiles through distributed shared memory in rank order, so the
// result is deterministic and there is no global partial buffer.
#include "tc_gemm.cuh"

#include <algorithm>

namespace dqn {
namespace {

constexpr int LT_BK = 32;                      // k per stage (4 MMA k-steps)
constexpr int LT_ST = 4;                       // pipeline stages
constexpr int LT_BM = 128;
constexpr int LT_THREADS = 192;                // warps 0-3 convert + epilogue, 4 TMA, 5 MMA

#ifdef DQN_TC_TRACE
// per-CTA %globaltimer marks (trace build): entry, after pdl_wait, first
// stage converted, MMAs done, partial staged, cluster-reduced + stored
__device__ unsigned long long g_lt_trace[1024 * 6];
#define LT_MARK(i)                                                          \
  if (threadIdx.x == 0) {                                                   \
    const int b_ = blockIdx.y * gridDim.x + blockIdx.x;                     \
    unsigned long long t_;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
    if (b_ < 1024) g_lt_trace[b_ * 6 + (i)] = t_;                           \
  }
#else
#define LT_MARK(i)
#endif

struct LinTcArgs {
  CUtensorMap amap, bmap;                      // A [M][K] (box {4, 128}), B [NB][K] (box {4, NB})
  int M, K, klen;                              // klen: k per cluster rank (multiple of LT_BK)
  int nrows;                                   // batch rows (<= NB; the rest of the box is zero)
  int mode;                                    // 0 forward, 1 dgrad
  const float *bias;                           // forward: bias[M]
  int relu;
  const float *mask;                           // dgrad: act of the layer below, [NB][M] (or null)
  float *out;                                  // forward: y [NB][M]; dgrad: dx [NB][M]
  int32_t *flags;
};

__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// K-major operand tile in the 128-byte-swizzle layout: rows of 32 fp32 (one
// 128 B swizzle atom wide), 8-row atoms 1024 B apart (what a TMA box of
// {32, rows} with CU_TENSOR_MAP_SWIZZLE_128B writes).  The MMA k-step kq
// starts 32 B further into the atom.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                   // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset: 8-row atoms
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                   // layout type SWIZZLE_128B
  return d;
}

// AT (the forward): A's lo pieces go to tensor memory as the converters
// transpose the weights (one row per thread, tcgen05.st) and the lo * hi MMA
// reads them there (TS form); a stage is then A_hi | [B_hi ; B_lo] | raw, and
// four stages fit.  The two k-parity accumulator pairs stay (one CTA per SM:
// TMEM has room), which keeps long K chains (large batch, one split) at the
// dual-pair accuracy.
template <int NB, bool AT>
struct LtPlan {
  static constexpr bool TS = true;
  static constexpr int RB = 2 * NB;                       // stacked B rows
  static constexpr int A_BYTES = LT_BM * LT_BK * 4;       // one piece of the A tile
  static constexpr int B_BYTES = RB * LT_BK * 4;
  static constexpr int RAW = AT ? A_BYTES : 0;            // A as loaded ([k][m]) when transposed
  static constexpr int A_PIECES = TS ? 1 : 2;
  static constexpr int STAGE = A_PIECES * A_BYTES + B_BYTES + RAW;   // A_hi | (A_lo) | [B_hi ; B_lo] | raw
  static constexpr int ST = AT ? 4 : 6;
  static constexpr int PIPE = ST * STAGE;
  static constexpr int EPI = NB * LT_BM * 4;              // staged partial [NB][128]
  static constexpr int BYTES = (PIPE > EPI ? PIPE : EPI) + 1024;   // + alignment slack
  static constexpr int LO_COL = 4 * NB;                   // TS: A_lo columns after the pairs
  static constexpr int TMEM = TS ? (LO_COL + ST * LT_BK <= 256 ? 256 : 512)
                                 : (4 * NB <= 32 ? 32 : (4 * NB <= 64 ? 64 : (4 * NB <= 128 ? 128 : 256)));
};

template <int NB, bool AT>
__global__ void __launch_bounds__(LT_THREADS, 1) lin_tc_kernel(const __grid_constant__ LinTcArgs p) {
  using PL = LtPlan<NB, AT>;
  constexpr int LT_ST = PL::ST;
  constexpr int RB = PL::RB;
  constexpr uint32_t ID_FULL = tc::make_idesc_tf32(RB), ID_HALF = tc::make_idesc_tf32(NB);
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[LT_ST], conv[LT_ST], empty[LT_ST], done;
  __shared__ uint32_t tmem_slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t sbase = (tc::smem_u32(smem) + 1023u) & ~1023u;      // swizzle atoms: 1 KB aligned
  const int m0 = blockIdx.x * LT_BM;
  const int cl = gridDim.y, rank = blockIdx.y;               // cluster = the K splits of a tile
  const int kbeg = rank * p.klen, kend = min(p.K, kbeg + p.klen);
  const int nkb = kend > kbeg ? (kend - kbeg + LT_BK - 1) / LT_BK : 0;
  LT_MARK(0)

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(PL::TMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 32 * 5) {
    for (int s = 0; s < LT_ST; ++s) {
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
  pdl_wait();                                 // operands come from earlier kernels
  const uint32_t tmem = tmem_slot;
  LT_MARK(1)

  auto a_hi = [&](int s) { return sbase + (uint32_t)(s * PL::STAGE); };
  auto a_lo = [&](int s) { return sbase + (uint32_t)(s * PL::STAGE + PL::A_BYTES); };
  auto b_st = [&](int s) { return sbase + (uint32_t)(s * PL::STAGE + PL::A_PIECES * PL::A_BYTES); };
  auto a_raw = [&](int s) {
    return sbase + (uint32_t)(s * PL::STAGE + PL::A_PIECES * PL::A_BYTES + PL::B_BYTES);
  };

  if (warp == 4) {
    if (lane == 0) {                          // TMA producer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % LT_ST, use = kb / LT_ST;
        if (use > 0) tc::mbar_wait(&empty[s], (use - 1) & 1);
        tc::mbar_expect_tx(&full[s], (uint32_t)((LT_BM + NB) * LT_BK * 4));   // A box + B box
        const int k0 = kbeg + kb * LT_BK;
        if constexpr (AT)
          tc::tma_load_2d(a_raw(s), &p.amap, m0, k0, &full[s]);   // 32 k-rows x 128 m (512 B)
        else
          tc::tma_load_2d(a_hi(s), &p.amap, k0, m0, &full[s]);    // 128 rows x 128 B
        tc::tma_load_2d(b_st(s), &p.bmap, k0, (int)blockIdx.z * NB, &full[s]);   // NB rows (hi)
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {                          // MMA issuer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % LT_ST, use = kb / LT_ST;
        tc::mbar_wait(&conv[s], use & 1);
        tc::tc_fence_after();
        const uint32_t dbig = tmem + (uint32_t)((kb & 1) * 2 * NB);
#pragma unroll
        for (int kq = 0; kq < LT_BK / 8; ++kq) {
          const uint64_t da = sw128_desc(a_hi(s) + 32 * kq);
          const uint64_t db = sw128_desc(b_st(s) + 32 * kq);
          if constexpr (PL::TS) {
            mma_ss(dbig, da, db, ID_FULL, (kb < 2 && kq == 0) ? 0u : 1u);
            tc::mma_ts(dbig + NB, tmem + (uint32_t)(PL::LO_COL + s * LT_BK + 8 * kq), db, ID_HALF, 1u);
          } else {
            const uint64_t dl = sw128_desc(a_lo(s) + 32 * kq);
            mma_ss(dbig, da, db, ID_FULL, (kb < 2 && kq == 0) ? 0u : 1u);
            mma_ss(dbig + NB, dl, db, ID_HALF, 1u);
          }
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&done);
    }
  } else {                                    // warps 0-3: the lo pieces
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % LT_ST, use = kb / LT_ST;
      tc::mbar_wait(&full[s], use & 1);
      if constexpr (AT) {
        // A from the raw [32 k][128 m] tile: unit (m, 4-k chunk c) -> row m,
        // 16-byte column c ^ (m % 8) of the swizzled K-major hi and lo tiles
        // (lanes = consecutive m: conflict-free reads and writes)
        // thread t owns row m = t (its TMEM lane): hi chunks to smem, the 32
        // lo pieces to TMEM columns LO_COL + 32 s ..
        const int m = t;
        float lo[LT_BK];
#pragma unroll
        for (int c = 0; c < LT_BK / 4; ++c) {
          float v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            asm volatile("ld.shared.f32 %0, [%1];"
                         : "=f"(v[i]) : "r"(a_raw(s) + (uint32_t)(((4 * c + i) * LT_BM + m) * 4)));
          const uint32_t off = (uint32_t)(m * 128 + ((c ^ (m & 7)) << 4));
          tc::st_shared_v4(a_hi(s) + off, make_float4(v[0], v[1], v[2], v[3]));
#pragma unroll
          for (int i = 0; i < 4; ++i) lo[4 * c + i] = tc::tf32_lo(v[i]);
        }
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(PL::LO_COL + s * LT_BK);
        tc::tmem_st16(ta, lo);
        tc::tmem_st16(ta + 16, lo + 16);
        tc::tmem_wait_st();
      } else {
        // A (W rows by TMA, swizzled K-major): row t's lo pieces to its TMEM lane
        float lo[LT_BK];
#pragma unroll
        for (int c = 0; c < LT_BK / 4; ++c) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(a_hi(s) + (uint32_t)(t * 128 + ((c ^ (t & 7)) << 4))));
          lo[4 * c] = tc::tf32_lo(v.x);
          lo[4 * c + 1] = tc::tf32_lo(v.y);
          lo[4 * c + 2] = tc::tf32_lo(v.z);
          lo[4 * c + 3] = tc::tf32_lo(v.w);
        }
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(PL::LO_COL + s * LT_BK);
        tc::tmem_st16(ta, lo);
        tc::tmem_st16(ta + 16, lo + 16);
        tc::tmem_wait_st();
      }
      // B: hi rows 0..NB-1, lo rows NB..2NB-1 -- the swizzle pattern repeats
      // every 8 rows, so lo is hi's bytes shifted by NB rows
      for (int i = t; i < NB * LT_BK / 4; i += 128) {
        const uint32_t src = b_st(s) + 16 * i;
        const uint32_t dst = src + NB * 128;
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src));
        tc::st_shared_v4(dst, make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z),
                                          tc::tf32_lo(v.w)));
      }
      tc::fence_proxy_async();                // generic smem writes -> tensor-core reads
      if constexpr (PL::TS) tc::tc_fence_before();   // TMEM stores -> the MMA thread
      tc::mbar_arrive(&conv[s]);
      if (kb == 0) {
        LT_MARK(2)
      }
    }
  }

  // ---- epilogue: accumulators -> this CTA's partial tile, staged [NB][128]
  __syncthreads();                            // all roles done issuing
  tc::mbar_wait(&done, 0);
  tc::tc_fence_after();
  LT_MARK(3)
  float *stage = reinterpret_cast<float *>(smem + (sbase - tc::smem_u32(smem)));
  if (warp < 4) {
    const int row = warp * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    const bool two = nkb > 1;
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
      for (int j = 0; j < 16; ++j) {
        float v = two ? __fadd_rn(__fadd_rn(s0[j], s1[j]), __fadd_rn(b0[j], b1[j]))
                      : __fadd_rn(s0[j], b0[j]);
        stage[(c + j) * LT_BM + row] = nkb > 0 ? v : 0.f;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(PL::TMEM)
                 : "memory");
  LT_MARK(4)
  // ---- cluster reduction: rank r owns batch rows j = r, r + cl, ... and sums
  // the ranks' partials in rank order (deterministic)
  if (cl > 1) tc::cluster_sync();
  // float4 units (batch row j, 4 consecutive weight rows); up to 4 units per
  // thread with every remote and global load in flight before any use
  const int njj = (NB - rank + cl - 1) / cl;          // batch rows rank, rank + cl, ...
  const int units = njj * (LT_BM / 4);
  for (int u0 = t; u0 < units; u0 += 4 * LT_THREADS) {
    float4 acc[4], aux[4];
    bool ok[4];
    int64_t off[4];
    int mm[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int u = u0 + h * LT_THREADS;
      const int jj = u / (LT_BM / 4), r4 = (u - jj * (LT_BM / 4)) * 4;
      const int j = rank + jj * cl;
      mm[h] = m0 + r4;
      ok[h] = u < units && (int)blockIdx.z * NB + j < p.nrows && mm[h] < p.M;
      off[h] = ((int64_t)blockIdx.z * NB + j) * p.M + mm[h];
      const int sidx = j * LT_BM + r4;
      acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      aux[h] = make_float4(1.f, 1.f, 1.f, 1.f);
      if (!ok[h]) continue;
      if (cl > 1) {
        const uint32_t la = tc::smem_u32(&stage[sidx]);
        float4 r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < cl) r[q] = tc::ld_dsmem4(tc::dsmem_addr(la, q));
        acc[h] = r[0];
#pragma unroll
        for (int q = 1; q < 16; ++q)
          if (q < cl) {
            acc[h].x = __fadd_rn(acc[h].x, r[q].x); acc[h].y = __fadd_rn(acc[h].y, r[q].y);
            acc[h].z = __fadd_rn(acc[h].z, r[q].z); acc[h].w = __fadd_rn(acc[h].w, r[q].w);
          }
      } else {
        acc[h] = *reinterpret_cast<const float4 *>(&stage[sidx]);
      }
      if (p.mode == 0)
        aux[h] = *reinterpret_cast<const float4 *>(p.bias + mm[h]);
      else if (p.mask)
        aux[h] = *reinterpret_cast<const float4 *>(p.mask + off[h]);
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (!ok[h]) continue;
      float v[4] = {acc[h].x, acc[h].y, acc[h].z, acc[h].w};
      const float a4[4] = {aux[h].x, aux[h].y, aux[h].z, aux[h].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (p.mode == 0) {
          v[e] = __fadd_rn(v[e], a4[e]);
          if (p.relu && v[e] < 0.f) v[e] = 0.f;
        } else if (p.mask && !(a4[e] > 0.f)) {
          v[e] = 0.f;
        }
      }
      *reinterpret_cast<float4 *>(p.out + off[h]) = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  if (cl > 1) tc::cluster_sync();             // peers' staged partials read
  LT_MARK(5)
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn lt_encode() {
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

// [rows][K] fp32, row stride K: boxes of 32 k (128 B) x box_rows rows in the
// 128-byte-swizzle layout (sw128_desc)
bool lt_map(CUtensorMap *m, const float *base, int K, int rows, int box_rows) {
  const EncodeTiledFn fn = lt_encode();
  if (!fn || ((uintptr_t)base % 16) || (K % 4)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  const cuuint32_t box[2] = {LT_BK, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// W [K][M] fp32 (M contiguous) read as raw [32 k][128 m] tiles (no swizzle)
bool lt_map_t(CUtensorMap *m, const float *base, int M, int K) {
  const EncodeTiledFn fn = lt_encode();
  if (!fn || ((uintptr_t)base % 16) || (M % 4)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  const cuuint64_t strides[1] = {(cuuint64_t)M * 4};
  const cuuint32_t box[2] = {LT_BM, LT_BK};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K split across a cluster of up to 16 CTAs (non-portable above 8), a
// multiple of LT_BK per rank
template <int NB, bool AT>
int lt_launch(cudaStream_t st, LinTcArgs &a, int cl, const char *what) {
  using PL = LtPlan<NB, AT>;
  auto kern = lin_tc_kernel<NB, AT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::BYTES);
    if (e != cudaSuccess) return cuda_status(e, what);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_status(e, what);
    configured = true;
  }
  const int chunks = (a.K + LT_BK - 1) / LT_BK;
  cl = std::max(1, std::min(cl, chunks));
  a.klen = ((chunks + cl - 1) / cl) * LT_BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.M + LT_BM - 1) / LT_BM, cl, (a.nrows + NB - 1) / NB);
  cfg.blockDim = dim3(LT_THREADS);
  cfg.dynamicSmemBytes = PL::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  attr[2].id = cudaLaunchAttributeClusterDimension;
  attr[2].val.clusterDim.x = 1;
  attr[2].val.clusterDim.y = cl;
  attr[2].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 3;
  cudaLaunchKernelEx(&cfg, kern, a);
  DQN_LAUNCH_CHECK(what);
  return DQN_OK;
}

template <bool AT>
int lt_run(cudaStream_t st, LinTcArgs &a, int nb, int cl, const char *what) {
  if (nb <= 16) return lt_launch<16, AT>(st, a, cl, what);
  if (nb <= 32) return lt_launch<32, AT>(st, a, cl, what);
  return lt_launch<64, AT>(st, a, cl, what);
}

inline int lt_rows(int nb) { return nb <= 16 ? 16 : (nb <= 32 ? 32 : 64); }

}  // namespace

// K-split cluster sizes: 16 CTAs, and 4 for a side trunk (DQN_NET_HINT_SIDE:
// the learner's target forward, which runs beside the online one on the
// critical path -- 16-CTA clusters there tie up whole GPCs the online launch
// then waits for).  Measured in the learner graph (cfg4): small / big =
// 16/16 6,676, 8/16 6,961, 4/16 6,989-7,003, 2/16 6,481, 1/16 5,370,
// 8/8 6,857, 4/8 6,858, 16/8 6,856, 12/16 6,713 updates/s (trace build).
#ifdef DQN_TC_TRACE
int g_lt_cl_small = 4, g_lt_cl_big = 16;     // diagnostic overrides
int g_lt_max_batch = 1 << 20, g_lt_cl_large = 0;   // 0: the fill rule
int g_ltd_min_batch = 64;                            // dgrad: lin_tc above this batch
int g_ltd_fill = 128;
#else
constexpr int g_lt_cl_small = 4, g_lt_cl_big = 16;
constexpr int g_lt_max_batch = 1 << 20, g_lt_cl_large = 0;
constexpr int g_ltd_min_batch = 64;
constexpr int g_ltd_fill = 128;
#endif

// hidden linear layer at learner batch sizes (<= 64 rows), weights rows >= 128
bool lin_tc_ok(const dqn_layer_desc &L, int batch) {
  const int F = L.in_h * L.in_w * L.in_c;
  return L.kind == DQN_LAYER_LINEAR && batch >= 1 && batch <= g_lt_max_batch && F % 4 == 0 &&
         L.out_c % 4 == 0 && F >= 128 && L.out_c >= 128;
}

// y [batch][N] = act(x [batch][F] W[F][N] + b): the weights tile read as
// [32 k][128 n] and transposed into the K-major A operand in shared memory
int lin_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const float *x, const float *params,
                   float *y, int batch, bool side) {
  const int F = L.in_h * L.in_w * L.in_c, N = L.out_c;
  const int nb = lt_rows(batch);
  LinTcArgs a{};
  if (!lt_map_t(&a.amap, params + L.w_off, N, F) || !lt_map(&a.bmap, x, F, batch, nb))
    return DQN_ERR_UNSUPPORTED;
  a.M = N;
  a.K = F;
  a.nrows = batch;
  a.mode = 0;
  a.bias = params + L.b_off;
  a.relu = L.relu;
  a.out = y;
  // K split over a cluster: 4 weight tiles x 16 = 64 CTAs for fc1 at batch 64
  // (measured alone: 8-CTA clusters 15.6 us, 16-CTA 11.0 us)
  // above batch 64: 64-row blocks of the batch on blockIdx.z and a K split
  // for ~128 CTAs (measured at B = 256 / 1024 / 4096: 21.9 / 39.2 / 136 us with
  // splits 4 / 2 / 1, the generic engine 37.4 / 75.4 / 246 us)
  int cl = side ? g_lt_cl_small : g_lt_cl_big;
  if (batch > 64) {
    const int ctas = ((N + LT_BM - 1) / LT_BM) * ((batch + 63) / 64);
    cl = g_lt_cl_large > 0 ? g_lt_cl_large : std::max(1, std::min(16, (128 + ctas - 1) / ctas));
  }
  return lt_run<true>(st, a, nb, cl, "lin_tc_forward");
}

// dX [batch][F] = mask(dY [batch][N] W[F][N]^T) above learner batch sizes: W's
// rows are K-major for this product and arrive as 128B-swizzle boxes (no
// transpose), 64-row batch blocks on blockIdx.z.  (At batch 32 the engine's
// LinDgradTmaPol is faster in the learner: DESIGN.md section 5.)
int lin_tc_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
                 const float *mask, float *dx, int batch) {
  if (batch <= g_ltd_min_batch || !lin_tc_ok(L, batch)) return DQN_ERR_UNSUPPORTED;
  const int F = L.in_h * L.in_w * L.in_c, N = L.out_c;
  const int nb = lt_rows(batch);
  LinTcArgs a{};
  if (!lt_map(&a.amap, w, N, F, LT_BM) || !lt_map(&a.bmap, dy, N, batch, nb))
    return DQN_ERR_UNSUPPORTED;
  a.M = F;
  a.K = N;
  a.nrows = batch;
  a.mode = 1;
  a.mask = mask;
  a.out = dx;
  const int ctas = ((F + LT_BM - 1) / LT_BM) * ((batch + nb - 1) / nb);
  return lt_run<false>(st, a, nb, std::max(1, std::min(16, (g_ltd_fill + ctas - 1) / ctas)),
                       "lin_tc_dgrad");
}

}  // namespace dqn


#ifdef DQN_TC_TRACE
extern "C" void dqn_lt_set_cluster(int small, int big) {
  dqn::g_lt_cl_small = small;
  dqn::g_lt_cl_big = big;
}
extern "C" void dqn_ltd_set_min_batch(int b) { dqn::g_ltd_min_batch = b; }
extern "C" void dqn_ltd_set_fill(int f) { dqn::g_ltd_fill = f; }
extern "C" void dqn_lt_set_large(int max_batch, int cl) {
  dqn::g_lt_max_batch = max_batch;
  dqn::g_lt_cl_large = cl;
}
extern "C" int dqn_lt_trace(unsigned long long *host) {
  return (int)cudaMemcpyFromSymbol(host, dqn::g_lt_trace, sizeof(dqn::g_lt_trace));
}
#endif
