// tcgen05 (5th-gen tensor core) implicit-GEMM engine for sm_100a.
//
// One CTA computes a 128 x BN tile of C = A * B^T (A: M x K, B: N x K in
// "math" orientation), fp32 in and out, with ~fp32 accuracy from 3xTF32:
//   x = hi + lo, hi = the top 19 bits of x (what a kind::tf32 MMA reads of an
//   fp32 operand -- measured: it truncates, so x itself serves as hi),
//   lo = x - hi, and A*B ~ hi*hi + hi*lo + lo*hi.
//
// Data paths (measured on B200: the 128 B/clk L1/shared-memory datapath is
// the limit of a register gather that stages both operands in shared memory,
// and a kind::tf32 MMA costs ~51 cycles for any N <= 64, 64 at N = 128):
//   * A lives in tensor memory (the "TS" MMA form): a producer thread owns one
//     tile row and a 16-k half of each 32-k block, loads its 16 values, and
//     writes hi and lo with tcgen05.st (lane = row, column = k) -- A never
//     touches shared memory;
//   * B is gathered through registers into shared memory in the canonical
//     no-swizzle K-major layout with its pieces stacked along N
//     ([B_hi ; B_lo], 2*BN rows), so one MMA A_hi * [B_hi ; B_lo] (N = 2*BN)
//     yields hi*hi and hi*lo side by side in TMEM and a second, A_lo * B_hi
//     (N = BN), adds lo*hi to the small-term half: 2 MMAs per 8-k step
//     instead of 3;
//   * accuracy: the residual error is dominated by the tensor pipe's
//     accumulation rounding, so hi*hi and the small terms accumulate in
//     separate TMEM columns and k-blocks round-robin over `nacc` accumulator
//     pairs; the epilogue sums them in fp32 in a fixed order (~5e-7 relative
//     vs fp32 SIMT per GEMM; a single bf16/tf32 pass misses
//     the 1e-3 one-step parity bar).
// Warp roles: kGroups producer groups of 8 warps gather alternating k-blocks
// (two k-blocks of loads in flight per thread) into a STAGES-deep ring (A
// columns in TMEM, B tiles in shared memory) and arrive on full[s]; the
// group's first thread waits full[s], issues the MMAs into the group's own
// accumulator pair and commits to empty[s].  No block-wide barrier inside the
// K loop.
// The epilogue reads TMEM with tcgen05.ld, stages the tile row-major in shared
// memory and hands coalesced float4s to the Policy (bias / ReLU / mask /
// split-K partial / gradient accumulate).  Exact operands (uint8 pixels) use
// one piece.
#pragma once

#include "common.cuh"

#include <cuda.h>

#include <stdlib.h>

namespace dqn {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                  // k per pipeline stage (8 MMA k-steps of 8)
constexpr int kKc = BK / 4;             // 16-byte k-chunks per row of a stage
constexpr int kGroupThreads = 256;      // 8 warps: lane quarter w % 4, k-half w / 4
constexpr int kGroups = 2;
constexpr int kProducers = kGroups * kGroupThreads;
// no separate MMA warp: thread 0 of group g issues the MMAs of its own
// k-blocks into accumulator pair g (16 warps = 4 per SMSP keep the 128
// register/thread budget; a 17th warp would cut it to 96)
constexpr int kThreads = kProducers;
constexpr int kNacc = kGroups;          // accumulator pairs, one per group
constexpr int kTmemCols = 512;          // accumulators + A stages (one CTA per SM)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// TMA 2-D tile load (cp.async.bulk.tensor), completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// TMA 4-D tile load (coordinates innermost first)
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, int c3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// No-swizzle shared-memory matrix descriptor (version 1 for sm_100).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;           // descriptor version (sm_100)
  return d;                         // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Instruction descriptor: kind::tf32, fp32 accumulate, M = 128, both K-major
// (kind::tf32 has no transposed operands: an MN-major B reads as zero).
__host__ __device__ constexpr uint32_t make_idesc_tf32(int n) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(BM >> 4) << 24); // M >> 4
}

// D[tmem] (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float v[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive columns of this thread's TMEM lane (warp-collective)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float v[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ float tf32_lo(float x) { return __fsub_rn(x, tf32_hi(x)); }

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w));
}

// hi piece (x itself: the MMA reads its top 19 bits) and lo = x - hi (the
// MMA reads the top 11 significant bits of lo)
__device__ __forceinline__ void store_split(uint32_t base, uint32_t piece_stride, float4 v,
                                            int pieces) {
  st_shared_v4(base, v);
  if (pieces > 1)
    st_shared_v4(base + piece_stride,
                 make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w)));
}

// Byte offset of a 16-byte chunk (row, 4 consecutive k) inside a K-major
// operand tile with R rows x BK k: core matrices of 8 rows x 16 B; LBO = R*16
// (stride between the two 16-B k-chunks of one MMA k-step), SBO = 128
// (stride between 8-row groups).
__device__ __forceinline__ uint32_t chunk_off(int R, int row, int k) {
  return (uint32_t)((k >> 2) * (R * 16) + (row >> 3) * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint64_t op_desc(uint32_t base, int R, int kstep) {
  return make_sdesc(base + kstep * 2 * R * 16, R * 16, 128);
}

// B chunks are gathered cooperatively: chunk c (16 B = row, 4 k) of an
// R x BK tile is owned by thread c % 256 of a producer group, so every thread
// owns the same rows in every k-block (row bases are computed once per CTA).
// A quarter-warp writes one contiguous 128-byte smem line (8 rows of one k-chunk).
__device__ __forceinline__ void chunk_coords(int c, int &row, int &k) {
  const int r8 = c & 7, kc = (c >> 3) % kKc, rg = c / (8 * kKc);
  row = rg * 8 + r8;
  k = kc * 4;
}

// thread-block cluster helpers (split-K reduced through distributed smem)
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ float comp(const float4 &v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// Gathers the BN x BK B tile of a k-block into registers and stores it
// K-major with its pieces stacked along N (layout rows RL = pieces * BN;
// piece p of row n is layout row p * BN + n).  Units are owned by thread
// (u + rot) % 256 of a producer group with the same rows in every k-block.
//  * MNC == false (source contiguous along k): unit = chunk (row, 4 k), one
//    16-byte load via ld(base, koff(k)); all units of a thread share k, so
//    the k-dependent address part is computed once per k-block;
//  * MNC == true (source contiguous along rows, e.g. W[k][n] or dY[pix][co]):
//    unit = 4 rows x 4 k, four 16-byte loads along the rows via
//    f4(base, k, kend, v[4]) (consecutive lanes = consecutive row quads =
//    coalesced), transposed in registers into four K-major chunks.
// Optionally accumulates the per-row sums of everything stored (bias grads).
template <bool MNC, int R, int RL>
struct Gather {
  static constexpr int UNITS = MNC ? R * BK / 16 : R * BK / 4;
  static constexpr int U = (UNITS + kGroupThreads - 1) / kGroupThreads;
  static constexpr int V = MNC ? 4 : 1;
  static_assert(!MNC || U == 1, "MNC gathers assume one unit per thread");
  long long base[U];
  int t0;                      // this thread's first unit (rotated, see init)
  uint32_t soff[U];            // byte offset of the unit's (first) chunk in the tile
  int kk;                      // the thread's k offset inside a k-block (same for all units)
  float bsum[U][V];
  using Regs = float4[U][V];   // one k-block's values (the caller double-buffers them)

  __device__ static void coords(int u, int &row, int &k) {
    if (!MNC) {
      chunk_coords(u, row, k);
    } else {
      const int q = u % (R / 4), kc = u / (R / 4);
      row = 4 * q;
      k = 4 * kc;
    }
  }
  template <class RowFn>
  __device__ void init(RowFn rowfn, int rot) {
    t0 = (threadIdx.x % kGroupThreads + kGroupThreads - rot) % kGroupThreads;
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int u = t0 + i * kGroupThreads;
      int row, k;
      coords(u, row, k);
      base[i] = u < UNITS ? rowfn(row) : -1;
      soff[i] = chunk_off(RL, row, k);
      kk = k;
#pragma unroll
      for (int j = 0; j < V; ++j) bsum[i][j] = 0.f;
    }
  }
  template <class KF, class LD, class F4>
  __device__ void fetch(Regs &v, int k0, int kend, KF &&koff, LD &&ld, F4 &&f4) {
    const int k = k0 + kk;
    if constexpr (!MNC) {
      const bool in = k < kend;
      const int ko = in ? koff(k) : 0;
#pragma unroll
      for (int i = 0; i < U; ++i)
        v[i][0] = (in && base[i] >= 0) ? ld(base[i], ko) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        if (base[i] < 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) v[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          f4(base[i], k, kend, v[i]);
        }
      }
    }
  }
  __device__ void store(const Regs &v, uint32_t tile, uint32_t piece_stride, int pieces,
                        bool bias) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (t0 + i * kGroupThreads >= UNITS) continue;
      if constexpr (!MNC) {
        store_split(tile + soff[i], piece_stride, v[i][0], pieces);
        if (bias)
          bsum[i][0] = __fadd_rn(bsum[i][0], __fadd_rn(__fadd_rn(v[i][0].x, v[i][0].y),
                                                       __fadd_rn(v[i][0].z, v[i][0].w)));
      } else {
        float4 c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          c[j] = make_float4(comp(v[i][0], j), comp(v[i][1], j), comp(v[i][2], j),
                             comp(v[i][3], j));                     // row row + j
          if (bias)
            bsum[i][j] = __fadd_rn(bsum[i][j], __fadd_rn(__fadd_rn(c[j].x, c[j].y),
                                                         __fadd_rn(c[j].z, c[j].w)));
        }
        // Store the four chunks in a lane-rotated order: at each store the
        // warp's rows then cover all 8 rows of a core matrix (row % 8), so the
        // 16-byte stores hit all 32 banks (4 wavefronts instead of 16).
        const int rot = (int)(soff[i] >> 7) & 3;          // (row / 8) % 4
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = (t + rot) & 3;
          const float4 cj = (j & 2) ? ((j & 1) ? c[3] : c[2]) : ((j & 1) ? c[1] : c[0]);
          store_split(tile + soff[i] + 16 * j, piece_stride, cj, pieces);
        }
      }
    }
  }
  template <int RR>
  __device__ void dump_bias(float (&red)[RR][kKc]) const {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int u = t0 + i * kGroupThreads;
      if (u >= UNITS) continue;
      int row, k;
      coords(u, row, k);
#pragma unroll
      for (int j = 0; j < V; ++j)
        if (row + j < RR) red[row + j][k >> 2] = bsum[i][j];
    }
  }
};

// Policies derive from this; it supplies the B gather form a policy does not
// use (never called: the Gather uses the form of its layout).
struct PolBase {
  static constexpr bool B_TMA = false;   // B hi tiles by TMA tensor loads (K-major dense B)
  // issue the TMA load of B's hi rows n0.. for the 4-k chunk at k (problem zp)
  __device__ void b_tma(uint32_t, int, int, int, uint64_t *) const {}
  __device__ int rows(int) const { return 0x7fffffff; }   // problem height (grouped launches)
  __device__ void note_bias(float) const {}      // BIAS_FROM_B: the written bias gradient
  __device__ int b_koff(int) const { return 0; }
  __device__ float4 b_ld(long long, int) const { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ void b4(long long, int, int, float4 (&)[4]) const {}
};

// Split-K tiles count arrivals (and finished reducers) in a per-binding int
// table (the tail of the binding scratch, zero-initialised, two ints per
// tile); the last reducer resets them, so the table is all-zero between
// launches (graph-replay safe) and two kernels on different streams with
// different bindings never share counters.
constexpr int kMaxTiles = 16384;

// Split-K reducers per tile: the last R = budget / tiles + 1 arrivals (<= 8,
// <= splits) each reduce a slice; R - 1 of them wait for the final arrival
// on their SM, at most `budget` CTAs per launch (deadlock-free beside another
// launch).  A kernel argument (reducer_budget(): 60).

// Shared/tensor memory plan of a policy.
template <class Pol>
struct Plan {
  static constexpr int BN = Pol::BN;
  static constexpr int NA = Pol::SPLIT_A ? 2 : 1, NB = Pol::SPLIT_B ? 2 : 1;
  static constexpr int RB = NB * BN;                   // stacked B rows (<= 256)
  static constexpr int B_BYTES = RB * BK * 4;
  static constexpr int A_COLS = NA * BK;               // TMEM columns per A stage
  static constexpr int STAGES_SMEM = (200 * 1024) / B_BYTES;
  static constexpr int STAGES_TMEM = (kTmemCols - 2 * kNacc * BN) / A_COLS;
  static constexpr int S0 = STAGES_SMEM < STAGES_TMEM ? STAGES_SMEM : STAGES_TMEM;
  // an even ring: the two producer groups alternate k-blocks, so every slot
  // stays with one group, and a group is never more than one phase ahead of a
  // slot's empty barrier.  With an odd ring a slot alternates between groups:
  // group 0 can reach its use 2 of slot 0 (waiting for parity 1) before use 0
  // completed -- the barrier is still in phase 0, parity 0 != 1, so the
  // parity wait passes at once and the slot is overwritten under the MMAs
  // (measured: LinDgradPol<32> with 3 stages raced).
  static constexpr int STAGES = (S0 > 4 ? 4 : S0) & ~1;
  static_assert(STAGES >= kGroups, "one ring slot per producer group at least");
  static_assert(RB <= 256 && RB % 16 == 0 && BN % 16 == 0, "MMA N limits");
  static constexpr int ACC_MAX = kTmemCols - STAGES * A_COLS;   // columns for accumulators
  static_assert(2 * kNacc * BN <= ACC_MAX, "accumulator pairs do not fit in TMEM");
  static constexpr int EPI_STRIDE = BN + 4;                      // floats per staged row
  static constexpr int EPI_BYTES = BM * EPI_STRIDE * 4;
  static constexpr int PIPE = STAGES * B_BYTES;
  static constexpr int BYTES = PIPE > EPI_BYTES ? PIPE : EPI_BYTES;
};

// Policy interface (all __device__, const):
//   static constexpr int BN; static constexpr bool SPLIT_A, SPLIT_B, BIAS_FROM_B, B_MNC;
//   int M, N, ksplits;  int kbeg(split), kend(split);
//   float *partial ([problems][ksplits][M][N] when ksplits > 1)
//   gridDim.z = problems * ksplits; a_row/b_row/final4 get the problem index
//   long long a_row(m) / b_row(n)          -- per-row base (-1: row out of range)
//   void a16(base, k, kend, float v[16])   -- A[row][k..k+15] (zero beyond kend;
//                                             k is a multiple of 16)
//   B K-major: int b_koff(k), float4 b_ld(base, koff) -- B[row][k..k+3];
//   B MN-contiguous: b4(base, k, kend, v[4]) -- rows base..+3 at k..k+3
//   void final4(m, n, float4 v)            -- epilogue for columns n..n+3 of row m
//   BIAS_FROM_B: float *bias_out (+= column sums of B over k), *bias_partial
// nacc: the K loop of a tile round-robins its k-blocks over nacc TMEM
// accumulator pairs that the epilogue sums in fixed order -- shorter
// tensor-core accumulation chains for ~fp32-SIMT accuracy on long reductions.
#ifdef DQN_TC_TRACE
// per-CTA record: {ctaid, smid, t_entry, t_setup, t_kloop, t_epilogue, t_exit, nk,
//                  t_first_store (producer 0), t_first_full (MMA warp), t_last_mma, launch id}
constexpr int kTraceCtas = 8192;
__device__ unsigned long long g_trace[kTraceCtas * 30];
__device__ unsigned int g_trace_n;
__device__ int g_skip;        // diagnostic: 1 = no MMAs, 2 = no global loads, 4 = no operand stores,
                              // 8 = no A stores to TMEM, 16 = no B stores to smem
#define TC_SKIP(bit) (g_skip & (bit))
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC_MARK(i) \
  if (threadIdx.x == 0) tr_[i] = gtimer();
#else
#define TC_SKIP(bit) false
#define TC_MARK(i)
#endif

template <class Pol>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ Pol p,
                                                               const int launch_id,
                                                               const int cluster_ks, const int reducer_budget) {
  using PL = Plan<Pol>;
  constexpr int nacc = kNacc;
  constexpr int BN = Pol::BN, STAGES = PL::STAGES, NA = PL::NA, NB = PL::NB, RB = PL::RB;
  constexpr int B_BYTES = PL::B_BYTES;
  constexpr uint32_t IDESC_FULL = make_idesc_tf32(RB), IDESC_HALF = make_idesc_tf32(BN);
  extern __shared__ __align__(1024) uint8_t smem[];
  // full[s]: the producer group that filled slot s is done (256 arrivals);
  // empty[s]: the MMAs reading slot s completed (tcgen05.commit); done: all
  // MMAs of every group
  __shared__ uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint64_t tbar[Pol::B_TMA ? STAGES : 1];     // TMA B tile landed
  __shared__ uint32_t tmem_slot;
  __shared__ float bias_red[Pol::BIAS_FROM_B ? kGroups : 1][Pol::BIAS_FROM_B ? BN : 1][kKc];

#ifdef DQN_TC_TRACE
  unsigned long long tr_[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long tk_[16];             // group 0, k-blocks 0, 2, 4, 6: enter, empty ok, arrived, mma issued
#pragma unroll
  for (int j = 0; j < 16; ++j) tk_[j] = 0;
  __shared__ unsigned long long tr_mma[2];
#endif
  TC_MARK(0)
  // problems of different heights share the grid: tiles past a problem's
  // rows exit before touching TMEM, barriers or split-K counters
  if ((int)blockIdx.x * BM >= p.rows((int)blockIdx.z / p.ksplits)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
#ifdef DQN_TC_TRACE
  unsigned long long t_alloc = 0, t_presync = 0;
  if (threadIdx.x == 0) t_alloc = gtimer();
#endif
  if (threadIdx.x == 32) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kGroupThreads);
      mbar_init(&empty[s], 1);
      if constexpr (Pol::B_TMA) mbar_init(&tbar[s], 1);
    }
    mbar_init(&done, kGroups);
    fence_barrier_init();
  }

  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, z = blockIdx.z;
  // blockIdx.z = problem * ksplits + split: a split of K (partials +
  // last-CTA fixup) and an independent problem index (e.g. a stride phase)
  const int ks = p.ksplits, zs = z % ks, zp = z / ks;
  const bool SPLITK = ks > 1;
  const int kbeg = p.kbeg(zs), kend = p.kend(zs);
  float *const part = p.partial + (SPLITK ? (int64_t)zp * ks * p.M * p.N : 0);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const uint32_t sbase = smem_u32(smem);
  constexpr bool producer = true;        // every warp gathers
  const int group = threadIdx.x / kGroupThreads;
  // A ownership: TMEM lane quarter = warp % 4 (the warp's accessible lanes),
  // k-half = (warp / 4) % 2 of each 32-k block
  const int quarter = warp & 3, khalf = (warp >> 2) & 1;
  const int arow = quarter * 32 + lane;

  long long abase = -1;
  Gather<Pol::B_MNC, BN, RB> gb;
  if (producer) {
    abase = p.a_row(m0 + arow, zp);
    gb.init([&](int r) { return p.b_row(n0 + r, zp); }, 0);
  }

#ifdef DQN_TC_TRACE
  if (threadIdx.x == 0) t_presync = gtimer();
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // everything above (TMEM allocation, barriers, row bases from kernel
  // parameters) overlapped the previous kernel; operands are read only now
  pdl_wait();
  const uint32_t tmem = tmem_slot;
  // accumulator pairs [big | small] at columns a * 2BN, A stages after them
  const uint32_t acol0 = (uint32_t)PL::ACC_MAX;
  const bool want_bias = Pol::BIAS_FROM_B && blockIdx.x == 0;
  TC_MARK(1)

  if (producer) {
    // group g gathers k-blocks g, g + kGroups, ... into ring slot kb % STAGES;
    // a slot is refilled once the MMAs of k-block kb - STAGES completed.
    // One register buffer per thread: a 64-k block's loads are in flight
    // while the previous block is stored and multiplied.
    using GB = Gather<Pol::B_MNC, BN, RB>;
    constexpr int AR = BK / 32;                  // 16-runs of A per thread
    float av[AR][16];
    typename GB::Regs bv;
    auto fetch = [&](int kb) {
      if (TC_SKIP(2)) return;
      const int k0 = kbeg + kb * BK;
#pragma unroll
      for (int h = 0; h < AR; ++h) {
        if (abase >= 0) {
          p.a16(abase, k0 + (BK / 2) * khalf + 16 * h, kend, av[h]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) av[h][j] = 0.f;
        }
      }
      if constexpr (!Pol::B_TMA)
        gb.fetch(bv, k0, kend, [&](int k) { return p.b_koff(k); },
                 [&](long long b, int ko) { return p.b_ld(b, ko); },
                 [&](long long b, int k, int ke, float4 (&v)[4]) { p.b4(b, k, ke, v); });
    };
    // the B hi tile of k-block kb by TMA (group leader): one 4-k x BN-row box
    // per 16-byte k-chunk, straight into the canonical K-major layout's hi
    // rows (chunk c at c * RB * 16, row r at r * 16); rows / k beyond the
    // tensor are zeros.  Issued one k-block ahead, right after the previous
    // block's MMAs, so the load overlaps that block's A store and MMAs.
    auto issue_b = [&](int kb) {
      if constexpr (Pol::B_TMA) {
        if (TC_SKIP(16)) return;
        const int s = kb % STAGES, use = kb / STAGES;
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);  // MMAs of kb - STAGES done
        fence_proxy_async();
        mbar_expect_tx(&tbar[s], (uint32_t)(BN * BK * 4));
        const int k0 = kbeg + kb * BK;
#pragma unroll 1
        for (int c = 0; c < kKc; ++c)
          p.b_tma(sbase + s * B_BYTES + c * RB * 16, n0, k0 + 4 * c, zp, &tbar[s]);
      }
    };
    auto put = [&](int kb) {
      const int s = kb % STAGES, use = kb / STAGES;
#ifdef DQN_TC_TRACE
      const bool tk = threadIdx.x == 0 && kb < 8;
      if (tk) tk_[(kb >> 1) * 4 + 0] = gtimer();
#endif
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);    // MMAs of kb - STAGES done
#ifdef DQN_TC_TRACE
      if (tk) tk_[(kb >> 1) * 4 + 1] = gtimer();
#endif
      tc_fence_after();
#ifdef DQN_TC_TRACE
      if (kb == 0 && threadIdx.x == 0) tr_[5] = gtimer();
#endif
      if (!TC_SKIP(4)) {
        // A: hi (= the values) and lo pieces into this stage's TMEM columns
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + acol0 +
                            (uint32_t)(s * PL::A_COLS + (BK / 2) * khalf);
        if (!TC_SKIP(8)) {
#pragma unroll
          for (int h = 0; h < AR; ++h) {
            tmem_st16(ta + 16 * h, av[h]);
            if (NA > 1) {
              float lo[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) lo[j] = tf32_lo(av[h][j]);
              tmem_st16(ta + BK + 16 * h, lo);
            }
          }
        }
        if constexpr (Pol::B_TMA) {
          if (!TC_SKIP(16)) {
            // lo = x - trunc_tf32(x) of the landed hi rows, into rows BN.. of each chunk
            mbar_wait(&tbar[s], use & 1);
            const uint32_t tb = sbase + s * B_BYTES;
            for (int i = threadIdx.x % kGroupThreads; i < BN * kKc; i += kGroupThreads) {
              const int c = i / BN, r = i - c * BN;
              const uint32_t a = tb + (uint32_t)(c * RB * 16 + r * 16);
              float4 h;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(h.x), "=f"(h.y), "=f"(h.z), "=f"(h.w) : "r"(a));
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a + BN * 16),
                           "f"(tf32_lo(h.x)), "f"(tf32_lo(h.y)), "f"(tf32_lo(h.z)), "f"(tf32_lo(h.w))
                           : "memory");
            }
          }
        } else {
          if (!TC_SKIP(16)) gb.store(bv, sbase + s * B_BYTES, BN * 16, NB, want_bias);
        }
        tmem_wait_st();
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&full[s]);
#ifdef DQN_TC_TRACE
      if (tk) tk_[(kb >> 1) * 4 + 2] = gtimer();
#endif
      // the group's first thread issues its k-block's MMAs into pair `group`
      // (one issuing thread per accumulator chain: fixed order)
      if (threadIdx.x % kGroupThreads == 0) {
        mbar_wait(&full[s], use & 1);
#ifdef DQN_TC_TRACE
        if (kb == 0) tr_mma[0] = gtimer();
#endif
        tc_fence_after();
        if (!TC_SKIP(1)) {
          const uint32_t dbig = tmem + (uint32_t)(group * 2 * BN);
          const uint32_t dsmall = dbig + (uint32_t)BN;
          const uint32_t ta = tmem + acol0 + (uint32_t)(s * PL::A_COLS);
          const uint32_t tb = sbase + s * B_BYTES;
#pragma unroll
          for (int kq = 0; kq < BK / 8; ++kq) {
            const uint64_t db = op_desc(tb, RB, kq);
            const uint32_t first = (kb < kGroups && kq == 0) ? 0u : 1u;
            // hi * [B_hi ; B_lo] -> [big | small]; the first touch of a pair overwrites
            mma_ts(dbig, ta + 8 * kq, db, NB > 1 ? IDESC_FULL : IDESC_HALF, first);
            // lo * B_hi -> small (initialised by the first MMA when B is split)
            if (NA > 1) mma_ts(dsmall, ta + BK + 8 * kq, db, IDESC_HALF, NB > 1 ? 1u : first);
          }
        }
        mma_commit(&empty[s]);
#ifdef DQN_TC_TRACE
        if (tk) tk_[(kb >> 1) * 4 + 3] = gtimer();
#endif
        if (kb + kGroups < nk) issue_b(kb + kGroups);
      }
    };
    if (group < nk && threadIdx.x % kGroupThreads == 0) issue_b(group);
    if (group < nk) fetch(group);
    for (int kb = group; kb < nk; kb += kGroups) {
      put(kb);
      if (kb + kGroups < nk) fetch(kb + kGroups);
    }
    if (threadIdx.x % kGroupThreads == 0) {
#ifdef DQN_TC_TRACE
      if (group == 0) tr_mma[1] = gtimer();
#endif
      mma_commit(&done);       // arrives once this group's MMAs completed
    }
  }
  mbar_wait(&done, 0);
  // the next kernel may be scheduled now (common.cuh): its prologue overlaps
  // this tile's epilogue and split-K fixup, not the K loop
  pdl_trigger();
  TC_MARK(2)
  tc_fence_after();

  // epilogue: TMEM -> registers -> smem (row-major staging) -> coalesced stores
  float *stage = reinterpret_cast<float *>(smem);
  constexpr int ES = PL::EPI_STRIDE;
  // producer warps w, w+4, ... read the same TMEM lane quarter (w % 4) and
  // split the 16-column chunks between them
  constexpr int CGROUPS = kProducers / 128;
  const int cgrp = warp >> 2;
  const int nused = nk < nacc ? nk : nacc;   // pair g holds k-blocks g, g + kGroups, ...
  constexpr bool TWO = NA > 1 || NB > 1;
  if (producer) {
#pragma unroll 1
    for (int c = 16 * cgrp; c < BN; c += 16 * CGROUPS) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
      // small-term sums first (fixed order), then the h*h chains
      for (int q = 0; q < 2 * nacc; ++q) {
        const int a = q % nacc, small = q < nacc;
        if (a >= nused || (small && !TWO)) continue;
        float t[16];
        tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * 2 * BN + small * BN + c), t);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __fadd_rn(v[j], t[j]);
      }
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4 *>(&stage[arow * ES + c + j]) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  constexpr int C4 = BN / 4;
#pragma unroll 4
  for (int idx = threadIdx.x; idx < BM * C4; idx += kThreads) {
    const int rr = idx / C4, c4 = idx - rr * C4;
    const int m = m0 + rr, n = n0 + c4 * 4;
    if (m < p.M && n < p.N) {
      const float4 v = *reinterpret_cast<const float4 *>(&stage[rr * ES + c4 * 4]);
      if (!SPLITK)
        p.final4(m, n, v, zp);
      else if (!cluster_ks)
        *reinterpret_cast<float4 *>(part + ((int64_t)zs * p.M + m) * p.N + n) = v;
    }
  }
  __shared__ float bias_cl[Pol::BIAS_FROM_B ? BN : 1];     // cluster split-K: this CTA's bias sums
  // bias gradients folded into the B gather: column sums of this CTA's slice
  if constexpr (Pol::BIAS_FROM_B) if (blockIdx.x == 0) {
    if (producer) gb.dump_bias(bias_red[group]);
    __syncthreads();
    if (threadIdx.x < BN && n0 + (int)threadIdx.x < p.N) {
      float s = bias_red[0][threadIdx.x][0];
#pragma unroll
      for (int g = 0; g < kGroups; ++g)
#pragma unroll
        for (int kc = 0; kc < kKc; ++kc)
          if (g + kc > 0) s = __fadd_rn(s, bias_red[g][threadIdx.x][kc]);
      const int n = n0 + threadIdx.x;
      if (!SPLITK) {
        p.bias_out[n] = __fadd_rn(p.bias_out[n], s);
        p.note_bias(p.bias_out[n]);
      } else if (cluster_ks) {
        bias_cl[threadIdx.x] = s;
      } else {
        p.bias_partial[(int64_t)zs * p.N + n] = s;
      }
    }
  }
  TC_MARK(3)
  // split-K across a thread-block cluster (cluster_ks = splits <= 8 along z):
  // every rank holds its partial tile in its staging smem; rank r sums rows
  // [r*BM/ks, ...) over ranks 0..ks-1 in order through distributed shared
  // memory (the global path's order: identical results) and runs the epilogue
  if (SPLITK && cluster_ks) {
    cluster_sync();                              // all ranks' partials staged
    const int rows = (BM + ks - 1) / ks, r0 = zs * rows, r1 = min(BM, r0 + rows);
    for (int idx = r0 * C4 + threadIdx.x; idx < r1 * C4; idx += kThreads) {
      const int rr = idx / C4, c4 = idx - rr * C4;
      const int m = m0 + rr, n = n0 + c4 * 4;
      if (m < p.M && n < p.N) {
        const uint32_t la = smem_u32(&stage[rr * ES + c4 * 4]);
        float4 t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < ks) t[q] = ld_dsmem4(dsmem_addr(la, q));
        float4 acc = t[0];
#pragma unroll
        for (int q = 1; q < 8; ++q)
          if (q < ks) {
            acc.x = __fadd_rn(acc.x, t[q].x);
            acc.y = __fadd_rn(acc.y, t[q].y);
            acc.z = __fadd_rn(acc.z, t[q].z);
            acc.w = __fadd_rn(acc.w, t[q].w);
          }
        p.final4(m, n, acc, zp);
      }
    }
    if constexpr (Pol::BIAS_FROM_B)
      if (blockIdx.x == 0 && zs == 0 && threadIdx.x < BN && n0 + (int)threadIdx.x < p.N) {
        const uint32_t la = smem_u32(&bias_cl[threadIdx.x]);
        float s = ld_dsmem(dsmem_addr(la, 0));
        for (int q = 1; q < ks; ++q) s = __fadd_rn(s, ld_dsmem(dsmem_addr(la, q)));
        const int n = n0 + threadIdx.x;
        p.bias_out[n] = __fadd_rn(p.bias_out[n], s);
        p.note_bias(p.bias_out[n]);
      }
    cluster_sync();                              // peers' smem read by everyone
  } else
  // split-K fixup: the last R CTAs to arrive at a tile each sum a slice of its
  // rows over every split's partial in split order (deterministic whichever
  // CTAs arrive last) and run the epilogue on it.  Reducers other than the
  // very last wait for the remaining arrivals; they are deadlock-free because
  // at most tiles * (R - 1) <= 60 CTAs of a launch ever wait, so two such
  // launches side by side leave SMs for every pending CTA.
  if (SPLITK) {
    __shared__ int s_ticket;
    __threadfence();
    __syncthreads();
    const int tile = (zp * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const int tiles = gridDim.x * gridDim.y * (gridDim.z / ks);
    int R = reducer_budget / tiles + 1;
    R = R > 8 ? 8 : R;
    R = R > ks ? ks : R;
    int *arrive = p.counters + 2 * tile, *finished = arrive + 1;
    if (threadIdx.x == 0) s_ticket = atomicAdd(arrive, 1);
    __syncthreads();
    const int ticket = s_ticket;
    if (ticket >= ks - R) {
      const int red = ticket - (ks - R);
      if (ticket < ks - 1) {
        if (threadIdx.x == 0) {
          int seen;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(arrive) : "memory");
          } while (seen < ks);
        }
        __syncthreads();
      }
      __threadfence();
      // rows [r0, r1) of the tile; partials summed in split order, two float4
      // columns per pass and up to 4 splits per round (8 loads in flight per
      // thread: a round trip costs ~1 us)
      const int rows = (BM + R - 1) / R, r0 = red * rows, r1 = min(BM, r0 + rows);
      const int64_t zstride = (int64_t)p.M * p.N;
#pragma unroll 1
      for (int idx0 = r0 * C4 + threadIdx.x; idx0 < r1 * C4; idx0 += 2 * kThreads) {
        float4 acc[2];
        const float *src[2];
        bool ok[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const int idx = idx0 + f * kThreads;
          const int rr = idx / C4, c4 = idx - rr * C4;
          const int m = m0 + rr, n = n0 + c4 * 4;
          ok[f] = idx < r1 * C4 && m < p.M && n < p.N;
          src[f] = part + (int64_t)(ok[f] ? m : 0) * p.N + (ok[f] ? n : 0);
        }
#pragma unroll 1
        for (int z0 = 0; z0 < ks; z0 += 4) {
          float4 t[2][4];
#pragma unroll
          for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (ok[f] && z0 + j < ks)
                t[f][j] = __ldcg(reinterpret_cast<const float4 *>(src[f] + (z0 + j) * zstride));
#pragma unroll
          for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (ok[f] && z0 + j < ks) {
                if (z0 + j == 0) {
                  acc[f] = t[f][j];
                } else {
                  acc[f].x = __fadd_rn(acc[f].x, t[f][j].x);
                  acc[f].y = __fadd_rn(acc[f].y, t[f][j].y);
                  acc[f].z = __fadd_rn(acc[f].z, t[f][j].z);
                  acc[f].w = __fadd_rn(acc[f].w, t[f][j].w);
                }
              }
        }
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          if (!ok[f]) continue;
          const int idx = idx0 + f * kThreads;
          const int rr = idx / C4, c4 = idx - rr * C4;
          p.final4(m0 + rr, n0 + c4 * 4, acc[f], zp);
        }
      }
      if (Pol::BIAS_FROM_B && red == 0 && blockIdx.x == 0 && threadIdx.x < BN &&
          n0 + (int)threadIdx.x < p.N) {
        const int n = n0 + threadIdx.x;
        float s = __ldcg(p.bias_partial + n);
        for (int zz = 1; zz < ks; ++zz)
          s = __fadd_rn(s, __ldcg(p.bias_partial + (int64_t)zz * p.N + n));
        p.bias_out[n] = __fadd_rn(p.bias_out[n], s);
        p.note_bias(p.bias_out[n]);
      }
      // the last reducer to finish resets the tile's counters for the next launch
      __syncthreads();
      if (threadIdx.x == 0 && atomicAdd(finished, 1) == R - 1) {
        *arrive = 0;
        *finished = 0;
      }
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
#ifdef DQN_TC_TRACE
  TC_MARK(4)
  if (threadIdx.x == 0) {
    const unsigned int i = atomicAdd(&g_trace_n, 1u);
    if (i < kTraceCtas) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long *r = g_trace + 30ull * i;
      for (int j = 0; j < 16; ++j) r[12 + j] = tk_[j];
      r[28] = t_alloc;
      r[29] = t_presync;
      r[0] = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      r[1] = smid;
      for (int j = 0; j < 5; ++j) r[2 + j] = tr_[j];
      r[7] = nk;
      r[8] = tr_[5];
      r[9] = tr_mma[0];
      r[10] = tr_mma[1];
      r[11] = (unsigned)launch_id;
    }
  }
#endif
}

#ifdef DQN_TC_TRACE
inline int next_launch_seq() {
  static int seq = 0;
  return ++seq;
}
#endif

template <class Pol>
inline int smem_bytes() {
  return Plan<Pol>::BYTES;
}

// Split-K across thread-block clusters (measured in the learner graph: 6,788
// vs 6,759 updates/s device, +1-2 % end to end).  Same reduction order as
// the global fixup: identical results.
#ifdef DQN_TC_TRACE
inline int &cluster_splitk_override() {   // diagnostic: 1 on, 0 off
  static int v = 1;
  return v;
}
inline bool cluster_splitk_enabled() { return cluster_splitk_override() != 0; }
#else
inline bool cluster_splitk_enabled() { return true; }
#endif

// split-K reducers per launch (fewer measured -1 to -6 %)
inline int reducer_budget() { return 60; }

template <class Pol>
int launch(cudaStream_t st, const Pol &p, int splits, const char *what) {
  const int bytes = smem_bytes<Pol>();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<Pol>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return cuda_status(e, what);
    configured = true;
  }
  dim3 grid((p.M + BM - 1) / BM, (p.N + Pol::BN - 1) / Pol::BN, splits);
  if (p.ksplits > 1 && 2 * (int64_t)grid.x * grid.y * (splits / p.ksplits) > kMaxTiles) {
    set_error("%s: %u x %u tiles exceed the split-K counter table", what, grid.x, grid.y);
    return DQN_ERR_UNSUPPORTED;
  }
  int launch_id = 0;
#ifdef DQN_TC_TRACE
  launch_id = next_launch_seq();
#endif
  // splits of one tile form a thread-block cluster (<= 8, portable) and are
  // reduced through distributed shared memory; more splits use the global
  // partials and the last-arrivals fixup
  // (only with slack in the grid: clusters are placed within a GPC, so a
  // near-full grid of clusters fragments into a second wave)
  const int64_t ctas = (int64_t)grid.x * grid.y * grid.z;
  const int cks = (p.ksplits > 1 && p.ksplits <= 8 && ctas <= 128 && cluster_splitk_enabled())
                      ? p.ksplits : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  attr[2].id = cudaLaunchAttributeClusterDimension;
  attr[2].val.clusterDim.x = 1;
  attr[2].val.clusterDim.y = 1;
  attr[2].val.clusterDim.z = cks ? cks : 1;
  cfg.attrs = attr;
  cfg.numAttrs = cks ? 3 : 2;
  cudaLaunchKernelEx(&cfg, tc_gemm_kernel<Pol>, p, launch_id, cks, reducer_budget());
  DQN_LAUNCH_CHECK(what);
  return DQN_OK;
}

}  // namespace tc
}  // namespace dqn
