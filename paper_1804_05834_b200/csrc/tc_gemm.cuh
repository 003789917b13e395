// tcgen05 (5th-gen tensor core) implicit-GEMM engine for sm_100a.
//
// One CTA = 8 warps computes a 128 x BN tile of C = A * B^T (A: M x K,
// B: N x K in "math" orientation) with the accumulator in TMEM:
//   * all 256 threads gather operand chunks (16 B = 4 fp32) from global
//     memory through a Policy (im2col addressing, transposed weights, ...),
//     one k-block ahead in registers, split each value exactly into tf32
//     pieces (x = hi + lo; kPieces = 3 gives h + m + l) and store them into
//     shared memory in the canonical no-swizzle K-major UMMA layout (core
//     matrices of 8 rows x 16 B);
//   * thread 0 issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) for the
//     significant piece products (hi*hi, hi*lo, lo*hi: "3xTF32") and
//     tcgen05.commit's an mbarrier per pipeline stage, so the gather of stage
//     s+1 overlaps the MMAs of stage s;
//   * accuracy: SURVEY.md App. A -- one bf16/tf32 pass misses the 1e-3
//     one-step parity bar.  Measured here, the residual error of 3xTF32 is
//     dominated by the tensor pipe's accumulation rounding, not by the
//     dropped lo*lo term, so hi*hi and the small products go to separate
//     TMEM accumulators and the K loop round-robins k-blocks over `nacc`
//     accumulator pairs; the epilogue sums them in fp32 (~3e-7 rel. vs fp32
//     SIMT per GEMM);
//   * the epilogue reads TMEM with tcgen05.ld (warps w and w+4 own lanes
//     32(w%4)..+31 = tile rows and split the columns), stages the tile
//     row-major in shared memory and hands coalesced float4s to the Policy
//     (bias / ReLU / mask / split-K partial / gradient accumulate).
// Operands that are exact in tf32 (uint8 pixels) use one piece.
#pragma once

#include "common.cuh"

#include <stdlib.h>

namespace dqn {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;               // fp32 elements per stage (4 MMA k-steps of 8)
constexpr int kThreads = 512;          // 16 warps: all gather; warps w, w+4, ... share TMEM lanes

#ifndef DQN_TC_PIECES
#define DQN_TC_PIECES 2
#endif
constexpr int kPieces = DQN_TC_PIECES;  // tf32 pieces per fp32 operand (2: hi/lo, 3: h/m/l)

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

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

// Instruction descriptor: kind::tf32, fp32 accumulate, M = 128.
__host__ __device__ constexpr uint32_t make_idesc_tf32(int n, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | ((a_mn ? 1u : 0u) << 15)     // a_major
         | ((b_mn ? 1u : 0u) << 16)     // b_major
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(BM >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
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

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w));
}

// x = h + m + l exactly, each exactly representable in tf32 (h: top 11
// significant bits, m: next 11, l: the last 2), so products of the pieces are
// exact in fp32 and the dropped m*l / l*m / l*l terms are below 2^-33 |x y|.
__device__ __forceinline__ void store_split(uint32_t base, uint32_t level_stride, float4 v,
                                            int levels) {
  if (levels == 1) {
    st_shared_v4(base, v);
    return;
  }
  const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  const float4 r = make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z),
                               __fsub_rn(v.w, h.w));
  if (kPieces == 2) {          // hi/lo: lo keeps up to 13 bits, the MMA reads its top 11
    st_shared_v4(base, h);
    st_shared_v4(base + level_stride, r);
    return;
  }
  const float4 m = make_float4(tf32_hi(r.x), tf32_hi(r.y), tf32_hi(r.z), tf32_hi(r.w));
  const float4 l = make_float4(__fsub_rn(r.x, m.x), __fsub_rn(r.y, m.y), __fsub_rn(r.z, m.z),
                               __fsub_rn(r.w, m.w));
  st_shared_v4(base, h);
  st_shared_v4(base + level_stride, m);
  st_shared_v4(base + 2 * level_stride, l);
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

// Operand tiles are gathered cooperatively: chunk c (16 B = row, 4 k) of an
// R x BK tile is owned by thread c % 128, so every thread owns the same rows
// in every k-block (row bases are computed once per CTA).  A quarter-warp
// writes one contiguous 128-byte smem line (8 rows of one k-chunk).
__device__ __forceinline__ void chunk_coords(int c, int &row, int &k) {
  const int r8 = c & 7, kc = (c >> 3) & 7, rg = c >> 6;
  row = rg * 8 + r8;
  k = kc * 4;
}

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int EPI_STRIDE = BN + 4;                // floats per staged row
  static constexpr int EPI_BYTES = BM * EPI_STRIDE * 4;
};

constexpr int tmem_cols(int bn) { return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256; }

// pipeline depth: the register-staged prefetch already overlaps the next
// gather with the MMAs, so two stages suffice; keeping a CTA under ~110 KB
// of shared memory lets two CTAs share an SM (16 warps hiding gather latency)
constexpr int auto_stages(int bn, bool split_a, bool split_b) {
  const int bytes = (split_a ? kPieces : 1) * BM * BK * 4 + (split_b ? kPieces : 1) * bn * BK * 4;
  const int s = (110 * 1024) / bytes;
  return s > 2 ? 2 : (s < 1 ? 1 : s);
}

__device__ __forceinline__ float comp(const float4 &v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// Gathers one R x BK operand tile per k-block into registers and stores it
// K-major.  Units are owned by thread u % 256 with the same rows in every
// k-block, so row bases are computed once.
//  * MNC == false (source contiguous along k): unit = chunk (row, 4 k), one
//    16-byte load via ld(base, koff(k)); all units of a thread share k, so
//    the k-dependent address part is computed once per k-block;
//  * MNC == true (source contiguous along rows, e.g. W[k][n] or dY[pix][co]):
//    unit = 4 rows x 4 k, four 16-byte loads along the rows via
//    f4(base, k, kend, v[4]) (consecutive lanes = consecutive row quads =
//    coalesced), transposed in registers into four K-major chunks.
// Optionally accumulates the per-row sums of everything stored (bias grads).
template <bool MNC, int R>
struct Gather {
  static constexpr int UNITS = MNC ? R * BK / 16 : R * BK / 4;
  static constexpr int U = (UNITS + kThreads - 1) / kThreads;
  static constexpr int V = MNC ? 4 : 1;
  static_assert(!MNC || U == 1, "MNC gathers assume one unit per thread");
  long long base[U];
  int t0;                      // this thread's first unit (rotated, see init)
  uint32_t soff[U];            // byte offset of the unit's (first) chunk in a piece tile
  int kk;                      // the thread's k offset inside a k-block (same for all units)
  float4 v[U][V];
  float bsum[U][V];

  __device__ static void coords(int u, int &row, int &k) {
    if (!MNC) {
      chunk_coords(u, row, k);
    } else {
      const int q = u % (R / 4), kc = u / (R / 4);
      row = 4 * q;
      k = 4 * kc;
    }
  }
  // rot: threads [rot, rot + UNITS) take the first units, so the A and B
  // gathers of a CTA can be laid on disjoint threads when both are short
  template <class RowFn>
  __device__ void init(RowFn rowfn, int rot) {
    t0 = (threadIdx.x + kThreads - rot) % kThreads;
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int u = t0 + i * kThreads;
      int row, k;
      coords(u, row, k);
      base[i] = u < UNITS ? rowfn(row) : -1;
      soff[i] = chunk_off(R, row, k);
      kk = k;
#pragma unroll
      for (int j = 0; j < V; ++j) bsum[i][j] = 0.f;
    }
  }
  // K-major: koff(k) once per k-block, ld(base, koff) per unit (k < kend
  // checked once: every unit of a thread shares k).  MNC: f4 per unit.
  template <class KF, class LD, class F4>
  __device__ void fetch(int k0, int kend, KF &&koff, LD &&ld, F4 &&f4) {
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
  __device__ void store(uint32_t tile, uint32_t piece_stride, int pieces, bool bias) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (t0 + i * kThreads >= UNITS) continue;
      if constexpr (!MNC) {
        store_split(tile + soff[i], piece_stride, v[i][0], pieces);
        if (bias)
          bsum[i][0] = __fadd_rn(bsum[i][0], __fadd_rn(__fadd_rn(v[i][0].x, v[i][0].y),
                                                       __fadd_rn(v[i][0].z, v[i][0].w)));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 c = make_float4(comp(v[i][0], j), comp(v[i][1], j), comp(v[i][2], j),
                                       comp(v[i][3], j));
          store_split(tile + soff[i] + 16 * j, piece_stride, c, pieces);   // rows row..row+3
          if (bias)
            bsum[i][j] =
                __fadd_rn(bsum[i][j], __fadd_rn(__fadd_rn(c.x, c.y), __fadd_rn(c.z, c.w)));
        }
      }
    }
  }
  template <int RR>
  __device__ void dump_bias(float (&red)[RR][8]) const {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int u = t0 + i * kThreads;
      if (u >= UNITS) continue;
      int row, k;
      coords(u, row, k);
#pragma unroll
      for (int j = 0; j < V; ++j)
        if (row + j < RR) red[row + j][k >> 2] = bsum[i][j];
    }
  }
};

// Policies derive from this; it supplies the gather form a policy does not
// use (never called: the Gather of that operand uses the other form).
struct PolBase {
  __device__ int a_koff(int) const { return 0; }
  __device__ int b_koff(int) const { return 0; }
  __device__ float4 a_ld(long long, int) const { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ float4 b_ld(long long, int) const { return make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ void a4(long long, int, int, float4 (&)[4]) const {}
  __device__ void b4(long long, int, int, float4 (&)[4]) const {}
};

// Split-K tiles count arrivals in a per-binding int table (the tail of the
// binding scratch, zero-initialised); the last CTA resets its counter, so the
// table is all-zero between launches (graph-replay safe) and two kernels on
// different streams with different bindings never share counters.
constexpr int kMaxTiles = 4096;

// Policy interface (all __device__, const):
//   static constexpr int BN, STAGES; static constexpr bool SPLIT_A, SPLIT_B, BIAS_FROM_B;
//   int M, N, ksplits;  int kbeg(split), kend(split);
//   float *partial ([problems][ksplits][M][N] when ksplits > 1)
//   gridDim.z = problems * ksplits; a_row/b_row/final4 get the problem index
//   long long a_row(m) / b_row(n)          -- per-row base (-1: row out of range)
//   K-major operand: int a_koff(k) -- k-dependent offset (once per k-block),
//     float4 a_ld(base, koff) -- values at k..k+3 (k < kend checked by the engine)
//   MN-contiguous operand: a4(base, k, kend, v[4]) -- rows base..+3 at k..k+3
//   void final4(m, n, float4 v)            -- epilogue for columns n..n+3 of row m
//   BIAS_FROM_B: float *bias_out (+= column sums of B over k), *bias_partial
// nacc: the K loop of a tile round-robins its k-blocks over nacc TMEM
// accumulators that the epilogue sums in fixed order -- shorter tensor-core
// accumulation chains (each chain rounds in the tensor pipe) for ~fp32-SIMT
// accuracy on long reductions.
template <class Pol>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const Pol p, const int nacc) {
  constexpr int BN = Pol::BN, STAGES = Pol::STAGES;
  constexpr int A_BYTES = Smem<BN>::A_BYTES, B_BYTES = Smem<BN>::B_BYTES;
  constexpr int NA = Pol::SPLIT_A ? kPieces : 1, NB = Pol::SPLIT_B ? kPieces : 1;
  constexpr int STAGE_BYTES = NA * A_BYTES + NB * B_BYTES;
  // accumulator pairs: [a] holds the h*h chain, [nacc + a] the small pieces
  constexpr bool TWO = Pol::SPLIT_A || Pol::SPLIT_B;
  const int TCOLS = tmem_cols(BN * nacc * (TWO ? 2 : 1));
  constexpr uint32_t IDESC = make_idesc_tf32(BN, false, false);   // both K-major
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[STAGES];
  __shared__ uint32_t tmem_slot;
  __shared__ float bias_red[Pol::BIAS_FROM_B ? BN : 1][8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
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

  // operand gathers (rows fixed per thread across k-blocks; see Gather)
  Gather<Pol::A_MNC, BM> ga;
  Gather<Pol::B_MNC, BN> gb;
  ga.init([&](int r) { return p.a_row(m0 + r, zp); }, 0);
  gb.init([&](int r) { return p.b_row(n0 + r, zp); }, Gather<Pol::A_MNC, BM>::UNITS % kThreads);

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  // register-staged prefetch: tile kb+1 is in flight while tile kb is
  // committed to smem and multiplied
  auto fetch = [&](int k0) {
    // generic lambdas: only the form matching the policy's layout is instantiated
    ga.fetch(k0, kend, [&](int k) { return p.a_koff(k); },
             [&](long long b, int ko) { return p.a_ld(b, ko); },
             [&](long long b, int k, int ke, float4 (&v)[4]) { p.a4(b, k, ke, v); });
    gb.fetch(k0, kend, [&](int k) { return p.b_koff(k); },
             [&](long long b, int ko) { return p.b_ld(b, ko); },
             [&](long long b, int k, int ke, float4 (&v)[4]) { p.b4(b, k, ke, v); });
  };
  if (nk > 0) fetch(kbeg);
  const bool want_bias = Pol::BIAS_FROM_B && blockIdx.x == 0;

  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % STAGES;
    if (kb >= STAGES) mbar_wait(&bars[s], ((kb / STAGES) - 1) & 1);
    const uint32_t st = sbase + s * STAGE_BYTES;
    const uint32_t a_t = st, b_t = st + NA * A_BYTES;     // piece p at +p*A_BYTES / +p*B_BYTES
    ga.store(a_t, A_BYTES, NA, false);
    gb.store(b_t, B_BYTES, NB, want_bias);
    if (kb + 1 < nk) fetch(kbeg + (kb + 1) * BK);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t dbig = tmem + (uint32_t)((kb % nacc) * BN);
      const uint32_t dsmall = dbig + (uint32_t)(nacc * BN);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        bool first_big = (kb < nacc && ks == 0), first_small = first_big;
        // piece products with significance 2^0, 2^-11, 2^-22: (ia, ib), ia + ib < kPieces
#pragma unroll
        for (int sum = 0; sum < kPieces; ++sum)
#pragma unroll
          for (int ia = 0; ia <= sum; ++ia) {
            const int ib = sum - ia;
            if (ia >= NA || ib >= NB) continue;
            bool &first = sum == 0 ? first_big : first_small;
            mma_tf32(sum == 0 ? dbig : dsmall, op_desc(a_t + ia * A_BYTES, BM, ks),
                     op_desc(b_t + ib * B_BYTES, BN, ks), IDESC, first ? 0u : 1u);
            first = false;
          }
      }
      mma_commit(&bars[s]);
    }
  }
  if (nk > 0) {
    const int s = (nk - 1) % STAGES;
    mbar_wait(&bars[s], ((nk - 1) / STAGES) & 1);
  }
  tc_fence_after();

  // epilogue: TMEM -> registers -> smem (row-major staging) -> coalesced stores
  float *stage = reinterpret_cast<float *>(smem);
  constexpr int ES = Smem<BN>::EPI_STRIDE;
  // warps w, w+4, ... read the same TMEM lane quarter (w % 4) and split the
  // 16-column chunks between them
  constexpr int GROUPS = kThreads / 128;
  const int quarter = warp & 3, half = warp >> 2;
  const int r = quarter * 32 + lane;
  const int nused = nk < nacc ? nk : nacc;
#pragma unroll 1
  for (int c = 16 * half; c < BN; c += 16 * GROUPS) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.f;
    // small-piece sums first (fixed order), then the h*h chains
    const int na = TWO ? 2 * nacc : nacc;
    for (int q = 0; q < na; ++q) {
      const int a = TWO ? (q < nacc ? nacc + q : q - nacc) : q;   // smalls, then bigs
      if ((a % nacc) >= nused) continue;
      float t[16];
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * BN + c), t);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __fadd_rn(v[j], t[j]);
    }
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4 *>(&stage[r * ES + c + j]) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
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
      else
        *reinterpret_cast<float4 *>(part + ((int64_t)zs * p.M + m) * p.N + n) = v;
    }
  }
  // bias gradients folded into the B gather: column sums of this CTA's slice
  if constexpr (Pol::BIAS_FROM_B) if (blockIdx.x == 0) {
    gb.dump_bias(bias_red);
    __syncthreads();
    if (threadIdx.x < BN && n0 + (int)threadIdx.x < p.N) {
      float s = bias_red[threadIdx.x][0];
#pragma unroll
      for (int kc = 1; kc < 8; ++kc) s = __fadd_rn(s, bias_red[threadIdx.x][kc]);
      const int n = n0 + threadIdx.x;
      if (!SPLITK)
        p.bias_out[n] = __fadd_rn(p.bias_out[n], s);
      else
        p.bias_partial[(int64_t)zs * p.N + n] = s;
    }
  }
  // split-K fixup: the last CTA of a tile sums every split's partial in split
  // order (deterministic, whichever CTA arrives last) and runs the epilogue
  if (SPLITK) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    const int tile = (zp * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) s_last = (atomicAdd(&p.counters[tile], 1) == ks - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      // partials summed in split order; 8 loads in flight per thread
      const int64_t zstride = (int64_t)p.M * p.N;
#pragma unroll 1
      for (int idx = threadIdx.x; idx < BM * C4; idx += kThreads) {
        const int rr = idx / C4, c4 = idx - rr * C4;
        const int m = m0 + rr, n = n0 + c4 * 4;
        if (m < p.M && n < p.N) {
          const float *src = part + (int64_t)m * p.N + n;
          float4 v = __ldcg(reinterpret_cast<const float4 *>(src));
          for (int z0 = 1; z0 < ks; z0 += 8) {
            float4 t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (z0 + j < ks) t[j] = __ldcg(reinterpret_cast<const float4 *>(src + (z0 + j) * zstride));
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (z0 + j < ks) {
                v.x = __fadd_rn(v.x, t[j].x);
                v.y = __fadd_rn(v.y, t[j].y);
                v.z = __fadd_rn(v.z, t[j].z);
                v.w = __fadd_rn(v.w, t[j].w);
              }
          }
          p.final4(m, n, v, zp);
        }
      }
      if (Pol::BIAS_FROM_B && blockIdx.x == 0 && threadIdx.x < BN && n0 + (int)threadIdx.x < p.N) {
        const int n = n0 + threadIdx.x;
        float s = __ldcg(p.bias_partial + n);
        for (int zz = 1; zz < ks; ++zz)
          s = __fadd_rn(s, __ldcg(p.bias_partial + (int64_t)zz * p.N + n));
        p.bias_out[n] = __fadd_rn(p.bias_out[n], s);
      }
      if (threadIdx.x == 0) p.counters[tile] = 0;      // reusable by the next launch
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS)
                 : "memory");
}

template <class Pol>
inline int smem_bytes() {
  constexpr int NA = Pol::SPLIT_A ? kPieces : 1, NB = Pol::SPLIT_B ? kPieces : 1;
  constexpr int pipe = Pol::STAGES * (NA * Smem<Pol::BN>::A_BYTES + NB * Smem<Pol::BN>::B_BYTES);
  constexpr int epi = Smem<Pol::BN>::EPI_BYTES;
  return pipe > epi ? pipe : epi;
}

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
  if (p.ksplits > 1 && (int64_t)grid.x * grid.y * (splits / p.ksplits) > kMaxTiles) {
    set_error("%s: %u x %u tiles exceed the split-K counter table", what, grid.x, grid.y);
    return DQN_ERR_UNSUPPORTED;
  }
  static const int env_nacc = [] {
    const char *e = getenv("DQN_TC_NACC");
    return e ? atoi(e) : 2;      // 2 accumulator pairs: <= 256 TMEM columns at BN <= 64
  }();
  int nacc = env_nacc < 1 ? 1 : env_nacc;
  const int pair = (Pol::SPLIT_A || Pol::SPLIT_B) ? 2 : 1;
  while (nacc > 1 && Pol::BN * nacc * pair > 256) --nacc;   // 2 CTAs/SM can always allocate
  tc_gemm_kernel<Pol><<<grid, kThreads, bytes, st>>>(p, nacc);
  DQN_LAUNCH_CHECK(what);
  return DQN_OK;
}

}  // namespace tc
}  // namespace dqn
