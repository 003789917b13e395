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
constexpr int kThreads = 256;          // 8 warps: all gather; warps w, w+4 share TMEM lanes

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

// pipeline depth that fits ~200 KB of operand stages
constexpr int auto_stages(int bn, bool split_a, bool split_b) {
  const int bytes = (split_a ? kPieces : 1) * BM * BK * 4 + (split_b ? kPieces : 1) * bn * BK * 4;
  const int s = (200 * 1024) / bytes;
  return s > 4 ? 4 : (s < 1 ? 1 : s);
}

// Policy interface (all __device__, const):
//   static constexpr int BN, STAGES; static constexpr bool SPLIT_A, SPLIT_B;
//   int M, N;  int kbeg(z), kend(z);
//   long long a_row(m) / b_row(n)          -- per-row base (-1: row out of range)
//   float4 a(base, k, kend) / b(base, k, kend) -- values at k..k+3 (0 beyond kend)
//   void store4(m, n, float4 v, z)         -- epilogue for columns n..n+3 of row m
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
  constexpr int CA = BM * BK / 4 / kThreads;                      // A chunks per thread (8)
  constexpr int CB = (BN * BK / 4 + kThreads - 1) / kThreads;     // B chunks per thread
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[STAGES];
  __shared__ uint32_t tmem_slot;

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
  const int kbeg = p.kbeg(z), kend = p.kend(z);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const uint32_t sbase = smem_u32(smem);

  // per-thread row bases (same rows in every k-block)
  long long abase[CA], bbase[CB];
#pragma unroll
  for (int i = 0; i < CA; ++i) {
    int row, k;
    chunk_coords(threadIdx.x + i * kThreads, row, k);
    abase[i] = p.a_row(m0 + row);
  }
#pragma unroll
  for (int i = 0; i < CB; ++i) {
    const int c = threadIdx.x + i * kThreads;
    int row, k;
    chunk_coords(c, row, k);
    bbase[i] = (c < BN * BK / 4) ? p.b_row(n0 + row) : -1;
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  // register-staged prefetch: tile kb+1 is in flight while tile kb is
  // committed to smem and multiplied
  float4 ra[CA], rb[CB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int i = 0; i < CA; ++i) {
      int row, k;
      chunk_coords(threadIdx.x + i * kThreads, row, k);
      ra[i] = abase[i] >= 0 ? p.a(abase[i], k0 + k, kend) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      int row, k;
      chunk_coords(threadIdx.x + i * kThreads, row, k);
      rb[i] = bbase[i] >= 0 ? p.b(bbase[i], k0 + k, kend) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (nk > 0) fetch(kbeg);

  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % STAGES;
    if (kb >= STAGES) mbar_wait(&bars[s], ((kb / STAGES) - 1) & 1);
    const uint32_t st = sbase + s * STAGE_BYTES;
    const uint32_t a_t = st, b_t = st + NA * A_BYTES;     // piece p at +p*A_BYTES / +p*B_BYTES
#pragma unroll
    for (int i = 0; i < CA; ++i) {
      int row, k;
      chunk_coords(threadIdx.x + i * kThreads, row, k);
      store_split(a_t + chunk_off(BM, row, k), A_BYTES, ra[i], NA);
    }
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const int c = threadIdx.x + i * kThreads;
      if (c < BN * BK / 4) {
        int row, k;
        chunk_coords(c, row, k);
        store_split(b_t + chunk_off(BN, row, k), B_BYTES, rb[i], NB);
      }
    }
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
  // warps w and w+4 read the same TMEM lane quarter (w % 4) and split the
  // 16-column chunks between them
  const int quarter = warp & 3, half = warp >> 2;
  const int r = quarter * 32 + lane;
  const int nused = nk < nacc ? nk : nacc;
#pragma unroll 1
  for (int c = 16 * half; c < BN; c += 32) {
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
    if (m < p.M && n < p.N)
      p.store4(m, n, *reinterpret_cast<const float4 *>(&stage[rr * ES + c4 * 4]), z);
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
  static const int env_nacc = [] {
    const char *e = getenv("DQN_TC_NACC");
    return e ? atoi(e) : 4;
  }();
  int nacc = env_nacc < 1 ? 1 : env_nacc;
  const int pair = (Pol::SPLIT_A || Pol::SPLIT_B) ? 2 : 1;
  while (nacc > 1 && Pol::BN * nacc * pair > 512) --nacc;
  tc_gemm_kernel<Pol><<<grid, kThreads, bytes, st>>>(p, nacc);
  DQN_LAUNCH_CHECK(what);
  return DQN_OK;
}

}  // namespace tc
}  // namespace dqn
