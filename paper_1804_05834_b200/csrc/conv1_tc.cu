// The trunk's first convolution (8x8 stride 4 over the uint8 frame stack:
// layers.py:226-255 forward, envs.py:300-311 pixel rule) on tcgen05 with the
// operands staged in shared memory by bulk copies.
//
//   y[pixel][n] = relu( (sum_k u[pixel][k] W[k][n]) / 255 + b[n] )
//
// The frame bytes enter the GEMM as the integers they are (exact in tf32, so
// A needs no lo piece) and the 1/255 is applied to the sum, as the generic
// engine's uint8 forward does (tc_gemm.cuh FwdPol); W is split hi/lo
// (3xTF32 without the A_lo term):  u * [W_hi ; W_lo]  (N = 2 x 32) in one MMA.
//
// One CTA computes GR whole output rows of one image (Atari: 5 rows = 100
// pixels, 4 CTAs per image).  The input rows those output rows read are
// contiguous in the frame (24 rows x 336 B = 8 KB), so one bulk copy brings
// the slab; a second brings W (256 x 32 fp32).  A k-block of 32 is one filter
// row r: for output pixel (oy, ox) its 32 values are the 8 pixels x 4
// channels at slab row 4 oy + r, bytes 16 ox .. 16 ox + 31.  Each converter
// thread owns one pixel row and writes those 32 exact integers to its TMEM
// lane (the A operand of a TS-form MMA: no A tile in shared memory, so six
// stages fit twice per SM), and the converters transpose W's rows
// r*32 .. r*32+31 into the K-major B tile in shared memory.
#include "tc_gemm.cuh"

#include <algorithm>

namespace dqn {
namespace {

constexpr int C1_THREADS = 192;                // warps 0-3 convert + epilogue, 4 loads, 5 MMA
constexpr int C1_BK = 32;
constexpr int C1_N = 32;                       // output channels
constexpr int C1_ST = 6;                       // operand stages (B in smem, A in TMEM)
constexpr int C1_ACOL = 64;                    // TMEM: accumulator [hi | lo] 0..63, A stages after
constexpr int C1_B_BYTES = 2 * C1_N * 128;     // [W_hi ; W_lo], K-major

#ifdef DQN_TC_TRACE
// per-CTA %globaltimer marks (trace build): entry, after pdl_wait, operands
// loaded, MMAs done, stored
__device__ unsigned long long g_c1_trace[1024 * 5];
#define C1_MARK(i)                                                          \
  {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                            \
      unsigned long long t_;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
      g_c1_trace[blockIdx.x * 5 + (i)] = t_;                                \
    }                                                                       \
  }
#else
#define C1_MARK(i)
#endif

struct Conv1Args {
  const uint8_t *x;                            // [B][H][W][C]
  const float *w;                              // [K][32] (K = fh * fw * C, (r, s, c) order)
  const float *bias;
  float *y;                                    // [B][OH][OW][32]
  int H, W, C, OH, OW, fh, S;
  int GR;                                      // output rows per CTA
  int tiles_per_img;
  int slab_rows;                               // S (GR - 1) + fh
  int a_bytes;                                 // A tile: GR * OW rows rounded up to 8, x 128 B
  int relu;
};

__device__ __forceinline__ uint64_t c1_desc(uint32_t addr) {   // K-major, 128-B swizzle
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void c1_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void c1_bulk(uint32_t dst, const void *src, uint32_t bytes,
                                        uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

// 4 bytes -> 4 exact floats (0x4B000000 | b is 2^23 + b)
__device__ __forceinline__ float4 c1_bytes(uint32_t v) {
  const float m = 8388608.f;
  return make_float4(__int_as_float(0x4B000000 | (v & 0xFF)) - m,
                     __int_as_float(0x4B000000 | ((v >> 8) & 0xFF)) - m,
                     __int_as_float(0x4B000000 | ((v >> 16) & 0xFF)) - m,
                     __int_as_float(0x4B000000 | (v >> 24)) - m);
}

__global__ void __launch_bounds__(C1_THREADS, 2) conv1_tc_kernel(const __grid_constant__ Conv1Args p) {
  constexpr uint32_t IDESC = tc::make_idesc_tf32(2 * C1_N);
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t loaded, conv[C1_ST], empty[C1_ST], done;
  __shared__ uint32_t tmem_slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t sbase = (tc::smem_u32(smem) + 1023u) & ~1023u;
  // layout: B stages | W (K x 32 fp32) | slab; the A tiles live in TMEM
  // (columns C1_ACOL + 32 s), the epilogue stages through the B stages
  const uint32_t a_st = sbase, b_st = sbase;
  const uint32_t w_s = b_st + C1_ST * C1_B_BYTES;
  const int K = p.fh * p.fh * p.C;
  const uint32_t slab = w_s + (uint32_t)K * C1_N * 4;
  const int img = blockIdx.x / p.tiles_per_img, g = blockIdx.x - img * p.tiles_per_img;
  const int oy0 = g * p.GR;
  const int rows = p.GR * p.OW;                 // valid A rows
  const int row_bytes = p.W * p.C;
  const uint32_t slab_bytes = (uint32_t)(p.slab_rows * row_bytes);
  const int nkb = p.fh;                         // one filter row per k-block
  C1_MARK(0)

  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 32 * 5) {
    tc::mbar_init(&loaded, 1);
    for (int s = 0; s < C1_ST; ++s) {
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
  pdl_wait();                                 // the frames come from the sample / gather
  const uint32_t tmem = tmem_slot;
  C1_MARK(1)

  if (warp == 4) {
    if (lane == 0) {
      const int y0 = p.S * oy0;
      const uint8_t *src = p.x + ((int64_t)img * p.H + y0) * row_bytes;
      // the last tile's slab may end past the image (never read): clip it
      const uint32_t avail = (uint32_t)((p.H - y0) * row_bytes);
      const uint32_t sb = std::min(slab_bytes, avail);
      tc::mbar_expect_tx(&loaded, sb + (uint32_t)K * C1_N * 4);
      c1_bulk(slab, src, sb, &loaded);
      c1_bulk(w_s, p.w, (uint32_t)K * C1_N * 4, &loaded);
    }
  } else if (warp == 5) {
    if (lane == 0) {                          // MMA issuer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % C1_ST, use = kb / C1_ST;
        tc::mbar_wait(&conv[s], use & 1);
        tc::tc_fence_after();
        const uint32_t b = b_st + s * C1_B_BYTES;
#pragma unroll
        for (int kq = 0; kq < C1_BK / 8; ++kq)
          tc::mma_ts(tmem, tmem + (uint32_t)(C1_ACOL + s * C1_BK + 8 * kq), c1_desc(b + 32 * kq),
                     IDESC, (kb == 0 && kq == 0) ? 0u : 1u);
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&done);
    }
  } else {                                    // warps 0-3: operand tiles
    // thread t owns pixel row q = t of the tile (its TMEM lane): the slab
    // offset of its 8 filter-column pixels at filter row 0
    const uint8_t *sl = smem + (slab - tc::smem_u32(smem));
    const float *ws = reinterpret_cast<const float *>(smem + (w_s - tc::smem_u32(smem)));
    const int q = t, oy = q / p.OW, ox = q - oy * p.OW;
    const int in0 = q < rows ? p.S * oy * row_bytes + p.S * ox * 4 : -1;
    const uint32_t ta0 = tmem + ((uint32_t)(warp * 32) << 16) + C1_ACOL;
    tc::mbar_wait(&loaded, 0);
    C1_MARK(2)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % C1_ST, use = kb / C1_ST;
      if (use > 0) tc::mbar_wait(&empty[s], (use - 1) & 1);
      const uint32_t b = b_st + s * C1_B_BYTES;
      // A row q, filter row kb: the 8 pixels x 4 channel bytes at slab row
      // S oy + kb, exact integers -> TMEM columns C1_ACOL + 32 s ..
      float av[C1_BK];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t v = in0 >= 0 ? *reinterpret_cast<const uint32_t *>(sl + in0 + kb * row_bytes + 4 * c) : 0u;
        const float4 f = c1_bytes(v);
        av[4 * c] = f.x;
        av[4 * c + 1] = f.y;
        av[4 * c + 2] = f.z;
        av[4 * c + 3] = f.w;
      }
      tc::tmem_st16(ta0 + (uint32_t)(s * C1_BK), av);
      tc::tmem_st16(ta0 + (uint32_t)(s * C1_BK + 16), av + 16);
      // B: W rows kb*32 .. kb*32+31 transposed: row n (hi), row 32 + n (lo)
      float w[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = t + 128 * h, n = u & (C1_N - 1), c = u / C1_N;
#pragma unroll
        for (int i = 0; i < 4; ++i) w[h][i] = ws[(kb * C1_BK + 4 * c + i) * C1_N + n];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = t + 128 * h, n = u & (C1_N - 1), c = u / C1_N;
        const uint32_t off = (uint32_t)(n * 128 + ((c ^ (n & 7)) << 4));
        tc::st_shared_v4(b + off, make_float4(w[h][0], w[h][1], w[h][2], w[h][3]));
        tc::st_shared_v4(b + (uint32_t)(C1_N * 128) + off,
                         make_float4(tc::tf32_lo(w[h][0]), tc::tf32_lo(w[h][1]),
                                     tc::tf32_lo(w[h][2]), tc::tf32_lo(w[h][3])));
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async();
      tc::tc_fence_before();                    // TMEM stores -> the MMA thread
      tc::mbar_arrive(&conv[s]);
    }
  }

  // ---- epilogue: row q of the accumulator = pixel q of this tile, staged
  // through shared memory (the A stages) for contiguous stores of the tile's
  // rows x 32 outputs
  __syncthreads();
  tc::mbar_wait(&done, 0);
  tc::tc_fence_after();
  C1_MARK(3)
  constexpr int LD = C1_N + 4;                  // staged row stride (floats)
  float *stage = reinterpret_cast<float *>(smem + (a_st - tc::smem_u32(smem)));
  if (warp < 4) {
    const int q = warp * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    float hi[16], lo[16];
#pragma unroll 1
    for (int c = 0; c < C1_N; c += 16) {
      tc::tmem_ld16(lb + (uint32_t)c, hi);
      tc::tmem_ld16(lb + (uint32_t)(C1_N + c), lo);
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4 *>(&stage[q * LD + c + j]) =
            make_float4(__fadd_rn(hi[j], lo[j]), __fadd_rn(hi[j + 1], lo[j + 1]),
                        __fadd_rn(hi[j + 2], lo[j + 2]), __fadd_rn(hi[j + 3], lo[j + 3]));
    }
  }
  __syncthreads();
  {
    float4 *out = reinterpret_cast<float4 *>(
        p.y + ((int64_t)img * p.OH * p.OW + (int64_t)oy0 * p.OW) * C1_N);
    for (int u = t; u < rows * (C1_N / 4); u += C1_THREADS) {
      const int q = u / (C1_N / 4), c4 = (u - q * (C1_N / 4)) * 4;
      const float4 s4 = *reinterpret_cast<const float4 *>(&stage[q * LD + c4]);
      const float4 b4 = __ldg(reinterpret_cast<const float4 *>(p.bias + c4));
      float v[4] = {__fadd_rn(__fdiv_rn(s4.x, 255.0f), b4.x), __fadd_rn(__fdiv_rn(s4.y, 255.0f), b4.y),
                    __fadd_rn(__fdiv_rn(s4.z, 255.0f), b4.z), __fadd_rn(__fdiv_rn(s4.w, 255.0f), b4.w)};
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = v[i] < 0.f ? 0.f : v[i];
      }
      out[u] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  C1_MARK(4)
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256)
                 : "memory");
}

}  // namespace

// uint8 first convolution with one filter row per 32-deep k-block (fw * C ==
// 32), 32 output channels, square filter and stride, whole output rows per
// CTA within 128 pixels, 16-byte aligned rows
bool conv1_tc_ok(const dqn_layer_desc &L) {
  if (L.kind != DQN_LAYER_CONV || L.out_c != C1_N || L.fh != L.fw || L.sh != L.sw ||
      L.fw * L.in_c != C1_BK || L.out_w > 128 || (L.in_w * L.in_c) % 16 || L.in_c != 4)
    return false;
  return true;
}

int conv1_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const uint8_t *x,
                     const float *params, float *y, int batch) {
  if (!conv1_tc_ok(L) || batch < 1 || ((uintptr_t)x % 16) || ((uintptr_t)(params + L.w_off) % 16))
    return DQN_ERR_UNSUPPORTED;
  Conv1Args a{};
  a.x = x;
  a.w = params + L.w_off;
  a.bias = params + L.b_off;
  a.y = y;
  a.H = L.in_h;
  a.W = L.in_w;
  a.C = L.in_c;
  a.OH = L.out_h;
  a.OW = L.out_w;
  a.fh = L.fh;
  a.S = L.sh;
  a.relu = L.relu;
  // the largest divisor of OH whose rows fit 128 pixels
  int gr = 1;
  for (int d = 1; d <= L.out_h; ++d)
    if (L.out_h % d == 0 && d * L.out_w <= 128) gr = d;
  a.GR = gr;
  a.tiles_per_img = L.out_h / gr;
  a.slab_rows = L.sh * (gr - 1) + L.fh;
  const int K = L.fh * L.fw * L.in_c;
  a.a_bytes = 0;
  if (gr * L.out_w > 128) return DQN_ERR_UNSUPPORTED;      // one TMEM lane per pixel
  const int smem = 1024 + C1_ST * C1_B_BYTES + K * C1_N * 4 +
                   ((a.slab_rows * L.in_w * L.in_c + 15) / 16) * 16;
  if (C1_ST * C1_B_BYTES < gr * L.out_w * (C1_N + 4) * 4) return DQN_ERR_UNSUPPORTED;  // epilogue stage
  if (smem > 227 * 1024) return DQN_ERR_UNSUPPORTED;
  static int configured = 0;
  if (smem > configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(conv1_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "conv1_tc_forward");
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * a.tiles_per_img);
  cfg.blockDim = dim3(C1_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1] = priority_attr(st);
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, conv1_tc_kernel, a);
  DQN_LAUNCH_CHECK("conv1_tc_forward");
  return DQN_OK;
}

}  // namespace dqn

#ifdef DQN_TC_TRACE
extern "C" int dqn_c1_trace(unsigned long long *host) {
  return (int)cudaMemcpyFromSymbol(host, dqn::g_c1_trace, sizeof(dqn::g_c1_trace));
}
#endif
