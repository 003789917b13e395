// Conv trunk on the 5th-gen tensor cores: every GEMM-shaped phase of the
// convolution / linear layers runs through the tcgen05 engine (tc_gemm.cuh)
// with implicit-GEMM operand gathers -- no im2col / col2im buffers in HBM and
// no separate reduction launches (split-K partials are reduced in-kernel by
// the last CTA of each tile, bias gradients are folded into the wgrad GEMM).
//
//   forward  (layers.py:226-233, 148-150):  Y[pix, co] = im2col(X)[pix, k] * W[k, co]
//            A gathered from NHWC X (uint8 frames: exact integers, the 1/255
//            of envs.py:300-311 applied in the epilogue), B = W gathered along
//            k; epilogue bias + ReLU.
//   dgrad    (layers.py:235-248, 152-155):  per stride phase (py, px),
//            dX[pix, c] = sum_{ti,tj,co} dY[y/s - ti, x/s - tj, co] * W[py+s*ti, px+s*tj, c, co]
//            -- the gather form of col2im, only the taps that exist (no 4x
//            zero work for the stride-2 layer), masked by the ReLU below.
//            Linear layers: dX = dY * W^T with the mask.
//   wgrad    (layers.py:250-255, 157-160):  dW[r, co] = sum_pix im2col(X)[pix, r] * dY[pix, co]
//            split over pixels; db[co] = sum_pix dY[pix, co] from the same B
//            gather.
//
// Geometries this engine does not tile fall back to the SIMT kernels of
// net_simt.cu (tc_layer_supported).
#include "tc_gemm.cuh"

#include <algorithm>

namespace dqn {
bool conv1_wgrad_u8_ok(const dqn_net_desc *net);
int64_t conv1_wgrad_u8_scratch(const dqn_net_desc *net, int batch);
bool lin_tc_ok(const dqn_layer_desc &L, int batch);
int lin_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const float *x, const float *params,
                   float *y, int batch, bool side);
bool conv_tc_ok(const dqn_layer_desc &L);
int lin_tc_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
                 const float *mask, float *dx, int batch);
int conv1_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const uint8_t *x,
                     const float *params, float *y, int batch);
int conv_tc_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
                  const float *mask, float *dx, int batch);
int conv_tc_forward(cudaStream_t st, const dqn_layer_desc &L, const float *x, const float *params,
                    float *y, int batch, bool side);

namespace {

__device__ __forceinline__ float4 ld4(const float *p) {
  // 16-byte aligned by construction (C % 4 == 0, k % 4 == 0)
  return __ldg(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ float4 ld4(const uint8_t *p) {
  const uint32_t u = __ldg(reinterpret_cast<const unsigned int *>(p));
  return make_float4((float)(u & 0xFF), (float)((u >> 8) & 0xFF), (float)((u >> 16) & 0xFF),
                     (float)(u >> 24));
}
__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// four scalar loads along k for sources that are contiguous along rows
template <typename T>
__device__ __forceinline__ float4 ld4_strided(const T *p, int64_t stride, int n) {
  float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < n) v[i] = (float)__ldg(p + i * stride);
  return make_float4(v[0], v[1], v[2], v[3]);
}

// NHWC offset of the top-left input element of output pixel m's window.
__device__ __forceinline__ long long pixel_base(const Geo &g, int m) {
  const int P = g.OH * g.OW;
  const int img = m / P, p = m - img * P;
  const int oy = p / g.OW, ox = p - oy * g.OW;
  return (((long long)img * g.H + (long long)oy * g.sh) * g.W + (long long)ox * g.sw) * g.C;
}

// offset of patch element k = (i, j, c) relative to the window base
__device__ __forceinline__ int patch_off(const Geo &g, int k) {
  const int rowlen = g.fw * g.C;
  const int i = k / rowlen;
  return i * g.W * g.C + (k - i * rowlen);
}

__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }

// 16 consecutive values (4-aligned run) into v, or zeros
template <typename T>
__device__ __forceinline__ void ld16(const T *p, float (&v)[16]) {
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float4 q = ld4(p + 4 * t);
    v[4 * t] = q.x;
    v[4 * t + 1] = q.y;
    v[4 * t + 2] = q.z;
    v[4 * t + 3] = q.w;
  }
}
__device__ __forceinline__ void zero16(float (&v)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = 0.f;
}
__device__ __forceinline__ float4 ld4_rw(const float *p) { return *reinterpret_cast<const float4 *>(p); }

__device__ __forceinline__ float4 relu_mask(float4 v, const float *mask) {
  const float4 mk = ld4_rw(mask);
  v.x = mk.x > 0.f ? v.x : 0.f;
  v.y = mk.y > 0.f ? v.y : 0.f;
  v.z = mk.z > 0.f ? v.z : 0.f;
  v.w = mk.w > 0.f ? v.w : 0.f;
  return v;
}

// ---------------------------------------------------------------- forward
template <typename InT, int BN_>
struct FwdPol : tc::PolBase {
  static constexpr bool U8 = sizeof(InT) == 1;
  static constexpr bool SPLIT_A = !U8, SPLIT_B = true, BIAS_FROM_B = false;
  static constexpr bool B_MNC = true;
  static constexpr int BN = BN_;
  const InT *x;
  const float *w, *bias;
  float *y, *partial;
  float *bias_out, *bias_partial;       // unused
  int *counters;
  Geo g;
  int M, N, K, klen, relu, ksplits;
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int m, int) const { return m < M ? pixel_base(g, m) : -1; }
  // 16 | fw * C: a 16-run of k stays inside one patch row
  __device__ void a16(long long base, int k, int ke, float (&v)[16]) const {
    if (k >= ke) return zero16(v);
    ld16(x + base + patch_off(g, k), v);
  }
  __device__ long long b_row(int n, int) const { return n < N ? n : -1; }
  // W[k][n..n+3] for k..k+3 (row-contiguous source, transposed by the engine)
  __device__ void b4(long long n, int k, int ke, float4 (&v)[4]) const {
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = (k + t < ke) ? ld4(w + (int64_t)(k + t) * N + n) : zero4();
  }
  __device__ void final4(int m, int n, float4 v, int) const {
    float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float u = U8 ? __fdiv_rn(t[j], 255.0f) : t[j];
      u = __fadd_rn(u, bias[n + j]);
      if (relu && u < 0.f) u = 0.f;
      t[j] = u;
    }
    st4(y + (int64_t)m * N + n, make_float4(t[0], t[1], t[2], t[3]));
  }
};

// --------------------------------------------------------- linear dgrad
// dX[m, f] = sum_co dY[m, co] * W[f, co]  (W row-major [F][Cout])
template <int BN_>
struct LinDgradPol : tc::PolBase {
  static constexpr bool SPLIT_A = true, SPLIT_B = true, BIAS_FROM_B = false;
  static constexpr bool B_MNC = false;
  static constexpr int BN = BN_;
  const float *dy, *w, *mask;
  float *out, *partial;
  float *bias_out, *bias_partial;
  int *counters;
  int M, N, K, klen, ksplits;
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int m, int) const { return m < M ? (long long)m * K : -1; }
  __device__ void a16(long long base, int k, int ke, float (&v)[16]) const {
    if (k >= ke) return zero16(v);
    ld16(dy + base + k, v);
  }
  __device__ long long b_row(int n, int) const { return n < N ? (long long)n * K : -1; }
  __device__ int b_koff(int k) const { return k; }
  __device__ float4 b_ld(long long base, int ko) const { return ld4(w + base + ko); }
  __device__ void final4(int m, int n, float4 v, int) const {
    const int64_t o = (int64_t)m * N + n;
    st4(out + o, mask ? relu_mask(v, mask + o) : v);
  }
};

// The same with B's hi tiles loaded by TMA tensor loads (W is dense and
// K-major: rows n = input features, k = output channels, row stride K).
template <int BN_>
struct LinDgradTmaPol : LinDgradPol<BN_> {
  static constexpr bool B_TMA = true;
  CUtensorMap map;
  __device__ void b_tma(uint32_t dst, int n0, int k, int, uint64_t *bar) const {
    tc::tma_load_2d(dst, &map, k, n0, bar);
  }
};

// ----------------------------------------------------------- conv dgrad
// One stride phase (py, px) per blockIdx.z: rows are the input pixels
// (img, yq, xq) with y = yq*sh + py, x = xq*sw + px; k = (ti, tj, co).
template <int BN_>
struct ConvDgradPol : tc::PolBase {
  static constexpr bool SPLIT_A = true, SPLIT_B = true, BIAS_FROM_B = false;
  static constexpr bool B_MNC = false;
  static constexpr int BN = BN_;
  const float *dy, *w, *mask;
  float *out, *partial;
  float *bias_out, *bias_partial;
  int *counters;
  Geo g;
  int M, N, K;         // M = batch * max phase extent, N = C, K = (fh/sh)(fw/sw)Cout
  int batch, klen, ksplits;
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ void phase(int z, int &py, int &px, int &hq, int &wq) const {
    py = z / g.sw;
    px = z - py * g.sw;
    hq = (g.H - py + g.sh - 1) / g.sh;
    wq = (g.W - px + g.sw - 1) / g.sw;
  }
  // row base packs (img, yq, xq) of the input pixel; -1 beyond this phase
  __device__ long long a_row(int m, int z) const {
    int py, px, hq, wq;
    phase(z, py, px, hq, wq);
    const int per = hq * wq;
    if (m >= batch * per) return -1;
    const int img = m / per, r = m - img * per, yq = r / wq, xq = r - yq * wq;
    return ((long long)img << 32) | ((long long)yq << 16) | xq;
  }
  // k = (tap (ti, tj), co); Cout % 16 == 0 keeps a 16-run inside one tap
  __device__ void a16(long long rb, int k, int ke, float (&v)[16]) const {
    if (k >= ke) return zero16(v);
    const int img = (int)(rb >> 32), yq = (int)((rb >> 16) & 0xFFFF), xq = (int)(rb & 0xFFFF);
    const int tw = g.fw / g.sw;
    const int tap = k / g.N, co = k - tap * g.N;
    const int ti = tap / tw, tj = tap - ti * tw;
    const int oy = yq - ti, ox = xq - tj;
    if (oy < 0 || ox < 0 || oy >= g.OH || ox >= g.OW) return zero16(v);
    ld16(dy + (((int64_t)img * g.OH + oy) * g.OW + ox) * g.N + co, v);
  }
  // W[py + sh*ti][px + sw*tj][c][co] = row part (py, px, c) + k part (ti, tj, co)
  __device__ long long b_row(int c, int z) const {
    if (c >= N) return -1;
    int py, px, hq, wq;
    phase(z, py, px, hq, wq);
    return (((long long)py * g.fw + px) * g.C + c) * g.N;
  }
  __device__ int b_koff(int k) const {
    const int tw = g.fw / g.sw;
    const int tap = k / g.N, co = k - tap * g.N;
    const int ti = tap / tw, tj = tap - ti * tw;
    return ((g.sh * ti) * g.fw + g.sw * tj) * g.C * g.N + co;
  }
  __device__ float4 b_ld(long long base, int ko) const { return ld4(w + base + ko); }
  __device__ void final4(int m, int c, float4 v, int z) const {
    int py, px, hq, wq;
    phase(z, py, px, hq, wq);
    const int per = hq * wq;
    if (m >= batch * per) return;
    const int img = m / per, r = m - img * per, yq = r / wq, xq = r - yq * wq;
    const int y = yq * g.sh + py, x = xq * g.sw + px;
    const int64_t o = (((int64_t)img * g.H + y) * g.W + x) * g.C + c;
    st4(out + o, mask ? relu_mask(v, mask + o) : v);
  }
};

// ------------------------------------------------------------------ wgrad
// C[r, co] = sum_pix im2col(x)[pix, r] * dY[pix, co]; the reduction runs
// over pixels, so both operands are gathered 4 pixels at a time; the bias
// gradient is the column sum of the same dY gather.
template <typename InT, int BN_>
struct WgradPol : tc::PolBase {
  static constexpr bool U8 = sizeof(InT) == 1;
  static constexpr bool SPLIT_A = !U8, SPLIT_B = true, BIAS_FROM_B = true;
  static constexpr bool B_MNC = true;
  static constexpr int BN = BN_;
  const InT *x;
  int32_t *flags;                 // non-finite gradients are flagged as written (or nullptr)
  const float *dy;
  float *grad, *partial;
  float *bias_out, *bias_partial;
  int *counters;
  Geo g;
  int M, N, K, klen, ksplits;     // M = R (patch length), N = Cout, K = pixels
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int r, int) const {
    if (r >= M) return -1;
    return patch_off(g, r);
  }
  // patch element r at pixels pix..pix+15: a walk of the window bases along
  // the output rows (a warp's 32 lanes = 32 consecutive patch elements:
  // coalesced)
  __device__ void a16(long long roff, int pix, int ke, float (&v)[16]) const {
    const int P = g.OH * g.OW;
    const int img = pix / P, p = pix - img * P;
    int oy = p / g.OW, ox = p - oy * g.OW;
    // incremental walk over the window bases (one add per pixel)
    const InT *src = x + roff +
                     (((long long)img * g.H + (long long)oy * g.sh) * g.W + (long long)ox * g.sw) * g.C;
    const long long step = (long long)g.sw * g.C;
    const long long row_jump = ((long long)g.sh * g.W - (long long)(g.OW - 1) * g.sw) * g.C;
    const long long img_jump = ((long long)g.H * g.W - (long long)(g.OH - 1) * g.sh * g.W -
                                (long long)(g.OW - 1) * g.sw) * g.C;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = pix + i < ke ? (float)__ldg(src) : 0.f;
      if (++ox == g.OW) {
        ox = 0;
        if (++oy == g.OH) {
          oy = 0;
          src += img_jump;
        } else {
          src += row_jump;
        }
      } else {
        src += step;
      }
    }
  }
  __device__ long long b_row(int n, int) const { return n < N ? n : -1; }
  // dY[pix..pix+3][n..n+3]
  __device__ void b4(long long n, int pix, int ke, float4 (&v)[4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (pix + i < ke) ? ld4(dy + (int64_t)(pix + i) * N + n) : zero4();
  }
  __device__ void final4(int r, int n, float4 v, int) const {
    float *gp = grad + (int64_t)r * N + n;
    float4 o = ld4_rw(gp);
    if (U8) {
      v.x = __fdiv_rn(v.x, 255.0f); v.y = __fdiv_rn(v.y, 255.0f);
      v.z = __fdiv_rn(v.z, 255.0f); v.w = __fdiv_rn(v.w, 255.0f);
    }
    o.x = __fadd_rn(o.x, v.x); o.y = __fadd_rn(o.y, v.y);
    o.z = __fadd_rn(o.z, v.z); o.w = __fadd_rn(o.w, v.w);
    st4(gp, o);
    note_grad4(flags, o);
  }
  __device__ void note_bias(float b) const { note_grad(flags, b); }
};

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
#ifndef DQN_WGRAD_CAP
#define DQN_WGRAD_CAP 8
#endif
#ifdef DQN_TC_TRACE
int kDgradCap = 16;                 // diagnostic override
int kWgradCap = DQN_WGRAD_CAP;      // diagnostic override
#else
constexpr int kDgradCap = 16;       // linear dgrad split cap (measured best in the learner)
constexpr int kWgradCap = DQN_WGRAD_CAP;   // fp32 conv wgrad split cap at learner sizes
#endif

// ------------------------------------------------------------ host helpers
bool conv_ok(const dqn_layer_desc &L) {
  if (L.kind == DQN_LAYER_DUELING) return false;
  return L.in_c % 4 == 0 && (L.fw * L.in_c) % 4 == 0 && L.out_c % 16 == 0;
}

// forward split length: a function of K only (batch-independent rows);
// measured in the learner's graph: conv2 / conv3 (K = 512 / 576) best at
// 256-k splits, fc1 (K = 3136) at 8 splits
inline int fwd_klen(int K) {
  if (K >= 2048) return ceil_div(ceil_div(K, 8), tc::BK) * tc::BK;   // 8 splits (fc1: 448)
  if (K >= 512) return 256;
  return K;
}

// Split count for a grid of `tiles` output tiles of width bn, from a latency
// model of the engine measured with the trace build (tools/tc_trace.py): one
// CTA per SM, ~3 us per CTA for setup + first k-block + epilogue, ~0.8 us per
// further 32-k block, and a split-K fixup of ~1.5 us plus the tile's partials
// read by R reducer CTAs at ~70 KB/us each (R as in tc_gemm_kernel).
inline void split_k(int tiles, int K, int bn, int cap, int &klen, int &splits) {
  const int nkb = ceil_div(K, tc::BK);
  double best = 1e30;
  int bs = 1;
  for (int s = 1; s <= std::min(cap, nkb); ++s) {
    const int kl = ceil_div(ceil_div(K, s), tc::BK) * tc::BK;
    if (ceil_div(K, kl) != s) continue;              // same split as a smaller s
    const int waves = ceil_div(tiles * s, kNumSMs);
    const int R = std::min({tc::reducer_budget() / tiles + 1, 8, s});
    double t = waves * (3.0 + (kl / tc::BK - 1) * 0.8);
    if (s > 1) t += 1.5 + (double)s * tc::BM * bn * 4 / (70e3 * R);
    if (t < best - 1e-9) {
      best = t;
      bs = s;
    }
  }
  klen = ceil_div(ceil_div(K, bs), tc::BK) * tc::BK;
  splits = ceil_div(K, klen);
}

template <typename InT, int BN>
int fwd_launch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *params,
               float *y, float *scratch, int *counters, int batch) {
  FwdPol<InT, BN> p{};
  p.counters = counters;
  p.x = x;
  p.w = params + L.w_off;
  p.bias = params + L.b_off;
  p.y = y;
  p.partial = scratch;
  p.g = geo_of(L);
  p.M = batch * L.out_h * L.out_w;
  p.N = L.out_c;
  p.K = L.fh * L.fw * L.in_c;
  p.klen = fwd_klen(p.K);
  p.relu = L.relu;
  p.ksplits = ceil_div(p.K, p.klen);
  return tc::launch(st, p, p.ksplits, "tc_fwd");
}

template <typename InT>
int fwd_dispatch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *params,
                 float *y, float *scratch, int *counters, int batch) {
  const int N = L.out_c;
  if (N == 32)
    return fwd_launch<InT, 32>(st, L, x, params, y, scratch, counters, batch);
  if (N == 64) return fwd_launch<InT, 64>(st, L, x, params, y, scratch, counters, batch);
  if (N % 64 == 0) return fwd_launch<InT, 64>(st, L, x, params, y, scratch, counters, batch);
  return DQN_ERR_UNSUPPORTED;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
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

// 2-D map of a row-major [rows][K] fp32 matrix with 4 x BN boxes (one
// 16-byte k-chunk of BN rows); out-of-range elements read as zero
static bool make_kmajor_map(CUtensorMap *m, const float *base, int K, int rows, int bn) {
  const EncodeTiledFn fn = encode_tiled();
  if (!fn || ((uintptr_t)base % 16) || (K % 4)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  const cuuint32_t box[2] = {4, (cuuint32_t)bn};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
int lin_dgrad_launch_tma(cudaStream_t st, const float *dy, const float *w, const float *mask,
                         float *out, float *partial, int *counters, int M, int N, int K,
                         int cap) {
  LinDgradTmaPol<BN> p{};
  if (!make_kmajor_map(&p.map, w, K, N, BN)) return DQN_ERR_UNSUPPORTED;
  p.counters = counters;
  p.dy = dy;
  p.w = w;
  p.mask = mask;
  p.out = out;
  p.partial = partial;
  p.M = M;
  p.N = N;
  p.K = K;
  split_k(ceil_div(M, tc::BM) * ceil_div(N, BN), K, BN, cap, p.klen, p.ksplits);
  return tc::launch(st, p, p.ksplits, "tc_lin_dgrad_tma");
}

template <int BN>
int lin_dgrad_launch(cudaStream_t st, const float *dy, const float *w, const float *mask,
                     float *out, float *partial, int *counters, int M, int N, int K) {
  {   // B (the weights, dense K-major) by TMA tensor loads when the map encodes
    const int rc = lin_dgrad_launch_tma<BN>(st, dy, w, mask, out, partial, counters, M, N, K,
                                            kDgradCap);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
  }
  LinDgradPol<BN> p{};
  p.counters = counters;
  p.dy = dy;
  p.w = w;
  p.mask = mask;
  p.out = out;
  p.partial = partial;
  p.M = M;
  p.N = N;
  p.K = K;
  split_k(ceil_div(M, tc::BM) * ceil_div(N, BN), K, BN, kDgradCap, p.klen, p.ksplits);
  return tc::launch(st, p, p.ksplits, "tc_lin_dgrad");
}

int lin_dgrad(cudaStream_t st, const float *dy, const float *w, const float *mask, float *out,
              float *partial, int *counters, int M, int N, int K) {
  // tiles of at most 64 columns: two [big | small] accumulator pairs + the A
  // stages fit in TMEM
  // measured in the learner: fc1 dgrad (N = 3136) 1.4 % faster in 32-column
  // tiles (needs the even producer ring, tc_gemm.cuh Plan::STAGES)
  for (int bn : {32, 16}) {
    if (N % bn) continue;
    switch (bn) {
      case 64: return lin_dgrad_launch<64>(st, dy, w, mask, out, partial, counters, M, N, K);
      case 32: return lin_dgrad_launch<32>(st, dy, w, mask, out, partial, counters, M, N, K);
      default: return lin_dgrad_launch<16>(st, dy, w, mask, out, partial, counters, M, N, K);
    }
  }
  return DQN_ERR_UNSUPPORTED;
}

template <int BN>
int conv_dgrad_launch(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
                      const float *mask, float *out, float *scratch, int *counters, int batch) {
  ConvDgradPol<BN> p{};
  p.counters = counters;
  p.partial = scratch;
  p.dy = dy;
  p.w = w;
  p.mask = mask;
  p.out = out;
  p.g = geo_of(L);
  p.batch = batch;
  p.M = batch * ceil_div(L.in_h, L.sh) * ceil_div(L.in_w, L.sw);
  p.N = L.in_c;
  p.K = (L.fh / L.sh) * (L.fw / L.sw) * L.out_c;
  // split K until phases x tiles x splits fill the machine (cap 4: measured
  // best in the learner; conv dgrad B by 4-D TMA tensor loads was bit-identical
  // but 6 % slower there -- few k-blocks per CTA leave its latency exposed)
  split_k(L.sh * L.sw * ceil_div(p.M, tc::BM) * ceil_div(p.N, BN), p.K, BN, 4, p.klen, p.ksplits);
  return tc::launch(st, p, L.sh * L.sw * p.ksplits, "tc_conv_dgrad");
}

bool dgrad_tile_ok(int C) { return C == 16 || C == 32 || C == 48 || C % 64 == 0; }

int conv_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *w,
               const float *mask, float *out, float *scratch, int *counters, int batch) {
  switch (L.in_c) {
    case 16: return conv_dgrad_launch<16>(st, L, dy, w, mask, out, scratch, counters, batch);
    case 32: return conv_dgrad_launch<32>(st, L, dy, w, mask, out, scratch, counters, batch);
    case 48: return conv_dgrad_launch<48>(st, L, dy, w, mask, out, scratch, counters, batch);
    case 64: return conv_dgrad_launch<64>(st, L, dy, w, mask, out, scratch, counters, batch);
    default: break;
  }
  if (L.in_c % 64 == 0) return conv_dgrad_launch<64>(st, L, dy, w, mask, out, scratch, counters, batch);
  set_error("tc_conv_dgrad: %d input channels not tiled", L.in_c);
  return DQN_ERR_UNSUPPORTED;
}

inline void wgrad_split(int M, int N, int K, int bn, bool u8, int &klen, int &splits) {
  // split lengths a multiple of BK, count from the latency model, capped at
  // learner-sized reductions (K <= 64k pixels): the wgrads run beside the
  // dgrad chain, and the model's count for one launch alone (conv3: 25
  // one-block splits over 125 CTAs) takes the SMs the chain needs.  Measured
  // in the learner's graph (cfg4, batch 32): round 2 with the register-fed
  // forward, caps 4 / 8 / 12 / 16 / 128 -> 8 best.  With the TMA-fed conv
  // kernels the trace build preferred 12 (+1.7 %), but two product builds
  // (cap 8 vs 12, bench.py interleaved three times) gave 7,531-7,542 vs
  // 7,521-7,526: the trace build's engine marks bias engine-side A/Bs.
  // Large batches (K > 64k) keep the model's count.
  const int cap = K <= 65536 ? (u8 ? 32 : kWgradCap) : 128;
  split_k(ceil_div(M, tc::BM) * ceil_div(N, bn), K, bn, cap, klen, splits);
}

template <typename InT, int BN>
int wgrad_launch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *dy, float *grads, float *scratch, int *counters, int batch,
                 int32_t *flags) {
  WgradPol<InT, BN> p{};
  p.flags = flags;
  p.counters = counters;
  p.x = x;
  p.dy = dy;
  p.grad = grads + L.w_off;
  p.bias_out = grads + L.b_off;
  p.g = geo_of(L);
  p.M = L.fh * L.fw * L.in_c;
  p.N = L.out_c;
  p.K = batch * L.out_h * L.out_w;
  int splits;
  wgrad_split(p.M, p.N, p.K, BN, sizeof(InT) == 1, p.klen, splits);
  p.partial = scratch;
  p.bias_partial = scratch + (int64_t)splits * p.M * p.N;
  p.ksplits = splits;
  return tc::launch(st, p, splits, "tc_wgrad");
}

template <typename InT>
int wgrad_dispatch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *dy, float *grads, float *scratch, int *counters, int batch,
                   int32_t *flags) {
  const int N = L.out_c;
  if (N == 32) return wgrad_launch<InT, 32>(st, L, x, dy, grads, scratch, counters, batch, flags);
  if (N % 64 == 0)
    return wgrad_launch<InT, 64>(st, L, x, dy, grads, scratch, counters, batch, flags);
  return DQN_ERR_UNSUPPORTED;
}

int64_t wgrad_scratch_tc(const dqn_layer_desc &L, int batch) {
  const int M = L.fh * L.fw * L.in_c, N = L.out_c, K = batch * L.out_h * L.out_w;
  int klen, splits = 1;
  for (int bn : {32, 64})                    // either tile width and input type
    for (bool u8 : {false, true}) {
      int sp;
      wgrad_split(M, N, K, bn, u8, klen, sp);
      splits = std::max(splits, sp);
    }
  return (int64_t)splits * M * N + (int64_t)splits * N;
}

}  // namespace

// phase: 0 forward, 1 dgrad, 2 wgrad
bool tc_layer_supported(const dqn_net_desc *net, int l, int phase) {
  const dqn_layer_desc &L = net->layer[l];
  if (!conv_ok(L)) return false;
  if (L.kind == DQN_LAYER_LINEAR && l == net->n_layers - 1 && L.out_c <= 32) return false;  // head
  const int N = L.out_c;
  if (!(N == 32 || N == 64 || N % 128 == 0)) return false;
  if (phase == 0 && (L.fw * L.in_c) % 16) return false;      // A rows gathered in 16-runs
  if (phase == 1 && L.kind == DQN_LAYER_CONV &&
      (L.fh % L.sh || L.fw % L.sw || !dgrad_tile_ok(L.in_c)))
    return false;
  return true;
}

int64_t tc_scratch_floats(const dqn_net_desc *net, int batch) {
  int64_t m = conv1_wgrad_u8_ok(net) ? conv1_wgrad_u8_scratch(net, batch) : 0;
  for (int l = 0; l < net->n_layers; ++l) {
    if (!tc_layer_supported(net, l, 0)) continue;
    const dqn_layer_desc &L = net->layer[l];
    const int M = batch * L.out_h * L.out_w, R = L.fh * L.fw * L.in_c, K = R;
    const int fs = ceil_div(K, fwd_klen(K));
    m = std::max(m, fs > 1 ? (int64_t)fs * M * L.out_c : 0);
    if (L.kind == DQN_LAYER_LINEAR)     // lin dgrad partials: split_k caps at 16 splits
      m = std::max(m, (int64_t)std::min(16, ceil_div(L.out_c, tc::BK)) * M * R);
    if (L.kind == DQN_LAYER_CONV && tc_layer_supported(net, l, 1)) {
      const int Kd = (L.fh / L.sh) * (L.fw / L.sw) * L.out_c;
      const int ds = std::max(1, std::min(ceil_div(Kd, tc::BK), 16));   // split_k upper bound
      const int64_t Md = (int64_t)batch * ceil_div(L.in_h, L.sh) * ceil_div(L.in_w, L.sw);
      if (ds > 1) m = std::max(m, (int64_t)L.sh * L.sw * ds * Md * L.in_c);
    }
    m = std::max(m, wgrad_scratch_tc(L, batch));
  }
  return m;
}

// split-K tile counters live in the last kMaxTiles slots of the binding scratch
static int *counters_of(const dqn_binding *b) {
  return reinterpret_cast<int *>(b->scratch + b->scratch_floats - tc::kMaxTiles);
}

#ifdef DQN_TC_TRACE
int g_c1_enabled = 1;   // diagnostic: 0 = conv1 forward on the generic engine
#else
constexpr int g_c1_enabled = 1;
#endif

int tc_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                     const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  // hidden linear layers at learner batch sizes: the TMA-fed weight-streaming
  // kernel (lin_tc.cu; measured +0.3 % in the learner -- its dgrad form was
  // slower than the engine's LinDgradTmaPol there and is not used)
  if (L.kind == DQN_LAYER_LINEAR && l > 0 && lin_tc_ok(L, b->batch)) {
    const int rc = lin_tc_forward(st, L, (const float *)in, params, b->act[l], b->batch,
                                  (net->hints & DQN_NET_HINT_SIDE) != 0);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
  }
  // fp32-input convolutions: both operands by TMA (conv_tc.cu)
  if (L.kind == DQN_LAYER_CONV && !(l == 0 && net->input_u8) && conv_tc_ok(L)) {
    const int rc = conv_tc_forward(st, L, (const float *)in, params, b->act[l], b->batch,
                                   (net->hints & DQN_NET_HINT_SIDE) != 0);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
  }
  // the uint8 first convolution: frame slab + W by bulk copies (conv1_tc.cu)
  if (l == 0 && net->input_u8 && g_c1_enabled) {
    const int rc = conv1_tc_forward(st, L, (const uint8_t *)in, params, b->act[l], b->batch);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
  }
  if (l == 0 && net->input_u8)
    return fwd_dispatch<uint8_t>(st, L, (const uint8_t *)in, params, b->act[l], b->scratch,
                                  counters_of(b), b->batch);
  return fwd_dispatch<float>(st, L, (const float *)in, params, b->act[l], b->scratch,
                              counters_of(b), b->batch);
}

int tc_layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                      const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  float *out = (l == 0) ? b->dx : b->dact[l - 1];
  if (out == nullptr) return DQN_OK;
  const float *mask = (l > 0 && net->layer[l - 1].relu) ? b->act[l - 1] : nullptr;
  const float *w = params + L.w_off;
  if (L.kind == DQN_LAYER_LINEAR) {
    const int M = b->batch, F = L.in_h * L.in_w * L.in_c;
    const int rc = lin_tc_dgrad(st, L, b->dact[l], w, mask, out, b->batch);
    if (rc != DQN_ERR_UNSUPPORTED) return rc;
    return lin_dgrad(st, b->dact[l], w, mask, out, b->scratch, counters_of(b), M, F, L.out_c);
  }
  // dY and W by TMA, one GEMM per stride phase (conv_tc.cu)
  const int rc = conv_tc_dgrad(st, L, b->dact[l], w, mask, out, b->batch);
  if (rc != DQN_ERR_UNSUPPORTED) return rc;
  return conv_dgrad(st, L, b->dact[l], w, mask, out, b->scratch, counters_of(b), b->batch);
}

int tc_layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                   const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  if (l == 0 && net->input_u8)
    return wgrad_dispatch<uint8_t>(st, L, (const uint8_t *)in, b->dact[l], grads, b->scratch,
                                    counters_of(b), b->batch, flags);
  return wgrad_dispatch<float>(st, L, (const float *)in, b->dact[l], grads, b->scratch,
                                counters_of(b), b->batch, flags);
}


}  // namespace dqn

#ifdef DQN_TC_TRACE
// copies (and resets) the per-CTA trace records of tc_gemm_kernel launches
extern "C" int dqn_tc_trace(unsigned long long *host, int max_ctas) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, dqn::tc::g_trace_n, sizeof(n));
  if (n > (unsigned)dqn::tc::kTraceCtas) n = dqn::tc::kTraceCtas;
  if ((int)n > max_ctas) n = max_ctas;
  if (n) cudaMemcpyFromSymbol(host, dqn::tc::g_trace, 30ull * n * sizeof(unsigned long long));
  const unsigned int zero = 0;
  cudaMemcpyToSymbol(dqn::tc::g_trace_n, &zero, sizeof(zero));
  return (int)n;
}
extern "C" void dqn_c1_set(int on) { dqn::g_c1_enabled = on; }
extern "C" void dqn_tc_set_dgrad_cap(int c) { dqn::kDgradCap = c; }
extern "C" void dqn_tc_set_wgrad_cap(int c) { dqn::kWgradCap = c; }
extern "C" void dqn_tc_set_cluster_splitk(int on) { dqn::tc::cluster_splitk_override() = on; }
extern "C" void dqn_tc_skip(int mask) { cudaMemcpyToSymbol(dqn::tc::g_skip, &mask, sizeof(mask)); }
#endif
