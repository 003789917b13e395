// Generic-geometry Q-network kernels (SIMT fp32).  These cover every layer
// geometry the reference accepts (layers.py:163-330: NHWC valid convolution,
// linear with implicit flatten, ReLU, dueling head) and are the parity
// baseline for the tcgen05 trunk in trunk_tc.cu.
//
// Reference call sites replaced:
//   ConvolutionLayer.forward       layers.py:226-233 -> conv_fwd_kernel (implicit GEMM, no im2col buffer)
//   ConvolutionLayer.backward      layers.py:235-248 -> conv_dgrad_kernel (gather form: no col2im scatter, no atomics)
//   ConvolutionLayer.calculate_gradient layers.py:250-255 -> wgrad_kernel + wgrad_reduce_kernel
//   LinearLayer.*                  layers.py:148-160 -> same kernels with 1x1 geometry
//   ReluLayer                      layers.py:108-112 -> fused into epilogues (fwd) / masks (bwd)
//   DuelingHeadLayer               layers.py:302-330 -> head_fwd/head_bwd/head_wgrad kernels
//
// Determinism (reference tests test_layers.py:60-67, test_network.py:95-103):
// every reduction has a fixed order that does not depend on the batch size
// of OTHER rows; split-K partials are summed in split order; no float atomics.
#include "common.cuh"

#include <algorithm>

namespace dqn {
namespace {

constexpr int BM = 64;
constexpr int BK = 16;
constexpr int APAD = 4;


__device__ __forceinline__ float lift(uint8_t v) { return __fdiv_rn((float)v, 255.0f); }
__device__ __forceinline__ float lift(float v) { return v; }

// 4x4 register micro-tile update from one BK slice in shared memory.
template <int BN>
__device__ __forceinline__ void micro_mma(const float (*As)[BM + APAD], const float (*Bs)[BN + APAD],
                                          int ty, int tx, float acc[4][4]) {
#pragma unroll
  for (int kk = 0; kk < BK; ++kk) {
    const float4 a = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
    const float4 b = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
  }
}

// ----------------------------------------------------------- forward GEMM
// y[m, n] = relu( sum_k x_im2col[m, k] * W[k, n] + b[n] ),  m = (img, oy, ox),
// k = (i, j, c) in the (fh, fw, cin, cout) filter order of layers.py:198-199.
// TB: B is stored transposed (W[n, k], the dgrad operand W^T); bias may be
// NULL; ``mask`` (optional) zeroes outputs whose mask value is <= 0 (ReLU
// backward of the layer below, layers.py:112).
template <typename InT, int BN, bool TB>
__global__ void __launch_bounds__(BM *BN / 16)
conv_fwd_kernel(const InT *__restrict__ x, const float *__restrict__ w,
                const float *__restrict__ bias, float *__restrict__ y,
                float *__restrict__ partial, Geo g, int M, int K, int klen, int relu,
                const float *__restrict__ mask) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  constexpr int THREADS = BM * BN / 16;
  __shared__ __align__(16) float As[BK][BM + APAD];
  __shared__ __align__(16) float Bs[BK][BN + APAD];
  __shared__ int64_t s_row[BM];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / 4), ty = tid / (BN / 4);
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * klen, kend = min(K, kbeg + klen);
  const int P = g.OH * g.OW;
  for (int r = tid; r < BM; r += THREADS) {
    const int m = m0 + r;
    int64_t off = -1;
    if (m < M) {
      const int img = m / P, p = m % P;
      const int oy = p / g.OW, ox = p % g.OW;
      off = (int64_t)img * g.H * g.W * g.C + ((int64_t)oy * g.sh * g.W + (int64_t)ox * g.sw) * g.C;
    }
    s_row[r] = off;
  }
  __syncthreads();
  const int rowlen = g.fw * g.C;        // (j, c) are contiguous in NHWC
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int q = 0; q < BM * BK / THREADS; ++q) {
      const int e = tid + q * THREADS;
      const int kk = e % BK, mm = e / BK;
      const int k = k0 + kk;
      float v = 0.f;
      const int64_t ro = s_row[mm];
      if (k < kend && ro >= 0) {
        const int i = k / rowlen, rem = k - i * rowlen;
        v = lift(x[ro + (int64_t)i * g.W * g.C + rem]);
      }
      As[kk][mm] = v;
    }
#pragma unroll
    for (int q = 0; q < BK * BN / THREADS; ++q) {
      const int e = tid + q * THREADS;
      if (TB) {                                   // coalesce along k
        const int kk = e % BK, nn = e / BK;
        const int k = k0 + kk, n = n0 + nn;
        Bs[kk][nn] = (k < kend && n < g.N) ? w[(int64_t)n * K + k] : 0.f;
      } else {
        const int nn = e % BN, kk = e / BN;
        const int k = k0 + kk, n = n0 + nn;
        Bs[kk][nn] = (k < kend && n < g.N) ? w[(int64_t)k * g.N + n] : 0.f;
      }
    }
    __syncthreads();
    micro_mma<BN>(As, Bs, ty, tx, acc);
    __syncthreads();
  }
  const bool split = gridDim.z > 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      if (split) {
        partial[((int64_t)blockIdx.z * M + m) * g.N + n] = acc[i][j];
      } else {
        float v = bias ? __fadd_rn(acc[i][j], bias[n]) : acc[i][j];
        if (relu && v < 0.f) v = 0.f;   // np.maximum(x, 0) keeps NaN
        const int64_t o = (int64_t)m * g.N + n;
        if (mask && !(mask[o] > 0.f)) v = 0.f;
        y[o] = v;
      }
    }
  }
}

// Fixed-order split-K reduction + bias + ReLU (+ mask).
__global__ void splitk_bias_kernel(const float *__restrict__ partial, int splits, int64_t MN,
                                   int N, const float *__restrict__ bias, float *__restrict__ y,
                                   int relu, const float *__restrict__ mask) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MN;
       e += (int64_t)gridDim.x * blockDim.x) {
    float s = partial[e];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, partial[(int64_t)z * MN + e]);
    float v = bias ? __fadd_rn(s, bias[e % N]) : s;
    if (relu && v < 0.f) v = 0.f;   // np.maximum(x, 0) keeps NaN
    if (mask && !(mask[e] > 0.f)) v = 0.f;
    y[e] = v;
  }
}

// col2im as a gather (layers.py:240-248 scatter-adds one strided slice per
// filter tap): dx[img, y, x, c] = sum over taps (i ascending, j ascending)
// with y = oy*sh + i, x = ox*sw + j of dpatch[(img, oy, ox), (i, j, c)] --
// the same per-element summation order as the reference's tap loop, no
// atomics.  Optional ReLU mask of the layer below.
__global__ void col2im_kernel(const float *__restrict__ dpatch, Geo g, int64_t total,
                              const float *__restrict__ mask, float *__restrict__ dx) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int R = g.fh * g.fw * g.C;
  // element index fits 32 bits for any learner batch (checked by the caller)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)total;
       e += gridDim.x * blockDim.x) {
    const int c = e % g.C;
    int t = e / g.C;
    const int x = t % g.W;
    t /= g.W;
    const int y = t % g.H;
    const int img = t / g.H;
    float s = 0.f;
    for (int i = y % g.sh; i < g.fh; i += g.sh) {
      const int oy = (y - i) / g.sh;
      if (y - i < 0 || oy >= g.OH) continue;
      for (int j = x % g.sw; j < g.fw; j += g.sw) {
        const int ox = (x - j) / g.sw;
        if (x - j < 0 || ox >= g.OW) continue;
        const int64_t m = ((int64_t)img * g.OH + oy) * g.OW + ox;
        s = __fadd_rn(s, dpatch[m * R + (i * g.fw + j) * g.C + c]);
      }
    }
    if (mask && !(mask[e] > 0.f)) s = 0.f;
    dx[e] = s;
  }
}

// ------------------------------------------------------------- wgrad GEMM
// partial[z, r, n] = sum_{m in split z} x_im2col[m, r] * dy[m, n]; the
// blocks of row tile 0 also produce partial column sums of dy (bias grads).
template <typename InT, int BN>
__global__ void __launch_bounds__(BM *BN / 16)
wgrad_kernel(const InT *__restrict__ x, const float *__restrict__ dy, float *__restrict__ partial,
             float *__restrict__ bpartial, Geo g, int M, int R, int mlen) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  constexpr int THREADS = BM * BN / 16;
  __shared__ __align__(16) float As[BK][BM + APAD];
  __shared__ __align__(16) float Bs[BK][BN + APAD];
  __shared__ int64_t s_koff[BM];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / 4), ty = tid / (BN / 4);
  const int r0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int mbeg = blockIdx.z * mlen, mend = min(M, mbeg + mlen);
  const int P = g.OH * g.OW;
  const int rowlen = g.fw * g.C;
  for (int rr = tid; rr < BM; rr += THREADS) {
    const int r = r0 + rr;
    int64_t off = -1;
    if (r < R) {
      const int i = r / rowlen, rem = r - i * rowlen;
      off = (int64_t)i * g.W * g.C + rem;
    }
    s_koff[rr] = off;
  }
  __syncthreads();
  const bool do_bias = (blockIdx.x == 0) && (ty == 0);
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  float acc[4][4] = {};
  for (int mk = mbeg; mk < mend; mk += BK) {
    // A slice: rows r (BM), reduction m (BK)
#pragma unroll
    for (int q = 0; q < BM * BK / THREADS; ++q) {
      const int e = tid + q * THREADS;
      const int rr = e % BM, kk = e / BM;
      const int m = mk + kk;
      float v = 0.f;
      if (m < mend && s_koff[rr] >= 0) {
        const int img = m / P, p = m - img * P;
        const int oy = p / g.OW, ox = p - oy * g.OW;
        const int64_t ro =
            (int64_t)img * g.H * g.W * g.C + ((int64_t)oy * g.sh * g.W + (int64_t)ox * g.sw) * g.C;
        v = lift(x[ro + s_koff[rr]]);
      }
      As[kk][rr] = v;
    }
#pragma unroll
    for (int q = 0; q < BK * BN / THREADS; ++q) {
      const int e = tid + q * THREADS;
      const int nn = e % BN, kk = e / BN;
      const int m = mk + kk, n = n0 + nn;
      Bs[kk][nn] = (m < mend && n < g.N) ? dy[(int64_t)m * g.N + n] : 0.f;
    }
    __syncthreads();
    micro_mma<BN>(As, Bs, ty, tx, acc);
    if (do_bias) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk)
#pragma unroll
        for (int j = 0; j < 4; ++j) bsum[j] = __fadd_rn(bsum[j], Bs[kk][tx * 4 + j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= R) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < g.N) partial[((int64_t)blockIdx.z * R + r) * g.N + n] = acc[i][j];
    }
  }
  if (do_bias) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < g.N) bpartial[(int64_t)blockIdx.z * g.N + n] = bsum[j];
    }
  }
}

// grad += sum_z partial[z]  (fixed order); bias likewise.
__global__ void wgrad_reduce_kernel(const float *__restrict__ partial,
                                    const float *__restrict__ bpartial, int splits, int64_t RN,
                                    int N, float *__restrict__ gw, float *__restrict__ gb,
                                    int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int64_t total = RN + N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < RN) {
      float s = partial[e];
      for (int z = 1; z < splits; ++z) s = __fadd_rn(s, partial[(int64_t)z * RN + e]);
      acc_grad(&gw[e], s, flags);
    } else {
      const int n = (int)(e - RN);
      float s = bpartial[n];
      for (int z = 1; z < splits; ++z) s = __fadd_rn(s, bpartial[(int64_t)z * N + n]);
      acc_grad(&gb[n], s, flags);
    }
  }
}

// -------------------------------------------------------------- the head
// One CTA per sample row: V/A (or plain linear) dot products over F features,
// fixed-order tree reduction in shared memory.
constexpr int kHeadThreads = 128;
constexpr int kMaxHeadOut = 33;   // 1 value + up to 32 actions

__global__ void __launch_bounds__(kHeadThreads)
head_fwd_kernel(const float *__restrict__ x, int F, const float *__restrict__ wv,
                const float *__restrict__ bv, const float *__restrict__ wa,
                const float *__restrict__ ba, int nA, int dueling, float *__restrict__ q,
                int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ float red[kMaxHeadOut][kHeadThreads];
  const int row = blockIdx.x, t = threadIdx.x;
  const float *xr = x + (int64_t)row * F;
  const int nout = dueling ? nA + 1 : nA;
  float part[kMaxHeadOut];
#pragma unroll
  for (int o = 0; o < kMaxHeadOut; ++o) part[o] = 0.f;
  for (int f = t; f < F; f += kHeadThreads) {
    const float xv = xr[f];
    if (dueling) {
      part[0] = fmaf(xv, wv[f], part[0]);
      for (int a = 0; a < nA; ++a) part[a + 1] = fmaf(xv, wa[(int64_t)f * nA + a], part[a + 1]);
    } else {
      for (int a = 0; a < nA; ++a) part[a] = fmaf(xv, wa[(int64_t)f * nA + a], part[a]);
    }
  }
  for (int o = 0; o < nout; ++o) red[o][t] = part[o];
  __syncthreads();
  for (int s = kHeadThreads / 2; s > 0; s >>= 1) {
    if (t < s)
      for (int o = 0; o < nout; ++o) red[o][t] = __fadd_rn(red[o][t], red[o][t + s]);
    __syncthreads();
  }
  if (t == 0) {
    bool bad = false;
    if (dueling) {
      // layers.py:302-310: y = V; y += A; y -= mean(A)
      const float v = __fadd_rn(red[0][0], bv[0]);
      float adv[kMaxHeadOut];
      float sum = 0.f;
      for (int a = 0; a < nA; ++a) {
        adv[a] = __fadd_rn(red[a + 1][0], ba[a]);
        sum = __fadd_rn(sum, adv[a]);
      }
      const float mean = __fdiv_rn(sum, (float)nA);
      for (int a = 0; a < nA; ++a) {
        const float qa = __fsub_rn(__fadd_rn(v, adv[a]), mean);
        bad |= !isfinite(qa);
        q[(int64_t)row * nA + a] = qa;
      }
    } else {
      for (int a = 0; a < nA; ++a) {
        const float qa = __fadd_rn(red[a][0], ba[a]);
        bad |= !isfinite(qa);
        q[(int64_t)row * nA + a] = qa;
      }
    }
    if (bad) raise_flag(flags, DQN_FLAG_NONFINITE_OUT);
  }
}

// Head backward (layers.py:312-323): gv = sum_a g, ga = g - gv/nA,
// dx = gv*Wv^T + ga*Wa^T (plain head: g*W^T), masked by the input ReLU.
__global__ void head_bwd_kernel(const float *__restrict__ dq, int B, int nA, int dueling,
                                const float *__restrict__ wv, const float *__restrict__ wa, int F,
                                const float *__restrict__ mask_act, float *__restrict__ dx) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  const int64_t total = (int64_t)B * F;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / F), f = (int)(e % F);
    const float *g = dq + (int64_t)row * nA;
    float v;
    if (dueling) {
      float gv = 0.f;
      for (int a = 0; a < nA; ++a) gv = __fadd_rn(gv, g[a]);
      const float gvn = __fdiv_rn(gv, (float)nA);
      float s = 0.f;
      for (int a = 0; a < nA; ++a) s = fmaf(__fsub_rn(g[a], gvn), wa[(int64_t)f * nA + a], s);
      v = __fadd_rn(__fmul_rn(gv, wv[f]), s);
    } else {
      float s = 0.f;
      for (int a = 0; a < nA; ++a) s = fmaf(g[a], wa[(int64_t)f * nA + a], s);
      v = s;
    }
    if (mask_act != nullptr && !(mask_act[e] > 0.f)) v = 0.f;
    dx[e] = v;
  }
}

// Head wgrad (layers.py:325-330): a CTA owns 128 consecutive input features
// (feature F = the bias row); per 64-row chunk the branch gradients
// (gv = sum_a g, ga = g - gv/nA) and the feature tile are staged in shared
// memory, then every thread reduces its feature over rows in fixed order.
constexpr int kHeadRows = 64;
__global__ void __launch_bounds__(128)
head_wgrad_kernel(const float *__restrict__ x, const float *__restrict__ dq, int B, int F, int nA,
                  int dueling, float *__restrict__ gwv, float *__restrict__ gbv,
                  float *__restrict__ gwa, float *__restrict__ gba, int32_t *flags) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  __shared__ float xs[kHeadRows][128];
  __shared__ float gs[kHeadRows][kMaxHeadOut];
  const int nout = dueling ? nA + 1 : nA;
  const int t = threadIdx.x;
  const int f = blockIdx.x * 128 + t;
  float acc[kMaxHeadOut];
#pragma unroll
  for (int o = 0; o < kMaxHeadOut; ++o) acc[o] = 0.f;
  for (int r0 = 0; r0 < B; r0 += kHeadRows) {
    const int nr = min(kHeadRows, B - r0);
    __syncthreads();
    for (int r = 0; r < nr; ++r)
      xs[r][t] = (f < F) ? x[(int64_t)(r0 + r) * F + f] : 1.f;
    for (int r = t; r < nr; r += 128) {
      const float *g = dq + (int64_t)(r0 + r) * nA;
      if (dueling) {
        float gv = 0.f;
        for (int a = 0; a < nA; ++a) gv = __fadd_rn(gv, g[a]);
        gs[r][0] = gv;
        const float gvn = __fdiv_rn(gv, (float)nA);
        for (int a = 0; a < nA; ++a) gs[r][a + 1] = __fsub_rn(g[a], gvn);
      } else {
        for (int a = 0; a < nA; ++a) gs[r][a] = g[a];
      }
    }
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      const float xv = xs[r][t];
#pragma unroll
      for (int o = 0; o < kMaxHeadOut; ++o)
        if (o < nout) acc[o] = fmaf(xv, gs[r][o], acc[o]);
    }
  }
  if (f > F) return;
#pragma unroll
  for (int o = 0; o < kMaxHeadOut; ++o) {
    if (o >= nout) break;
    const float s = acc[o];
    if (dueling) {
      if (o == 0) {
        if (f < F) acc_grad(&gwv[f], s, flags); else acc_grad(&gbv[0], s, flags);
      } else {
        if (f < F) acc_grad(&gwa[(int64_t)f * nA + o - 1], s, flags);
        else acc_grad(&gba[o - 1], s, flags);
      }
    } else {
      if (f < F) acc_grad(&gwa[(int64_t)f * nA + o], s, flags);
      else acc_grad(&gba[o], s, flags);
    }
  }
}

// ------------------------------------------------------------ host plans


inline bool is_head(const dqn_net_desc *net, int l) {
  const dqn_layer_desc &L = net->layer[l];
  return L.kind == DQN_LAYER_DUELING || (l == net->n_layers - 1 && L.kind == DQN_LAYER_LINEAR &&
                                         L.out_c <= kMaxHeadOut - 1);
}

// split-K factor of a forward GEMM.  It depends on the reduction length
// only, never on the batch, so every output row is computed in the same order
// whatever batch it arrives in (batch-rebinding bit-exactness,
// test_network.py:95-103).
inline int fwd_splits(int /*M*/, int /*N*/, int K, int /*BN*/) {
  if (K >= 2048) return 16;
  if (K >= 512) return 4;
  return 1;
}

inline int wgrad_splits(int R, int N, int M, int BN) {
  const int tiles = ((R + BM - 1) / BM) * ((N + BN - 1) / BN);
  int s = 1;
  while (tiles * s < 2 * kNumSMs && M / (s + 1) >= 8 * BK) ++s;
  return s;
}

inline int pick_bn(int N) { return N <= 32 ? 32 : 64; }

inline int64_t gemm_scratch(int M, int N, int K) {
  const int s = fwd_splits(M, N, K, pick_bn(N));
  return s > 1 ? (int64_t)s * M * N : 0;
}

inline int64_t fwd_scratch(const dqn_layer_desc &L, int batch) {
  if (L.kind == DQN_LAYER_DUELING) return 0;
  return gemm_scratch(batch * L.out_h * L.out_w, L.out_c, L.fh * L.fw * L.in_c);
}

// dgrad = GEMM dY * W^T (conv: into a dpatch buffer, then col2im gather)
inline int64_t dgrad_scratch(const dqn_layer_desc &L, int batch) {
  if (L.kind == DQN_LAYER_DUELING) return 0;
  const int M = batch * L.out_h * L.out_w, R = L.fh * L.fw * L.in_c;
  const bool conv = L.kind == DQN_LAYER_CONV;
  return (conv ? (int64_t)M * R : 0) + gemm_scratch(M, R, L.out_c);
}

inline int64_t wgrad_scratch(const dqn_layer_desc &L, int batch) {
  if (L.kind == DQN_LAYER_DUELING) return 0;
  const int M = batch * L.out_h * L.out_w, R = L.fh * L.fw * L.in_c;
  const int s = wgrad_splits(R, L.out_c, M, pick_bn(L.out_c));
  return (int64_t)s * R * L.out_c + (int64_t)s * L.out_c;
}

// C[M, g.N] = A_im2col(x; g)[M, K] * B[K, g.N] (B transposed when TB), with
// optional bias / ReLU / mask epilogue; fixed K-only split-K.
template <typename InT, bool TB>
int launch_gemm(cudaStream_t st, const InT *x, const Geo &g, const float *w, const float *bias,
                const float *mask, int relu, float *y, float *scratch, int M, int K) {
  const int bn = pick_bn(g.N);
  const int s = fwd_splits(M, g.N, K, bn);
  int klen = (K + s - 1) / s;
  klen = (klen + BK - 1) / BK * BK;
  const int splits = (K + klen - 1) / klen;
  dim3 grid((M + BM - 1) / BM, (g.N + bn - 1) / bn, splits);
  if (bn == 32)
    launch_k(conv_fwd_kernel<InT, 32, TB>, grid, BM * 32 / 16, 0, st, x, w, bias, y, scratch, g, M, K,
                                                                klen, relu, mask);
  else
    launch_k(conv_fwd_kernel<InT, 64, TB>, grid, BM * 64 / 16, 0, st, x, w, bias, y, scratch, g, M, K,
                                                                klen, relu, mask);
  DQN_LAUNCH_CHECK("gemm");
  if (splits > 1) {
    const int64_t MN = (int64_t)M * g.N;
    launch_k(splitk_bias_kernel, (int)std::min<int64_t>((MN + 255) / 256, 148 * 8), 256, 0, st, 
        scratch, splits, MN, g.N, bias, y, relu, mask);
    DQN_LAUNCH_CHECK("splitk_bias");
  }
  return DQN_OK;
}

template <typename InT>
int launch_fwd(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *params,
               float *y, float *scratch, int batch) {
  Geo g = geo_of(L);
  const int M = batch * g.OH * g.OW, K = g.fh * g.fw * g.C;
  return launch_gemm<InT, false>(st, x, g, params + L.w_off, params + L.b_off, nullptr, L.relu,
                                 y, scratch, M, K);
}

template <typename InT>
int launch_wgrad(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *dy,
                 float *grads, float *scratch, int batch, int32_t *flags) {
  Geo g = geo_of(L);
  const int M = batch * g.OH * g.OW, R = g.fh * g.fw * g.C;
  const int bn = pick_bn(g.N);
  const int s = wgrad_splits(R, g.N, M, bn);
  int mlen = (M + s - 1) / s;
  mlen = (mlen + BK - 1) / BK * BK;
  const int splits = (M + mlen - 1) / mlen;
  float *partial = scratch;
  float *bpartial = scratch + (int64_t)splits * R * g.N;
  dim3 grid((R + BM - 1) / BM, (g.N + bn - 1) / bn, splits);
  if (bn == 32)
    launch_k(wgrad_kernel<InT, 32>, grid, BM * 32 / 16, 0, st, x, dy, partial, bpartial, g, M, R, mlen);
  else
    launch_k(wgrad_kernel<InT, 64>, grid, BM * 64 / 16, 0, st, x, dy, partial, bpartial, g, M, R, mlen);
  DQN_LAUNCH_CHECK("wgrad");
  const int64_t RN = (int64_t)R * g.N;
  launch_k(wgrad_reduce_kernel, (int)std::min<int64_t>((RN + g.N + 255) / 256, 148 * 8), 256, 0, st, 
      partial, bpartial, splits, RN, g.N, grads + L.w_off, grads + L.b_off, flags);
  DQN_LAUNCH_CHECK("wgrad_reduce");
  return DQN_OK;
}

// dX = dY * W^T: linear layers write dX directly (masked); convolutions form
// dpatch[M, R] then gather it back with col2im.
int launch_dgrad(cudaStream_t st, const dqn_layer_desc &L, const float *dy, const float *params,
                 const float *mask_act, float *dx, float *scratch, int batch) {
  Geo g = geo_of(L);
  const int M = batch * g.OH * g.OW, R = g.fh * g.fw * g.C;
  // dY viewed as a 1x1 "image" of Cout channels per output pixel
  Geo a;
  a.H = a.W = a.OH = a.OW = 1;
  a.C = g.N;
  a.N = R;
  a.fh = a.fw = a.sh = a.sw = 1;
  const float *w = params + L.w_off;
  if (L.kind == DQN_LAYER_LINEAR)
    return launch_gemm<float, true>(st, dy, a, w, nullptr, mask_act, 0, dx, scratch, M, g.N);
  float *dpatch = scratch;
  int rc = launch_gemm<float, true>(st, dy, a, w, nullptr, nullptr, 0, dpatch,
                                    scratch + (int64_t)M * R, M, g.N);
  if (rc) return rc;
  const int64_t total = (int64_t)batch * g.H * g.W * g.C;
  launch_k(col2im_kernel, (int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st, 
      dpatch, g, total, mask_act, dx);
  DQN_LAUNCH_CHECK("col2im");
  return DQN_OK;
}

int validate(const dqn_net_desc *net) {
  if (!net || net->n_layers < 1 || net->n_layers > DQN_MAX_LAYERS) {
    set_error("net: bad layer count");
    return DQN_ERR_GEOMETRY;
  }
  for (int l = 0; l < net->n_layers; ++l) {
    const dqn_layer_desc &L = net->layer[l];
    if (L.kind == DQN_LAYER_DUELING && l != net->n_layers - 1) {
      set_error("net: dueling head must be last");
      return DQN_ERR_GEOMETRY;
    }
    if (is_head(net, l) && L.out_c > kMaxHeadOut - 1) {
      set_error("net: at most %d actions", kMaxHeadOut - 1);
      return DQN_ERR_UNSUPPORTED;
    }
  }
  return DQN_OK;
}

}  // namespace

int launch_splitk_reduce(cudaStream_t st, const float *partial, int splits, int64_t MN, int N,
                         const float *bias, float *y, int relu, const float *mask) {
  launch_k(splitk_bias_kernel, (int)std::min<int64_t>((MN + 255) / 256, 148 * 8), 256, 0, st, 
      partial, splits, MN, N, bias, y, relu, mask);
  DQN_LAUNCH_CHECK("splitk_reduce");
  return DQN_OK;
}

int launch_col2im(cudaStream_t st, const float *dpatch, const Geo &g, int batch,
                  const float *mask, float *dx) {
  const int64_t total = (int64_t)batch * g.H * g.W * g.C;
  launch_k(col2im_kernel, (int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st, 
      dpatch, g, total, mask, dx);
  DQN_LAUNCH_CHECK("col2im");
  return DQN_OK;
}

// Called by dqn_net_forward for layers the tcgen05 trunk does not own.
// ------------------------------------------------ small-batch forward
// Acting (select_action at batch 1, evaluate): a latency-bound forward.  One
// CTA per (output pixel, 32 output channels): lane = channel (weight rows
// W[k][n0..n0+31] load coalesced, the input element is a warp broadcast),
// the 8 warps split the reduction length, partial sums combined in warp
// order; bias + ReLU fused.  A linear layer is the full-size conv of its
// input (fh = in_h, fw = in_w), so one kernel serves both.
template <typename InT>
__global__ void __launch_bounds__(256)
small_fwd_kernel(const InT *__restrict__ x, const float *__restrict__ w,
                 const float *__restrict__ bias, float *__restrict__ y, Geo g, int relu,
                 float *__restrict__ partial) {
  // partial != nullptr: split-K over blockIdx.y (one output pixel layers);
  // the block writes its 32 partial sums, small_fwd_reduce_kernel finishes
  pdl_begin();
  __shared__ float part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ngrp = (g.N + 31) / 32;
  const int pix = blockIdx.x / ngrp, n = (blockIdx.x - pix * ngrp) * 32 + lane;
  const int P = g.OH * g.OW, img = pix / P, pp = pix - img * P;
  const int oy = pp / g.OW, ox = pp - oy * g.OW;
  const int64_t base = (((int64_t)img * g.H + (int64_t)oy * g.sh) * g.W + (int64_t)ox * g.sw) * g.C;
  const int K = g.fh * g.fw * g.C, rowlen = g.fw * g.C;
  const int kspan = (K + gridDim.y - 1) / gridDim.y;
  const int kb = blockIdx.y * kspan, ke = min(K, kb + kspan);
  const int per = (ke - kb + 7) / 8, k0 = kb + warp * per, k1 = min(ke, k0 + per);
  float a0 = 0.f, a1 = 0.f;                      // two chains, summed at the end
  int k = k0;
  for (; k + 1 < k1; k += 2) {
    const int i0 = k / rowlen, i1 = (k + 1) / rowlen;
    float x0 = (float)x[base + (int64_t)i0 * g.W * g.C + (k - i0 * rowlen)];
    float x1 = (float)x[base + (int64_t)i1 * g.W * g.C + (k + 1 - i1 * rowlen)];
    if (sizeof(InT) == 1) {
      x0 = __fdiv_rn(x0, 255.0f);
      x1 = __fdiv_rn(x1, 255.0f);
    }
    if (n < g.N) {
      a0 = fmaf(x0, __ldg(w + (int64_t)k * g.N + n), a0);
      a1 = fmaf(x1, __ldg(w + (int64_t)(k + 1) * g.N + n), a1);
    }
  }
  if (k < k1) {
    const int i0 = k / rowlen;
    float x0 = (float)x[base + (int64_t)i0 * g.W * g.C + (k - i0 * rowlen)];
    if (sizeof(InT) == 1) x0 = __fdiv_rn(x0, 255.0f);
    if (n < g.N) a0 = fmaf(x0, __ldg(w + (int64_t)k * g.N + n), a0);
  }
  part[warp][lane] = __fadd_rn(a0, a1);
  __syncthreads();
  if (warp != 0 || n >= g.N) return;
  float v = part[0][lane];
#pragma unroll
  for (int q = 1; q < 8; ++q) v = __fadd_rn(v, part[q][lane]);
  if (partial) {
    const int64_t npix = gridDim.x / ngrp;                             // [split][pix][n]
    partial[((int64_t)blockIdx.y * npix + pix) * g.N + n] = v;
    return;
  }
  v = __fadd_rn(v, bias[n]);
  if (relu && v < 0.f) v = 0.f;
  y[(int64_t)pix * g.N + n] = v;
}

// splits summed in split order, then bias + ReLU
__global__ void small_fwd_reduce_kernel(const float *__restrict__ partial, int splits,
                                        int64_t outputs, int N, const float *__restrict__ bias,
                                        float *__restrict__ y, int relu) {
  pdl_begin();
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= outputs) return;
  float v = partial[o];
  for (int s = 1; s < splits; ++s) v = __fadd_rn(v, partial[(int64_t)s * outputs + o]);
  v = __fadd_rn(v, bias[o % N]);
  if (relu && v < 0.f) v = 0.f;
  y[o] = v;
}

int small_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                        const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  const Geo g = geo_of(L);
  const int64_t blocks = (int64_t)b->batch * g.OH * g.OW * ((g.N + 31) / 32);
  const int K = g.fh * g.fw * g.C;
  // few output blocks (linear layers): split K so that about one wave runs,
  // at least 64 reduction steps per warp
  int splits = 1;
  if (blocks < kNumSMs)
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs / blocks, K / (8 * 64)));
  const int64_t outputs = (int64_t)b->batch * g.OH * g.OW * g.N;
  float *partial = nullptr;
  if (splits > 1) {
    if ((int64_t)splits * outputs > b->scratch_floats) splits = 1;
    else partial = b->scratch;
  }
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  const dim3 grid((unsigned)blocks, (unsigned)splits);
  if (l == 0 && net->input_u8)
    launch_k(small_fwd_kernel<uint8_t>, grid, 256, 0, st, (const uint8_t *)in, params + L.w_off,
             params + L.b_off, b->act[l], g, (int)L.relu, partial);
  else
    launch_k(small_fwd_kernel<float>, grid, 256, 0, st, (const float *)in, params + L.w_off,
             params + L.b_off, b->act[l], g, (int)L.relu, partial);
  DQN_LAUNCH_CHECK("small_fwd");
  if (partial) {
    launch_k(small_fwd_reduce_kernel, (unsigned)((outputs + 255) / 256), 256, 0, st, partial,
             splits, outputs, g.N, params + L.b_off, b->act[l], (int)L.relu);
    DQN_LAUNCH_CHECK("small_fwd_reduce");
  }
  return DQN_OK;
}

int simt_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                       const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  if (is_head(net, l)) {
    const int F = L.in_h * L.in_w * L.in_c;
    const bool duel = L.kind == DQN_LAYER_DUELING;
    if (l == 0 && net->input_u8) {
      set_error("head cannot read u8 input");
      return DQN_ERR_UNSUPPORTED;
    }
    launch_k(head_fwd_kernel, b->batch, kHeadThreads, 0, st, 
        (const float *)in, F, duel ? params + L.w_off : nullptr, duel ? params + L.b_off : nullptr,
        duel ? params + L.w2_off : params + L.w_off, duel ? params + L.b2_off : params + L.b_off,
        L.out_c, duel, b->act[l], flags);
    DQN_LAUNCH_CHECK("head_fwd");
    return DQN_OK;
  }
  if (l == 0 && net->input_u8)
    return launch_fwd<uint8_t>(st, L, (const uint8_t *)in, params, b->act[l], b->scratch, b->batch);
  return launch_fwd<float>(st, L, (const float *)in, params, b->act[l], b->scratch, b->batch);
}

int simt_layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                        const dqn_binding *b) {
  // produces the gradient w.r.t. layer l's INPUT: dact[l-1] (masked by the
  // ReLU fused into layer l-1) or dx for l == 0.
  const dqn_layer_desc &L = net->layer[l];
  float *out = (l == 0) ? b->dx : b->dact[l - 1];
  if (out == nullptr) return DQN_OK;
  const float *mask = (l > 0 && net->layer[l - 1].relu) ? b->act[l - 1] : nullptr;
  if (is_head(net, l)) {
    const int F = L.in_h * L.in_w * L.in_c;
    const bool duel = L.kind == DQN_LAYER_DUELING;
    const int64_t total = (int64_t)b->batch * F;
    launch_k(head_bwd_kernel, (int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, st, 
        b->dact[l], b->batch, L.out_c, duel, duel ? params + L.w_off : nullptr,
        duel ? params + L.w2_off : params + L.w_off, F, mask, out);
    DQN_LAUNCH_CHECK("head_bwd");
    return DQN_OK;
  }
  return launch_dgrad(st, L, b->dact[l], params, mask, out, b->scratch, b->batch);
}

// ------------------------------------------------ small-K linear wgrad
// dW[F][N] += X^T dY and db[N] += sum_r dY[r] for a linear layer at learner
// batch sizes (B <= 64 rows, network.py:124-126 / layers.py:157-160): an
// outer-product sum that is bandwidth-bound on dW (read-modify-write), so
// plain fp32 FMAs (exact products, sequential sum over rows) instead of a
// tensor-core GEMM with a half-empty 64-k block per CTA.  CTA = 64 features x
// 128 outputs, all B rows of both operands in shared memory, 4 x 8 outputs
// per thread; non-finite results raise DQN_FLAG_NONFINITE_GRAD.
constexpr int kLwF = 64, kLwN = 128, kLwMaxB = 64;

__global__ void __launch_bounds__(256)
lin_wgrad_smallk_kernel(const float *__restrict__ x, const float *__restrict__ dy, int B, int F,
                        int N, float *__restrict__ gw, float *__restrict__ gb, int32_t *flags) {
  pdl_begin();
  __shared__ __align__(16) float xs[kLwMaxB][kLwF];
  __shared__ __align__(16) float ys[kLwMaxB][kLwN];
  const int f0 = blockIdx.x * kLwF, n0 = blockIdx.y * kLwN, t = threadIdx.x;
  for (int i = t; i < B * kLwF; i += 256) {
    const int r = i / kLwF, c = i - r * kLwF;
    xs[r][c] = f0 + c < F ? x[(int64_t)r * F + f0 + c] : 0.f;
  }
  for (int i = t; i < B * kLwN; i += 256) {
    const int r = i / kLwN, c = i - r * kLwN;
    ys[r][c] = n0 + c < N ? dy[(int64_t)r * N + n0 + c] : 0.f;
  }
  __syncthreads();
  const int tf = (t >> 4) * 4, tn = (t & 15) * 8;     // 16 x 16 threads, 4 x 8 outputs each
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int r = 0; r < B; ++r) {
    const float4 a = *reinterpret_cast<const float4 *>(&xs[r][tf]);
    const float4 b0 = *reinterpret_cast<const float4 *>(&ys[r][tn]);
    const float4 b1 = *reinterpret_cast<const float4 *>(&ys[r][tn + 4]);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
  }
  const bool vec = (N % 4 == 0) && n0 + tn + 8 <= N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f0 + tf + i;
    if (f >= F) break;
    float *row = gw + (int64_t)f * N + n0 + tn;
    if (vec) {
      float4 *p4 = reinterpret_cast<float4 *>(row);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 v = p4[h];
        v.x = __fadd_rn(v.x, acc[i][4 * h]);
        v.y = __fadd_rn(v.y, acc[i][4 * h + 1]);
        v.z = __fadd_rn(v.z, acc[i][4 * h + 2]);
        v.w = __fadd_rn(v.w, acc[i][4 * h + 3]);
        p4[h] = v;
        note_grad4(flags, v);
      }
    } else {
      for (int j = 0; j < 8; ++j)
        if (n0 + tn + j < N) acc_grad(row + j, acc[i][j], flags);
    }
  }
  if (blockIdx.x == 0 && gb != nullptr && t < kLwN && n0 + t < N) {
    float sb = 0.f;
    for (int r = 0; r < B; ++r) sb = __fadd_rn(sb, ys[r][t]);
    acc_grad(gb + n0 + t, sb, flags);
  }
}

int lin_wgrad_smallk(cudaStream_t st, const float *x, const float *dy, int B, int F, int N,
                     float *gw, float *gb, int32_t *flags) {
  if (B < 1 || B > kLwMaxB) return DQN_ERR_UNSUPPORTED;
  dim3 grid((F + kLwF - 1) / kLwF, (N + kLwN - 1) / kLwN);
  launch_k(lin_wgrad_smallk_kernel, grid, 256, 0, st, x, dy, B, F, N, gw, gb, flags);
  DQN_LAUNCH_CHECK("lin_wgrad_smallk");
  return DQN_OK;
}


int simt_layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                     const dqn_binding *b, int32_t *flags) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  if (is_head(net, l)) {
    const int F = L.in_h * L.in_w * L.in_c;
    const bool duel = L.kind == DQN_LAYER_DUELING;
    launch_k(head_wgrad_kernel, (F + 1 + 127) / 128, 128, 0, st, 
        (const float *)in, b->dact[l], b->batch, F, L.out_c, duel,
        duel ? grads + L.w_off : nullptr, duel ? grads + L.b_off : nullptr,
        duel ? grads + L.w2_off : grads + L.w_off, duel ? grads + L.b2_off : grads + L.b_off,
        flags);
    DQN_LAUNCH_CHECK("head_wgrad");
    return DQN_OK;
  }
  if (l == 0 && net->input_u8)
    return launch_wgrad<uint8_t>(st, L, (const uint8_t *)in, b->dact[l], grads, b->scratch,
                                 b->batch, flags);
  return launch_wgrad<float>(st, L, (const float *)in, b->dact[l], grads, b->scratch, b->batch,
                             flags);
}

int64_t simt_scratch_floats(const dqn_net_desc *net, int batch) {
  int64_t m = 0;
  for (int l = 0; l < net->n_layers; ++l) {
    if (is_head(net, l)) continue;
    m = std::max(m, fwd_scratch(net->layer[l], batch));
    m = std::max(m, wgrad_scratch(net->layer[l], batch));
    m = std::max(m, dgrad_scratch(net->layer[l], batch));
  }
  return m;
}

int simt_validate(const dqn_net_desc *net) { return validate(net); }

}  // namespace dqn
