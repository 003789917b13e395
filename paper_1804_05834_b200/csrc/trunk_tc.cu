// Conv trunk on the 5th-gen tensor cores: every GEMM-shaped phase of the
// convolution / linear layers runs through the tcgen05 engine (tc_gemm.cuh)
// with implicit-GEMM operand gathers -- no im2col buffer in HBM.
//
//   forward  (layers.py:226-233, 148-150):  C[pix, co]  = im2col(x)[pix, k] * W[k, co]
//            A gathered from NHWC x (uint8 frames: exact integers, the
//            1/255 of envs.py:300-311 applied in the epilogue), B = W gathered
//            along k, epilogue bias + ReLU (or split-K partials).
//   dgrad    (layers.py:235-248, 152-155):  dpatch[pix, r] = dY[pix, co] * W[r, co]
//            (then the deterministic col2im gather), linear layers write dX
//            directly with the ReLU mask of the layer below.
//   wgrad    (layers.py:250-255, 157-160):  dW[r, co] = sum_pix im2col(x)[pix, r] * dY[pix, co]
//            reduction over pixels, split over pixels, fixed-order reduce;
//            bias grads by a fixed-order column sum.
//
// Returns DQN_ERR_UNSUPPORTED for geometries this engine does not tile
// (channel counts not multiple of 4 / 16); the caller then uses the SIMT
// kernels of net_simt.cu.
#include "tc_gemm.cuh"

#include <algorithm>

namespace dqn {

int launch_splitk_reduce(cudaStream_t st, const float *partial, int splits, int64_t MN, int N,
                         const float *bias, float *y, int relu, const float *mask);
int launch_col2im(cudaStream_t st, const float *dpatch, const Geo &g, int batch,
                  const float *mask, float *dx);

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

__device__ __forceinline__ void store4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ float4 load4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// ---------------------------------------------------------------- forward
template <typename InT, int BN_>
struct FwdPol {
  static constexpr bool U8 = sizeof(InT) == 1;
  static constexpr bool SPLIT_A = !U8, SPLIT_B = true;
  static constexpr int BN = BN_, STAGES = tc::auto_stages(BN_, SPLIT_A, SPLIT_B);
  const InT *x;
  const float *w, *bias;
  float *y, *partial;
  Geo g;
  int M, N, K, klen, relu, split;
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int m) const { return m < M ? pixel_base(g, m) : -1; }
  __device__ float4 a(long long base, int k, int ke) const {
    if (k >= ke) return zero4();
    return ld4(x + base + patch_off(g, k));
  }
  __device__ long long b_row(int n) const { return n < N ? n : -1; }
  __device__ float4 b(long long n, int k, int ke) const {     // W[k][n]: gather along k
    if (k >= ke) return zero4();
    return ld4_strided(w + (int64_t)k * N + n, N, min(4, ke - k));
  }
  __device__ void store4(int m, int n, float4 v, int z) const {
    if (split) {
      dqn::store4(partial + ((int64_t)z * M + m) * N + n, v);
      return;
    }
    float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float u = U8 ? __fdiv_rn(t[j], 255.0f) : t[j];
      u = __fadd_rn(u, bias[n + j]);
      if (relu && u < 0.f) u = 0.f;
      t[j] = u;
    }
    dqn::store4(y + (int64_t)m * N + n, make_float4(t[0], t[1], t[2], t[3]));
  }
};

// ------------------------------------------------------------------ dgrad
// C[m, n] = sum_k dY[m, k] * W[n, k]  (W row-major [R][Cout])
template <int BN_>
struct DgradPol {
  static constexpr bool SPLIT_A = true, SPLIT_B = true;
  static constexpr int BN = BN_, STAGES = tc::auto_stages(BN_, SPLIT_A, SPLIT_B);
  const float *dy, *w, *mask;
  float *out, *partial;
  int M, N, K, klen, split;
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int m) const { return m < M ? (long long)m * K : -1; }
  __device__ float4 a(long long base, int k, int ke) const {
    return k < ke ? ld4(dy + base + k) : zero4();
  }
  __device__ long long b_row(int n) const { return n < N ? (long long)n * K : -1; }
  __device__ float4 b(long long base, int k, int ke) const {
    return k < ke ? ld4(w + base + k) : zero4();
  }
  __device__ void store4(int m, int n, float4 v, int z) const {
    if (split) {
      dqn::store4(partial + ((int64_t)z * M + m) * N + n, v);
      return;
    }
    const int64_t o = (int64_t)m * N + n;
    if (mask != nullptr) {
      const float4 mk = load4(mask + o);
      v.x = mk.x > 0.f ? v.x : 0.f;
      v.y = mk.y > 0.f ? v.y : 0.f;
      v.z = mk.z > 0.f ? v.z : 0.f;
      v.w = mk.w > 0.f ? v.w : 0.f;
    }
    dqn::store4(out + o, v);
  }
};

// ------------------------------------------------------------------ wgrad
// C[r, co] = sum_pix im2col(x)[pix, r] * dY[pix, co]; the reduction runs
// over pixels, so both operands are gathered 4 pixels at a time.
template <typename InT, int BN_>
struct WgradPol {
  static constexpr bool U8 = sizeof(InT) == 1;
  static constexpr bool SPLIT_A = !U8, SPLIT_B = true;
  static constexpr int BN = BN_, STAGES = tc::auto_stages(BN_, SPLIT_A, SPLIT_B);
  const InT *x;
  const float *dy;
  float *grad, *partial;
  Geo g;
  int M, N, K, klen, split;     // M = R (patch length), N = Cout, K = pixels
  __device__ int kbeg(int z) const { return z * klen; }
  __device__ int kend(int z) const { return min(K, (z + 1) * klen); }
  __device__ long long a_row(int r) const { return r < M ? patch_off(g, r) : -1; }
  __device__ float4 a(long long roff, int pix, int ke) const {
    if (pix >= ke) return zero4();
    // window bases of 4 consecutive pixels: walk along the output row
    const int P = g.OH * g.OW;
    int img = pix / P, p = pix - img * P;
    int oy = p / g.OW, ox = p - oy * g.OW;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (pix + i < ke) {
        const long long base =
            (((long long)img * g.H + (long long)oy * g.sh) * g.W + (long long)ox * g.sw) * g.C;
        v[i] = (float)__ldg(x + base + roff);
      }
      if (++ox == g.OW) {
        ox = 0;
        if (++oy == g.OH) { oy = 0; ++img; }
      }
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ long long b_row(int n) const { return n < N ? n : -1; }
  __device__ float4 b(long long n, int pix, int ke) const {
    if (pix >= ke) return zero4();
    return ld4_strided(dy + (int64_t)pix * N + n, N, min(4, ke - pix));
  }
  __device__ void store4(int r, int n, float4 v, int z) const {
    if (split) {
      dqn::store4(partial + ((int64_t)z * M + r) * N + n, v);
      return;
    }
    float *gp = grad + (int64_t)r * N + n;
    float4 o = load4(gp);
    if (U8) {
      v.x = __fdiv_rn(v.x, 255.0f); v.y = __fdiv_rn(v.y, 255.0f);
      v.z = __fdiv_rn(v.z, 255.0f); v.w = __fdiv_rn(v.w, 255.0f);
    }
    o.x = __fadd_rn(o.x, v.x); o.y = __fadd_rn(o.y, v.y);
    o.z = __fadd_rn(o.z, v.z); o.w = __fadd_rn(o.w, v.w);
    dqn::store4(gp, o);
  }
};

// grad += scale(sum_z partial[z])  (fixed split order)
__global__ void tc_wgrad_reduce_kernel(const float *__restrict__ partial, int splits, int64_t RN,
                                       int u8, float *__restrict__ grad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < RN;
       e += (int64_t)gridDim.x * blockDim.x) {
    float s = partial[e];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, partial[(int64_t)z * RN + e]);
    if (u8) s = __fdiv_rn(s, 255.0f);
    grad[e] = __fadd_rn(grad[e], s);
  }
}

// Bias gradients: db[n] += sum_m dY[m, n].  Pass 1: 32 columns x row blocks.
constexpr int kColRowBlocks = 32;
__global__ void colsum_partial_kernel(const float *__restrict__ dy, int M, int N,
                                      float *__restrict__ part) {
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + tx;
  const int rows = (M + kColRowBlocks - 1) / kColRowBlocks;
  const int r0 = blockIdx.y * rows, r1 = min(M, r0 + rows);
  float s = 0.f;
  if (n < N)
    for (int m = r0 + ty; m < r1; m += 8) s = __fadd_rn(s, dy[(int64_t)m * N + n]);
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && n < N) {
    float t = red[0][tx];
    for (int i = 1; i < 8; ++i) t = __fadd_rn(t, red[i][tx]);
    part[(int64_t)blockIdx.y * N + n] = t;
  }
}

__global__ void colsum_final_kernel(const float *__restrict__ part, int N, float *__restrict__ db) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = part[n];
  for (int b = 1; b < kColRowBlocks; ++b) s = __fadd_rn(s, part[(int64_t)b * N + n]);
  db[n] = __fadd_rn(db[n], s);
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------------------ host helpers
bool conv_ok(const dqn_layer_desc &L) {
  if (L.kind == DQN_LAYER_DUELING) return false;
  return L.in_c % 4 == 0 && (L.fw * L.in_c) % 4 == 0 && L.out_c % 16 == 0;
}

// forward split length: a function of K only (batch-independent rows)
inline int fwd_klen(int K) {
  if (K >= 2048) return 128;
  if (K >= 512) return 192;
  return K;
}

template <typename InT, int BN>
int fwd_launch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *params,
               float *y, float *scratch, int batch) {
  FwdPol<InT, BN> p;
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
  const int splits = ceil_div(p.K, p.klen);
  p.split = splits > 1;
  p.relu = L.relu;
  int rc = tc::launch(st, p, splits, "tc_fwd");
  if (rc || splits == 1) return rc;
  if (FwdPol<InT, BN>::U8) {
    set_error("tc_fwd: split-K with uint8 input is not supported");
    return DQN_ERR_UNSUPPORTED;
  }
  return launch_splitk_reduce(st, scratch, splits, (int64_t)p.M * p.N, p.N, p.bias, y, L.relu,
                              nullptr);
}

template <typename InT>
int fwd_dispatch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *params,
                 float *y, float *scratch, int batch) {
  const int N = L.out_c;
  if (N == 32) return fwd_launch<InT, 32>(st, L, x, params, y, scratch, batch);
  if (N == 64) return fwd_launch<InT, 64>(st, L, x, params, y, scratch, batch);
  if (N % 128 == 0) return fwd_launch<InT, 128>(st, L, x, params, y, scratch, batch);
  return DQN_ERR_UNSUPPORTED;
}

template <int BN>
int dgrad_gemm(cudaStream_t st, const float *dy, const float *w, const float *mask, float *out,
               float *partial, int M, int N, int K, int klen) {
  DgradPol<BN> p;
  p.dy = dy;
  p.w = w;
  p.mask = mask;
  p.out = out;
  p.partial = partial;
  p.M = M;
  p.N = N;
  p.K = K;
  p.klen = klen;
  const int splits = ceil_div(K, klen);
  p.split = splits > 1;
  int rc = tc::launch(st, p, splits, "tc_dgrad");
  if (rc || splits == 1) return rc;
  return launch_splitk_reduce(st, partial, splits, (int64_t)M * N, N, nullptr, out, 0, mask);
}

int dgrad_pick(cudaStream_t st, const float *dy, const float *w, const float *mask, float *out,
               float *partial, int M, int N, int K, int klen) {
  // widest tile <= 128 columns that divides N (N % 16 == 0 is guaranteed)
  for (int bn : {128, 112, 96, 64, 32, 16}) {
    if (N % bn) continue;
    switch (bn) {
      case 112: return dgrad_gemm<112>(st, dy, w, mask, out, partial, M, N, K, klen);
      case 128: return dgrad_gemm<128>(st, dy, w, mask, out, partial, M, N, K, klen);
      case 96: return dgrad_gemm<96>(st, dy, w, mask, out, partial, M, N, K, klen);
      case 64: return dgrad_gemm<64>(st, dy, w, mask, out, partial, M, N, K, klen);
      case 32: return dgrad_gemm<32>(st, dy, w, mask, out, partial, M, N, K, klen);
      default: return dgrad_gemm<16>(st, dy, w, mask, out, partial, M, N, K, klen);
    }
  }
  return DQN_ERR_UNSUPPORTED;
}

template <typename InT, int BN>
int wgrad_launch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *dy,
                 float *grads, float *scratch, int batch) {
  WgradPol<InT, BN> p;
  p.x = x;
  p.dy = dy;
  p.grad = grads + L.w_off;
  p.partial = scratch;
  p.g = geo_of(L);
  p.M = L.fh * L.fw * L.in_c;
  p.N = L.out_c;
  p.K = batch * L.out_h * L.out_w;
  // ~2 CTA waves over the machine, split lengths a multiple of BK
  const int tiles = ceil_div(p.M, tc::BM) * ceil_div(p.N, BN);
  int splits = std::max(1, std::min(ceil_div(2 * kNumSMs, tiles), ceil_div(p.K, 4 * tc::BK)));
  p.klen = ceil_div(ceil_div(p.K, splits), tc::BK) * tc::BK;
  splits = ceil_div(p.K, p.klen);
  p.split = splits > 1;
  int rc = tc::launch(st, p, splits, "tc_wgrad");
  if (rc) return rc;
  float *bpart = scratch + (p.split ? (int64_t)splits * p.M * p.N : 0);
  if (p.split) {
    const int64_t RN = (int64_t)p.M * p.N;
    tc_wgrad_reduce_kernel<<<(int)std::min<int64_t>((RN + 255) / 256, 148 * 8), 256, 0, st>>>(
        scratch, splits, RN, WgradPol<InT, BN>::U8 ? 1 : 0, p.grad);
    DQN_LAUNCH_CHECK("tc_wgrad_reduce");
  }
  colsum_partial_kernel<<<dim3(ceil_div(p.N, 32), kColRowBlocks), 256, 0, st>>>(dy, p.K, p.N, bpart);
  DQN_LAUNCH_CHECK("colsum_partial");
  colsum_final_kernel<<<ceil_div(p.N, 128), 128, 0, st>>>(bpart, p.N, grads + L.b_off);
  DQN_LAUNCH_CHECK("colsum_final");
  return DQN_OK;
}

template <typename InT>
int wgrad_dispatch(cudaStream_t st, const dqn_layer_desc &L, const InT *x, const float *dy,
                   float *grads, float *scratch, int batch) {
  const int N = L.out_c;
  if (N == 32) return wgrad_launch<InT, 32>(st, L, x, dy, grads, scratch, batch);
  if (N == 64) return wgrad_launch<InT, 64>(st, L, x, dy, grads, scratch, batch);
  if (N % 128 == 0) return wgrad_launch<InT, 128>(st, L, x, dy, grads, scratch, batch);
  return DQN_ERR_UNSUPPORTED;
}

int64_t wgrad_scratch_tc(const dqn_layer_desc &L, int batch) {
  const int M = L.fh * L.fw * L.in_c, N = L.out_c, K = batch * L.out_h * L.out_w;
  const int bn = N == 32 ? 32 : N == 64 ? 64 : 128;
  const int tiles = ceil_div(M, tc::BM) * ceil_div(N, bn);
  int splits = std::max(1, std::min(ceil_div(2 * kNumSMs, tiles), ceil_div(K, 4 * tc::BK)));
  const int klen = ceil_div(ceil_div(K, splits), tc::BK) * tc::BK;
  splits = ceil_div(K, klen);
  return (splits > 1 ? (int64_t)splits * M * N : 0) + (int64_t)kColRowBlocks * N;
}

}  // namespace

bool tc_layer_supported(const dqn_net_desc *net, int l) {
  const dqn_layer_desc &L = net->layer[l];
  if (!conv_ok(L)) return false;
  if (L.kind == DQN_LAYER_LINEAR && l == net->n_layers - 1 && L.out_c <= 32) return false;  // head
  const int N = L.out_c;
  if (!(N == 32 || N == 64 || N % 128 == 0)) return false;
  if (l == 0 && net->input_u8 && fwd_klen(L.fh * L.fw * L.in_c) < L.fh * L.fw * L.in_c)
    return false;
  return true;
}

int64_t tc_scratch_floats(const dqn_net_desc *net, int batch) {
  int64_t m = 0;
  for (int l = 0; l < net->n_layers; ++l) {
    if (!tc_layer_supported(net, l)) continue;
    const dqn_layer_desc &L = net->layer[l];
    const int M = batch * L.out_h * L.out_w, R = L.fh * L.fw * L.in_c, K = R;
    const int kl = fwd_klen(K);
    const int fs = ceil_div(K, kl);
    m = std::max(m, fs > 1 ? (int64_t)fs * M * L.out_c : 0);
    // dgrad: dpatch (conv) or split partials (linear, klen 128 over Cout)
    const int ds = ceil_div(L.out_c, 128);
    int64_t d = (L.kind == DQN_LAYER_CONV ? (int64_t)M * R : 0) + (ds > 1 ? (int64_t)ds * M * R : 0);
    m = std::max(m, d);
    m = std::max(m, wgrad_scratch_tc(L, batch));
  }
  return m;
}

int tc_layer_forward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                     const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  if (l == 0 && net->input_u8)
    return fwd_dispatch<uint8_t>(st, L, (const uint8_t *)in, params, b->act[l], b->scratch, b->batch);
  return fwd_dispatch<float>(st, L, (const float *)in, params, b->act[l], b->scratch, b->batch);
}

int tc_layer_backward(cudaStream_t st, const dqn_net_desc *net, int l, const float *params,
                      const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  float *out = (l == 0) ? b->dx : b->dact[l - 1];
  if (out == nullptr) return DQN_OK;
  const float *mask = (l > 0 && net->layer[l - 1].relu) ? b->act[l - 1] : nullptr;
  const int M = b->batch * L.out_h * L.out_w, R = L.fh * L.fw * L.in_c, K = L.out_c;
  const float *w = params + L.w_off;
  if (L.kind == DQN_LAYER_LINEAR)
    return dgrad_pick(st, b->dact[l], w, mask, out, b->scratch, M, R, K, std::min(K, 128));
  float *dpatch = b->scratch;
  int rc = dgrad_pick(st, b->dact[l], w, nullptr, dpatch, b->scratch + (int64_t)M * R, M, R, K,
                      std::min(K, 128));
  if (rc) return rc;
  return launch_col2im(st, dpatch, geo_of(L), b->batch, mask, out);
}

int tc_layer_wgrad(cudaStream_t st, const dqn_net_desc *net, int l, float *grads,
                   const dqn_binding *b) {
  const dqn_layer_desc &L = net->layer[l];
  const void *in = (l == 0) ? b->x : b->act[l - 1];
  if (l == 0 && net->input_u8)
    return wgrad_dispatch<uint8_t>(st, L, (const uint8_t *)in, b->dact[l], grads, b->scratch, b->batch);
  return wgrad_dispatch<float>(st, L, (const float *)in, b->dact[l], grads, b->scratch, b->batch);
}

}  // namespace dqn

