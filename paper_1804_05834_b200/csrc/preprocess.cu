// Frame preprocessing: the reference's
// preprocess_frame (envs.py:264-311) for batches of raw 8-bit emulator frames,
// bit-exact.  Per output pixel, in fp64 with every operation individually
// rounded (explicit __dmul_rn / __dadd_rn: no FMA contraction), in numpy's
// order:
//   v      = u8 / 255.0                                  (per channel)
//   gray   = (0.299 * R + 0.587 * G) + 0.114 * B          (3-channel input)
//   ys     = clip((i + 0.5) * (H / out_h) - 0.5, 0, H - 1) ; y0 = floor, y1 = min(y0 + 1, H - 1)
//   rows   = gray[y0, x] * (1 - fy) + gray[y1, x] * fy     (fy = ys - y0)
//   out    = f32(rows[x0] * (1 - fx) + rows[x1] * fx)
// Identity size returns f32(gray).  The per-channel terms w_c * (k / 255.0)
// come from exact 256-entry shared-memory tables (no fp64 divides in the
// loop); one thread per output pixel, the 2x2 source taps (x 3 channels) are
// L1/L2 hits shared by neighbouring threads.
#include "common.cuh"

namespace dqn {
namespace {

struct Taps {
  int lo, hi;
  double f;
};

__device__ __forceinline__ Taps axis_taps(int o, int n_in, double scale) {
  double p = __dadd_rn(__dmul_rn(__dadd_rn((double)o, 0.5), scale), -0.5);
  p = fmin(fmax(p, 0.0), (double)(n_in - 1));
  Taps t;
  t.lo = (int)floor(p);
  t.hi = min(t.lo + 1, n_in - 1);
  t.f = __dadd_rn(p, -(double)t.lo);
  return t;
}

// A byte has 256 values, so the per-channel terms are exact table lookups:
// lut[0][k] = k / 255.0 (gray input), lut[1..3][k] = w_c * (k / 255.0).
struct Luts {
  double v[4][256];
};

__device__ __forceinline__ double gray_at(const uint8_t *__restrict__ img, int w, int c, int y,
                                          int x, const Luts &L) {
  const uint8_t *px = img + ((int64_t)y * w + x) * c;
  if (c == 1) return L.v[0][px[0]];
  return __dadd_rn(__dadd_rn(L.v[1][px[0]], L.v[2][px[1]]), L.v[3][px[2]]);
}

__global__ void __launch_bounds__(256) preprocess_kernel(
    const uint8_t *__restrict__ frames, int64_t n, int h, int w, int c, int oh, int ow,
    float *__restrict__ out, int64_t frame_stride, int64_t pix_stride) {
  __shared__ Luts L;
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    const double v = __ddiv_rn((double)k, 255.0);
    L.v[0][k] = v;
    L.v[1][k] = __dmul_rn(0.299, v);
    L.v[2][k] = __dmul_rn(0.587, v);
    L.v[3][k] = __dmul_rn(0.114, v);
  }
  __syncthreads();
  pdl_begin();
  const int64_t per = (int64_t)oh * ow;
  const int64_t total = n * per;
  const bool ident = (h == oh && w == ow);
  const double sy = __ddiv_rn((double)h, (double)oh), sx = __ddiv_rn((double)w, (double)ow);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / per;
    const int rem = (int)(t - f * per);
    const int i = rem / ow, j = rem - (rem / ow) * ow;
    const uint8_t *img = frames + f * (int64_t)h * w * c;
    double v;
    if (ident) {
      v = gray_at(img, w, c, i, j, L);
    } else {
      const Taps ty = axis_taps(i, h, sy), tx = axis_taps(j, w, sx);
      const double wy0 = __dadd_rn(1.0, -ty.f), wx0 = __dadd_rn(1.0, -tx.f);
      const double r0 = __dadd_rn(__dmul_rn(gray_at(img, w, c, ty.lo, tx.lo, L), wy0),
                                  __dmul_rn(gray_at(img, w, c, ty.hi, tx.lo, L), ty.f));
      const double r1 = __dadd_rn(__dmul_rn(gray_at(img, w, c, ty.lo, tx.hi, L), wy0),
                                  __dmul_rn(gray_at(img, w, c, ty.hi, tx.hi, L), ty.f));
      v = __dadd_rn(__dmul_rn(r0, wx0), __dmul_rn(r1, tx.f));
    }
    out[f * frame_stride + (int64_t)rem * pix_stride] = __double2float_rn(v);
  }
}

}  // namespace
}  // namespace dqn

using namespace dqn;

extern "C" int dqn_preprocess_frames(void *stream, const uint8_t *frames, int64_t n, int h, int w,
                                     int c, int out_h, int out_w, float *out,
                                     int64_t frame_stride, int64_t pix_stride) {
  DQN_CHECK_ARG(n >= 0 && h >= 1 && w >= 1 && out_h >= 1 && out_w >= 1 && (c == 1 || c == 3),
                "preprocess_frames: bad geometry");
  DQN_CHECK_ARG(n == 0 || (frames && out), "preprocess_frames: null pointer");
  DQN_CHECK_ARG(pix_stride >= 1 && (n <= 1 || frame_stride >= (int64_t)out_h * out_w * pix_stride -
                                                                    (pix_stride - 1)),
                "preprocess_frames: overlapping output strides");
  if (n == 0) return DQN_OK;
  const int64_t total = n * (int64_t)out_h * out_w;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = (int)(want < kNumSMs * 16 ? want : kNumSMs * 16);
  launch_k(preprocess_kernel, blocks, threads, 0, as_stream(stream), frames, n, h, w, c, out_h,
           out_w, out, frame_stride, pix_stride);
  DQN_LAUNCH_CHECK("preprocess_frames");
  return DQN_OK;
}
