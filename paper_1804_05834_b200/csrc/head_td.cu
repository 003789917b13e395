// Fused learner head: both networks' Q heads, the Double-DQN TD block, the
// head backward and the head weight gradient in two launches.
//
//   online/target head forward    layers.py:302-310 (dueling) / 148-150   K1
//   targets, TD error, loss, dq   agent.py:58-73, 110-124 (td_row.cuh)    K1 (last CTA)
//   head backward (dX, ReLU mask) layers.py:312-323                       K2
//   head wgrad (dWv, dbv, dWa, dba) layers.py:325-330                     K2
//
// As separate kernels the head is five dependent launches (head fwd x2, TD,
// head bwd, head wgrad) on the critical path of the update.  The TD block,
// head backward and wgrad keep exactly the arithmetic and order of
// td_loss_kernel, head_bwd_kernel and head_wgrad_kernel; the Q heads reduce
// each output over a warp (lane-strided fmaf chains, fixed shuffle tree).
// The action count is a template parameter (1..18): no predicated work.
#include "common.cuh"
#include "td_row.cuh"

namespace dqn {
namespace {

constexpr int kHeadCta = 256;           // 8 warps: 8 Q rows per CTA (K1); 256 outputs (K2)
constexpr int kFusedMaxA = 18;          // Atari's largest action set
constexpr int kFusedMaxRows = 1024;     // learner batch k

struct HeadNet {
  const float *x;          // [rows][F] head input (post-ReLU features)
  const float *wv, *bv;    // dueling value branch (nullptr for a plain head)
  const float *wa, *ba;    // [F][nA] advantage / plain weights, [nA] bias
  float *q;                // [rows][nA] head output
  int rows;
};

struct HeadTdArgs {
  HeadNet on, tg;          // on.rows = k (single) or 2k ([s; s'] for Double DQN)
  int F, dueling, k;
  const int64_t *actions;
  const double *rewards;
  const uint8_t *terminals;
  const double *weights;
  double gamma;
  int td_flags;
  double *targets, *td, *losses, *stats;
  float *dq;               // [k][nA] online dact of the head
  float *dx;               // [k][F] gradient w.r.t. the head input (nullptr: skip)
  const float *mask;       // ReLU mask of the head input (online rows < k) or nullptr
  float *gwv, *gbv, *gwa, *gba;
  float *gs;               // work: [k][nA + 1] branch gradients (gv, ga) or g
  int *ticket;             // work: CTA arrival counter (0 at rest)
  int32_t *flags;
  double *host_out;        // optional pinned host copy: targets | td | losses | stats
};

// td_flags & DQN_TD_HEAD_LAST_CTA selects the last-CTA form (head_q_td +
// head_bwd_wgrad) instead of the two-phase form -- an explicit argument, so a
// captured graph's form is fixed by its caller, not by the environment
inline bool head_two_phase(int td_flags) { return !(td_flags & DQN_TD_HEAD_LAST_CTA); }

// Head weight-gradient epilogue: grads[f][o] += s[o] for the NO outputs of
// feature f (f == F: the bias row).  Every old value is read before the first
// write: a read-add-write per output would chain NO L2 round trips.
template <int NA>
__device__ __forceinline__ void head_acc_grads(const HeadTdArgs &p, int f, const float (&s)[NA + 1]) {
  constexpr int NO = NA + 1;
  const int F = p.F, no = p.dueling ? NO : NA;
  float *gp[NO];
  float old[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (p.dueling)
      gp[o] = o == 0 ? (f < F ? &p.gwv[f] : &p.gbv[0])
                     : (f < F ? &p.gwa[(int64_t)f * NA + o - 1] : &p.gba[o - 1]);
    else
      gp[o] = f < F ? &p.gwa[(int64_t)f * NA + o] : &p.gba[o];
    old[o] = o < no ? *gp[o] : 0.f;
  }
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (o >= no) break;
    const float v = __fadd_rn(old[o], s[o]);
    *gp[o] = v;
    note_grad(p.flags, v);
  }
}

// K1: Q heads of both networks (one warp per row: lane-strided fmaf chains,
// fixed shuffle tree read from lane 0), then -- in the last CTA to finish --
// the TD block (td_loss_kernel's per-row arithmetic and 256-slot statistics
// tree) and the per-row branch gradients for K2.
template <int NA>
__global__ void __launch_bounds__(kHeadCta) head_q_td_kernel(const HeadTdArgs p) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  constexpr int NO = NA + 1;                    // outputs incl. the value branch
  const int F = p.F, k = p.k, R = p.on.rows + p.tg.rows;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  __shared__ int s_last;
  __shared__ double s_abs[kHeadCta], s_loss[kHeadCta];
  const int r = blockIdx.x * (kHeadCta / 32) + warp;
  if (r < R) {
    const bool on = r < p.on.rows;
    const int row = on ? r : r - p.on.rows;
    const float *xr = (on ? p.on.x : p.tg.x) + (int64_t)row * F;
    const float *wv = on ? p.on.wv : p.tg.wv, *wa = on ? p.on.wa : p.tg.wa;
    const float *bv = on ? p.on.bv : p.tg.bv, *ba = on ? p.on.ba : p.tg.ba;
    float acc[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) acc[o] = 0.f;
#pragma unroll 4
    for (int f = lane; f < F; f += 32) {
      const float xv = __ldg(xr + f);
      if (p.dueling) acc[NA] = fmaf(xv, __ldg(wv + f), acc[NA]);
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = fmaf(xv, __ldg(wa + (int64_t)f * NA + a), acc[a]);
    }
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) acc[o] = __fadd_rn(acc[o], __shfl_down_sync(0xffffffffu, acc[o], s));
    if (lane == 0) {
      bool bad = false;
      float *qr = (on ? p.on.q : p.tg.q) + (int64_t)row * NA;
      if (p.dueling) {
        // layers.py:302-310: y = V; y += A; y -= mean(A)
        const float v = __fadd_rn(acc[NA], bv[0]);
        float adv[NA], sum = 0.f;
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          adv[a] = __fadd_rn(acc[a], ba[a]);
          sum = __fadd_rn(sum, adv[a]);
        }
        const float mean = __fdiv_rn(sum, (float)NA);
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          const float qa = __fsub_rn(__fadd_rn(v, adv[a]), mean);
          bad |= !isfinite(qa);
          qr[a] = qa;
        }
      } else {
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          const float qa = __fadd_rn(acc[a], ba[a]);
          bad |= !isfinite(qa);
          qr[a] = qa;
        }
      }
      if (bad) raise_flag(p.flags, DQN_FLAG_NONFINITE_OUT);
    }
  }
  // last CTA to finish its rows runs the TD block over all of them
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(p.ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float *q_on = p.on.q;                                     // online rows [0, k)
  const float *q_next_on = p.on.q + (int64_t)k * NA;              // online rows [k, 2k)
  double acc_abs = 0.0, acc_loss = 0.0;
  for (int j = t; j < k; j += kHeadCta) {
    double ad, l;
    td_row(j, q_on, q_next_on, p.tg.q, p.actions, p.rewards, p.terminals, p.weights, NA,
           p.gamma, p.td_flags, p.targets, p.td, p.losses, p.dq, ad, l);
    acc_abs = __dadd_rn(acc_abs, ad);
    acc_loss = __dadd_rn(acc_loss, l);
    // branch gradients of row j (head_bwd_kernel / head_wgrad_kernel formulas)
    const float *g = p.dq + (int64_t)j * NA;
    float *gs = p.gs + (int64_t)j * NO;
    if (p.dueling) {
      float gv = 0.f;
      for (int a = 0; a < NA; ++a) gv = __fadd_rn(gv, g[a]);
      gs[0] = gv;
      const float gvn = __fdiv_rn(gv, (float)NA);
      for (int a = 0; a < NA; ++a) gs[a + 1] = __fsub_rn(g[a], gvn);
    } else {
      for (int a = 0; a < NA; ++a) gs[a] = g[a];
    }
  }
  s_abs[t] = acc_abs;
  s_loss[t] = acc_loss;
  __syncthreads();
  for (int s = kHeadCta / 2; s > 0; s >>= 1) {
    if (t < s) {
      s_abs[t] = __dadd_rn(s_abs[t], s_abs[t + s]);
      s_loss[t] = __dadd_rn(s_loss[t], s_loss[t + s]);
    }
    __syncthreads();
  }
  if (t == 0) {
    if (p.stats) {
      p.stats[0] = s_abs[0];
      p.stats[1] = s_loss[0];
    }
    *p.ticket = 0;                            // reusable by the next launch
  }
}

// K2: head backward (CTAs [0, nb_dx)) and head wgrad (the rest: one input
// feature per thread, feature F = the bias row, rows in order).
template <int NA>
__global__ void __launch_bounds__(kHeadCta) head_bwd_wgrad_kernel(const HeadTdArgs p, int nb_dx) {
  pdl_begin();   // programmatic dependent launch (common.cuh)
  constexpr int NO = NA + 1;
  const int F = p.F, k = p.k;
  const int no = p.dueling ? NA + 1 : NA;
  if ((int)blockIdx.x < nb_dx) {
    const int e = blockIdx.x * kHeadCta + threadIdx.x;
    if (e >= k * F) return;
    const int row = e / F, f = e - row * F;
    const float *gs = p.gs + (int64_t)row * NO;
    float v;
    if (p.dueling) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < NA; ++a) s = fmaf(gs[a + 1], __ldg(p.on.wa + (int64_t)f * NA + a), s);
      v = __fadd_rn(__fmul_rn(gs[0], __ldg(p.on.wv + f)), s);
    } else {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < NA; ++a) s = fmaf(gs[a], __ldg(p.on.wa + (int64_t)f * NA + a), s);
      v = s;
    }
    if (p.mask != nullptr && !(p.mask[e] > 0.f)) v = 0.f;
    p.dx[e] = v;
    return;
  }
  const int f = (blockIdx.x - nb_dx) * kHeadCta + threadIdx.x;
  if (f > F) return;
  float acc[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) acc[o] = 0.f;
#pragma unroll 8
  for (int r = 0; r < k; ++r) {
    const float xv = f < F ? __ldg(p.on.x + (int64_t)r * F + f) : 1.f;
    const float *gs = p.gs + (int64_t)r * NO;
#pragma unroll
    for (int o = 0; o < NO; ++o)
      if (o < no) acc[o] = fmaf(xv, gs[o], acc[o]);
  }
  head_acc_grads<NA>(p, f, acc);
}

// ---- two-phase form for learner batches (k * (nA + 1) <= kGsMax) ----------
// K1q: the Q heads only (CTA per row, features split over 8 warps).
// K2t: every CTA recomputes the k-row TD block into shared memory (a few
// hundred L2 bytes and fp64 ops per row), so no CTA waits on a last-arrival
// ticket; CTA 0 alone stores targets / TD / losses / dq / statistics; then
// head dX (first nb_dx CTAs) and head wgrad (the rest, 32-feature x 8-row-
// group tiles).  Same formulas as head_q_td + head_bwd_wgrad; the Q-head and
// wgrad sums run in a different fixed order (not bit-identical to that form).
constexpr int kGsMax = 2048;

template <int NA>
__global__ void __launch_bounds__(kHeadCta) head_q_kernel(const HeadTdArgs p) {
  // one CTA per Q row; warp w owns features [w F/8, (w+1) F/8) (lane-strided,
  // every load of the row in flight at once); partial sums of the 8 warps are
  // added in warp order
  pdl_begin();
  constexpr int NO = NA + 1, NW = kHeadCta / 32;
  __shared__ float s_part[NW][NO];
  const int F = p.F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x;
  const bool on = r < p.on.rows;
  const int row = on ? r : r - p.on.rows;
  const float *xr = (on ? p.on.x : p.tg.x) + (int64_t)row * F;
  const float *wv = on ? p.on.wv : p.tg.wv, *wa = on ? p.on.wa : p.tg.wa;
  const float *bv = on ? p.on.bv : p.tg.bv, *ba = on ? p.on.ba : p.tg.ba;
  const int per = (F + NW - 1) / NW, f0 = warp * per, f1 = min(F, f0 + per);
  float acc[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) acc[o] = 0.f;
#pragma unroll 4
  for (int f = f0 + lane; f < f1; f += 32) {
    const float xv = __ldg(xr + f);
    if (p.dueling) acc[NA] = fmaf(xv, __ldg(wv + f), acc[NA]);
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = fmaf(xv, __ldg(wa + (int64_t)f * NA + a), acc[a]);
  }
#pragma unroll
  for (int o = 0; o < NO; ++o) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc[o] = __fadd_rn(acc[o], __shfl_down_sync(0xffffffffu, acc[o], s));
    if (lane == 0) s_part[warp][o] = acc[o];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    float v = s_part[0][o];
    for (int w = 1; w < NW; ++w) v = __fadd_rn(v, s_part[w][o]);
    acc[o] = v;
  }
  bool bad = false;
  float *qr = (on ? p.on.q : p.tg.q) + (int64_t)row * NA;
  if (p.dueling) {
    const float v = __fadd_rn(acc[NA], bv[0]);
    float adv[NA], sum = 0.f;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      adv[a] = __fadd_rn(acc[a], ba[a]);
      sum = __fadd_rn(sum, adv[a]);
    }
    const float mean = __fdiv_rn(sum, (float)NA);
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const float qa = __fsub_rn(__fadd_rn(v, adv[a]), mean);
      bad |= !isfinite(qa);
      qr[a] = qa;
    }
  } else {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const float qa = __fadd_rn(acc[a], ba[a]);
      bad |= !isfinite(qa);
      qr[a] = qa;
    }
  }
  if (bad) raise_flag(p.flags, DQN_FLAG_NONFINITE_OUT);
}

template <int NA>
__global__ void __launch_bounds__(kHeadCta) head_td_bwd_kernel(const HeadTdArgs p, int nb_dx) {
  pdl_begin();
  constexpr int NO = NA + 1;
  const int F = p.F, k = p.k, t = threadIdx.x;
  const int no = p.dueling ? NA + 1 : NA;
  __shared__ float s_gs[kGsMax];
  __shared__ double s_abs[kHeadCta], s_loss[kHeadCta];
  const bool writer = blockIdx.x == 0;
  const float *q_on = p.on.q, *q_next_on = p.on.q + (int64_t)k * NA;
  double acc_abs = 0.0, acc_loss = 0.0;
  for (int j = t; j < k; j += kHeadCta) {
    int64_t a;
    double y, d, loss;
    float gf;
    td_core(j, q_on, q_next_on, p.tg.q, p.actions, p.rewards, p.terminals, p.weights, NA,
            p.gamma, p.td_flags, a, y, d, loss, gf);
    // dq row j is gf at the taken action, 0 elsewhere; branch gradients as
    // head_q_td_kernel derives them from that row (sums in the same order)
    float *gs = s_gs + j * NO;
    if (p.dueling) {
      float gv = 0.f;
      for (int c = 0; c < NA; ++c) gv = __fadd_rn(gv, c == a ? gf : 0.f);
      gs[0] = gv;
      const float gvn = __fdiv_rn(gv, (float)NA);
      for (int c = 0; c < NA; ++c) gs[c + 1] = __fsub_rn(c == a ? gf : 0.f, gvn);
    } else {
      for (int c = 0; c < NA; ++c) gs[c] = c == a ? gf : 0.f;
    }
    if (writer) {
      p.targets[j] = y;
      p.td[j] = d;
      p.losses[j] = loss;
      if (p.host_out) {
        p.host_out[j] = y;
        p.host_out[k + j] = d;
        p.host_out[2 * k + j] = loss;
      }
      for (int c = 0; c < NA; ++c) p.dq[(int64_t)j * NA + c] = (c == a) ? gf : 0.f;
      acc_abs = __dadd_rn(acc_abs, fabs(d));
      acc_loss = __dadd_rn(acc_loss, loss);
    }
  }
  __syncthreads();
  if (writer && p.stats) {
    s_abs[t] = acc_abs;
    s_loss[t] = acc_loss;
    __syncthreads();
    for (int s = kHeadCta / 2; s > 0; s >>= 1) {
      if (t < s) {
        s_abs[t] = __dadd_rn(s_abs[t], s_abs[t + s]);
        s_loss[t] = __dadd_rn(s_loss[t], s_loss[t + s]);
      }
      __syncthreads();
    }
    if (t == 0) {
      p.stats[0] = s_abs[0];
      p.stats[1] = s_loss[0];
      if (p.host_out) {
        p.host_out[3 * k] = s_abs[0];
        p.host_out[3 * k + 1] = s_loss[0];
      }
    }
  }
  if (writer && p.host_out) __threadfence_system();     // before any later completion signal
  if ((int)blockIdx.x < nb_dx) {
    const int e = blockIdx.x * kHeadCta + t;
    if (e >= k * F) return;
    const int row = e / F, f = e - row * F;
    const float *gs = s_gs + row * NO;
    float v;
    if (p.dueling) {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < NA; ++a) s = fmaf(gs[a + 1], __ldg(p.on.wa + (int64_t)f * NA + a), s);
      v = __fadd_rn(__fmul_rn(gs[0], __ldg(p.on.wv + f)), s);
    } else {
      float s = 0.f;
#pragma unroll
      for (int a = 0; a < NA; ++a) s = fmaf(gs[a], __ldg(p.on.wa + (int64_t)f * NA + a), s);
      v = s;
    }
    if (p.mask != nullptr && !(p.mask[e] > 0.f)) v = 0.f;
    p.dx[e] = v;
    return;
  }
  // head wgrad: CTA = 32 features (f = F is the bias row) x 8 row groups;
  // each thread sums its rows (all loads in flight), the 8 group partials are
  // added in group order
  __shared__ float s_w[kHeadCta / 32][32][NO];
  const int fl = t & 31, rg = t >> 5;
  const int f = (blockIdx.x - nb_dx) * 32 + fl;
  const int rows_per = (k + 7) / 8, r0 = rg * rows_per, r1 = min(k, r0 + rows_per);
  float acc[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) acc[o] = 0.f;
  if (f <= F) {
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
      const float xv = f < F ? __ldg(p.on.x + (int64_t)r * F + f) : 1.f;
      const float *gs = s_gs + r * NO;
#pragma unroll
      for (int o = 0; o < NO; ++o)
        if (o < no) acc[o] = fmaf(xv, gs[o], acc[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < NO; ++o) s_w[rg][fl][o] = acc[o];
  __syncthreads();
  if (rg != 0 || f > F) return;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    acc[o] = s_w[0][fl][o];
    for (int g = 1; g < kHeadCta / 32; ++g) acc[o] = __fadd_rn(acc[o], s_w[g][fl][o]);
  }
  head_acc_grads<NA>(p, f, acc);
}

template <int NA>
int launch_head_td(cudaStream_t st, const HeadTdArgs &p) {
  const int R = p.on.rows + p.tg.rows;
  const int nb_dx = p.dx ? (p.k * p.F + kHeadCta - 1) / kHeadCta : 0;
  const int nb_w = (p.F + 1 + kHeadCta - 1) / kHeadCta;
  if (p.host_out && !(p.k * (NA + 1) <= kGsMax && head_two_phase(p.td_flags))) {
    set_error("head_td: host_out needs the two-phase form (batch * (nA + 1) <= %d)", kGsMax);
    return DQN_ERR_UNSUPPORTED;
  }
  if (p.k * (NA + 1) <= kGsMax && head_two_phase(p.td_flags)) {
    launch_k(head_q_kernel<NA>, R, kHeadCta, 0, st, p);
    DQN_LAUNCH_CHECK("head_q");
    launch_k(head_td_bwd_kernel<NA>, nb_dx + (p.F + 1 + 31) / 32, kHeadCta, 0, st, p, nb_dx);
    DQN_LAUNCH_CHECK("head_td_bwd");
    return DQN_OK;
  }
  launch_k(head_q_td_kernel<NA>, (R + kHeadCta / 32 - 1) / (kHeadCta / 32), kHeadCta, 0, st, p);
  DQN_LAUNCH_CHECK("head_q_td");
  launch_k(head_bwd_wgrad_kernel<NA>, nb_dx + nb_w, kHeadCta, 0, st, p, nb_dx);
  DQN_LAUNCH_CHECK("head_bwd_wgrad");
  return DQN_OK;
}

int dispatch_head_td(cudaStream_t st, int nA, const HeadTdArgs &p) {
  switch (nA) {
#define DQN_HEAD_CASE(n) \
  case n: return launch_head_td<n>(st, p);
    DQN_HEAD_CASE(1) DQN_HEAD_CASE(2) DQN_HEAD_CASE(3) DQN_HEAD_CASE(4) DQN_HEAD_CASE(5)
    DQN_HEAD_CASE(6) DQN_HEAD_CASE(7) DQN_HEAD_CASE(8) DQN_HEAD_CASE(9) DQN_HEAD_CASE(10)
    DQN_HEAD_CASE(11) DQN_HEAD_CASE(12) DQN_HEAD_CASE(13) DQN_HEAD_CASE(14) DQN_HEAD_CASE(15)
    DQN_HEAD_CASE(16) DQN_HEAD_CASE(17) DQN_HEAD_CASE(18)
#undef DQN_HEAD_CASE
    default: break;
  }
  set_error("head_td: %d actions (at most %d)", nA, kFusedMaxA);
  return DQN_ERR_UNSUPPORTED;
}

bool is_head_layer(const dqn_net_desc *net, int l) {
  const dqn_layer_desc &L = net->layer[l];
  return l == net->n_layers - 1 && (L.kind == DQN_LAYER_DUELING || L.kind == DQN_LAYER_LINEAR);
}

HeadNet head_of(const dqn_net_desc *net, const float *params, const dqn_binding *b) {
  const int l = net->n_layers - 1;
  const dqn_layer_desc &L = net->layer[l];
  const bool duel = L.kind == DQN_LAYER_DUELING;
  HeadNet h;
  h.x = b->act[l - 1];
  h.wv = duel ? params + L.w_off : nullptr;
  h.bv = duel ? params + L.b_off : nullptr;
  h.wa = duel ? params + L.w2_off : params + L.w_off;
  h.ba = duel ? params + L.b2_off : params + L.b_off;
  h.q = b->act[l];
  h.rows = b->batch;
  return h;
}

}  // namespace
}  // namespace dqn

using namespace dqn;

extern "C" int64_t dqn_head_td_work_bytes(int32_t batch, int32_t n_actions) {
  return 256 + (int64_t)batch * (n_actions + 1) * (int64_t)sizeof(float);
}

extern "C" int dqn_head_td(void *stream, const dqn_net_desc *on_net, const float *on_params,
                           float *on_grads, const dqn_binding *on_bind,
                           const dqn_binding *on_view, const dqn_net_desc *tg_net,
                           const float *tg_params, const dqn_binding *tg_bind,
                           const int64_t *actions, const double *rewards,
                           const uint8_t *terminals, const double *weights, double gamma,
                           int32_t td_flags, double *targets, double *td, double *losses,
                           double *stats, void *work, int32_t *flags, double *host_out) {
  DQN_CHECK_ARG(on_net && on_params && on_grads && on_bind && on_view && tg_net && tg_params &&
                    tg_bind && actions && rewards && terminals && weights && targets && td &&
                    losses && work,
                "head_td: bad args");
  const int L = on_net->n_layers;
  if (L < 2 || tg_net->n_layers != L || !is_head_layer(on_net, L - 1) ||
      !is_head_layer(tg_net, L - 1)) {
    set_error("head_td: both networks need a linear or dueling head after a hidden layer");
    return DQN_ERR_UNSUPPORTED;
  }
  const dqn_layer_desc &H = on_net->layer[L - 1];
  const int F = H.in_h * H.in_w * H.in_c, nA = H.out_c, k = on_view->batch;
  const dqn_layer_desc &HT = tg_net->layer[L - 1];
  if (HT.kind != H.kind || HT.in_h * HT.in_w * HT.in_c != F || HT.out_c != nA ||
      nA > kFusedMaxA || k > kFusedMaxRows || tg_bind->batch != k ||
      !(on_bind->batch == k || on_bind->batch == 2 * k) ||
      ((td_flags & DQN_TD_DOUBLE) && on_bind->batch != 2 * k)) {
    set_error("head_td: unsupported head geometry / batch (nA <= 18, batch <= 1024)");
    return DQN_ERR_UNSUPPORTED;
  }
  HeadTdArgs p{};
  p.on = head_of(on_net, on_params, on_bind);
  p.tg = head_of(tg_net, tg_params, tg_bind);
  p.F = F;
  p.dueling = H.kind == DQN_LAYER_DUELING;
  p.k = k;
  p.actions = actions;
  p.rewards = rewards;
  p.terminals = terminals;
  p.weights = weights;
  p.gamma = gamma;
  p.td_flags = td_flags;
  p.targets = targets;
  p.td = td;
  p.losses = losses;
  p.stats = stats;
  p.dq = on_view->dact[L - 1];
  p.dx = on_view->dact[L - 2];
  p.mask = on_net->layer[L - 2].relu ? on_view->act[L - 2] : nullptr;
  const bool duel = p.dueling;
  p.gwv = duel ? on_grads + H.w_off : nullptr;
  p.gbv = duel ? on_grads + H.b_off : nullptr;
  p.gwa = duel ? on_grads + H.w2_off : on_grads + H.w_off;
  p.gba = duel ? on_grads + H.b2_off : on_grads + H.b_off;
  p.ticket = reinterpret_cast<int *>(work);
  p.gs = reinterpret_cast<float *>(reinterpret_cast<char *>(work) + 256);
  p.flags = flags;
  p.host_out = host_out;
  if (!p.dq) {
    set_error("head_td: on_view has no head gradient buffer");
    return DQN_ERR_INVALID_ARG;
  }
  return dispatch_head_td(as_stream(stream), nA, p);
}
