// The TD block of one batch row, shared by td_loss_kernel (td_optim.cu) and
// the fused head kernel (head_td.cu).
#pragma once

#include "common.cuh"

namespace dqn {

// One batch row of the TD block (agent.py:58-73, 110-124), fp64 in the
// reference's operation order; shared by td_loss_kernel and the fused head
// kernel (head_td.cu).  Writes targets/td/losses[j] and dq row j; returns
// |d| and the loss for the batch statistics.
// The arithmetic of td_row without the stores: action a, target y, TD error
// d, loss and the float output gradient g of the taken action.
__device__ __forceinline__ void td_core(int j, const float *__restrict__ q_on,
                                        const float *__restrict__ q_next_on,
                                        const float *__restrict__ q_next_tg,
                                        const int64_t *__restrict__ actions,
                                        const double *__restrict__ rewards,
                                        const uint8_t *__restrict__ terminals,
                                        const double *__restrict__ weights, int nA, double gamma,
                                        int flags, int64_t &a_out, double &y_out, double &d_out,
                                        double &loss_out, float &g_out) {
  const float *qt = q_next_tg + (int64_t)j * nA;
  double boot;
  if (flags & DQN_TD_DOUBLE) {
    const float *qo = q_next_on + (int64_t)j * nA;
    int best = 0;
    float bv = qo[0];
    for (int a = 1; a < nA; ++a)
      if (qo[a] > bv) { bv = qo[a]; best = a; }
    boot = __dmul_rn(gamma, (double)qt[best]);
  } else {
    float mx = qt[0];
    for (int a = 1; a < nA; ++a) mx = fmaxf(mx, qt[a]);
    boot = __dmul_rn(gamma, (double)mx);
  }
  double r = rewards[j];
  if (flags & DQN_TD_REWARD_CLIP) r = fmin(fmax(r, -1.0), 1.0);
  const double y = __dadd_rn(r, terminals[j] ? 0.0 : boot);
  const int64_t a = actions[j];
  const double d = __dsub_rn(y, (double)q_on[(int64_t)j * nA + a]);
  const double w = weights[j];
  double loss, g;
  if (flags & DQN_TD_HUBER) {
    const double ad = fabs(d);
    loss = __dmul_rn(w, ad <= 1.0 ? __dmul_rn(__dmul_rn(0.5, d), d) : __dsub_rn(ad, 0.5));
    g = __dmul_rn(-w, fmin(fmax(d, -1.0), 1.0));
  } else {
    loss = __dmul_rn(__dmul_rn(__dmul_rn(0.5, w), d), d);
    g = __dmul_rn(-w, d);
  }
  a_out = a;
  y_out = y;
  d_out = d;
  loss_out = loss;
  g_out = __double2float_rn(g);
}

__device__ __forceinline__ void td_row(int j, const float *__restrict__ q_on, const float *__restrict__ q_next_on,
                       const float *__restrict__ q_next_tg, const int64_t *__restrict__ actions,
                       const double *__restrict__ rewards, const uint8_t *__restrict__ terminals,
                       const double *__restrict__ weights, int nA, double gamma, int flags,
                       double *__restrict__ targets, double *__restrict__ td,
                       double *__restrict__ losses, float *__restrict__ dq, double &abs_d,
                       double &loss_out) {
  const float *qt = q_next_tg + (int64_t)j * nA;
  double boot;
  if (flags & DQN_TD_DOUBLE) {
    // a* = argmax_a Q_online(s', a), first maximum (agent.py:70)
    const float *qo = q_next_on + (int64_t)j * nA;
    int best = 0;
    float bv = qo[0];
    for (int a = 1; a < nA; ++a)
      if (qo[a] > bv) { bv = qo[a]; best = a; }
    boot = __dmul_rn(gamma, (double)qt[best]);
  } else {
    float mx = qt[0];
    for (int a = 1; a < nA; ++a) mx = fmaxf(mx, qt[a]);
    boot = __dmul_rn(gamma, (double)mx);   // gamma * q_next.max(axis=1)
  }
  double r = rewards[j];
  if (flags & DQN_TD_REWARD_CLIP) r = fmin(fmax(r, -1.0), 1.0);   // agent.py:102-103
  const double y = __dadd_rn(r, terminals[j] ? 0.0 : boot);       // r + where(t, 0, boot)
  const int64_t a = actions[j];
  const double qsa = (double)q_on[(int64_t)j * nA + a];
  const double d = __dsub_rn(y, qsa);
  const double w = weights[j];
  double loss, g;
  if (flags & DQN_TD_HUBER) {
    const double ad = fabs(d);
    loss = __dmul_rn(w, ad <= 1.0 ? __dmul_rn(__dmul_rn(0.5, d), d) : __dsub_rn(ad, 0.5));
    g = __dmul_rn(-w, fmin(fmax(d, -1.0), 1.0));
  } else {
    loss = __dmul_rn(__dmul_rn(__dmul_rn(0.5, w), d), d);   // ((0.5*w)*d)*d
    g = __dmul_rn(-w, d);                                   // (-w)*d
  }
  targets[j] = y;
  td[j] = d;
  losses[j] = loss;
  const float gf = __double2float_rn(g);
  for (int c = 0; c < nA; ++c) dq[(int64_t)j * nA + c] = (c == a) ? gf : 0.f;
  abs_d = fabs(d);
  loss_out = loss;
}

}  // namespace dqn

