"""Shared test helpers: build oracle learners on the synthetic data and
compare with the norm-wise metrics the parity protocol prescribes
(SURVEY.md Appendix A.3)."""

from __future__ import annotations

import numpy as np

from oracle import deepq_oracle as O
from paper_1804_05834_b200 import synth

ATARI = (84, 84, 4)


def rel_norm(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b.ravel())
    num = np.linalg.norm((a - b).ravel())
    if den == 0.0:
        return float(num)
    return float(num / den)


def ulp_diff(a, b) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(a - b)


def oracle_fill(mem, n, seed, per: bool):
    """Fill an oracle ring/PER like make_golden.fill_reference_memory."""
    ring = mem.ring if per else mem
    slots = np.arange(n)
    s = synth.frames(seed, 0, slots)
    s2 = synth.frames(seed, 1, slots)
    a, r, t = synth.metadata(seed, n)
    for i in range(n):
        if per:
            mem.store(s[i], a[i], r[i], s2[i], t[i])
        else:
            ring.store(s[i], a[i], r[i], s2[i], t[i])
    if per:
        mem.update_priorities(np.arange(n), synth.warmup_td(seed, n))
    return ring


def oracle_learner(dueling, double, per, huber=False, cap=64, seed=7, beta_end=1000,
                   online_seed=1, target_seed=2):
    online = O.QNet(O.ATARI_TRUNK, ATARI, 4, dueling)
    target = O.QNet(O.ATARI_TRUNK, ATARI, 4, dueling)
    online.init(online_seed)
    target.init(target_seed)
    opt = O.RmsPropState(online)
    if per:
        mem = O.PerReplay(cap, ATARI, 0.6, 0.01, (0.4, 1.0, beta_end))
    else:
        mem = O.Ring(cap, ATARI)
    oracle_fill(mem, cap, seed, per)
    cfg = O.LearnCfg(double=double, huber=huber)
    return online, target, mem, opt, cfg


def follow_device_relu_kinks(o_net, dev_acts, tol: float = 1e-5) -> list:
    """Resolve ReLU kinks the way the device did, for the oracle's NEXT
    backward pass (``o_net.backward`` is wrapped once).

    A pre-activation within fp32 rounding of zero (|z| / max|z| below
    rounding level) may land on either side of the kink depending on the
    summation order, and the first RMSprop step (w -= lr g / (sqrt(0.05 g^2) +
    eps), about lr * sign(g) * 4.5) turns the resulting change of a near-zero
    gradient element into a full-size weight difference.  Every mask
    disagreement between the oracle's forward (``o_net._acts``) and the
    device's (``dev_acts[u] > 0``, the fused-ReLU unit outputs, batch rows
    first) must sit at |z| / max|z| < ``tol``; those elements then take the
    device's side.  Returns [(relu op index, flips, worst |z| / max|z|)]."""
    flips = []
    orig = o_net.backward

    def backward(dq):
        unit = 0
        for li, (kind, _name, _geo) in enumerate(o_net.ops):
            if kind != "relu":
                continue
            z, aux = o_net._acts[li]
            dev = np.asarray(dev_acts[unit]).ravel()[: z.size].reshape(z.shape) > 0
            unit += 1
            diff = dev != (z > 0)
            if diff.any():
                worst = float(np.abs(z[diff]).max() / np.abs(z).max())
                assert worst < tol, f"ReLU mask differs away from the kink: relu op {li}, {worst:.2e}"
                z2 = z.copy()
                z2[diff] = np.where(dev[diff], np.finfo(z.dtype).tiny, 0)
                o_net._acts[li] = (z2, aux)
                flips.append((li, int(diff.sum()), worst))
        o_net.backward = orig
        return orig(dq)

    o_net.backward = backward
    return flips
