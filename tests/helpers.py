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
