"""Synthetic Atari-shaped transitions (SURVEY.md §8(d) "Synthetic inputs").

Frames are a pure function of (seed, kind, slot, byte) through a splitmix64
counter hash, so the host (numpy, for the CPU oracle) and the device
(``dqn_ring_fill_hash`` in csrc/replay.cu) produce identical bytes without
moving 56 GB across PCIe.  Metadata (actions, rewards, terminals) and the
warm-up priorities come from ``np.random.SeedSequence([seed, k])`` streams
like the reference's named substreams (agent.py:33-38).
"""

from __future__ import annotations

import numpy as np

FRAME_SHAPE = (84, 84, 4)
FRAME_BYTES = 84 * 84 * 4          # 28,224 B per stacked state
STREAM_META, STREAM_TD = 11, 12

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def frame_counter_base(seed: int, kind: int) -> int:
    """64-bit counter base for (seed, kind); kind 0 = state, 1 = next_state."""
    return ((int(seed) & 0xFFFF) << 48) | ((int(kind) & 1) << 47)


def frames(seed: int, kind: int, slots, slot_bytes: int = FRAME_BYTES,
           shape=FRAME_SHAPE) -> np.ndarray:
    """uint8 frames for ``slots`` (array of slot ids) -> (n, *shape)."""
    slots = np.asarray(slots, dtype=np.uint64).reshape(-1)
    words = slot_bytes // 8
    base = np.uint64(frame_counter_base(seed, kind))
    ctr = base | (slots[:, None] * np.uint64(words) + np.arange(words, dtype=np.uint64)[None, :])
    h = splitmix64(ctr)
    return h.astype("<u8").view(np.uint8).reshape((len(slots),) + tuple(shape))


def metadata(seed: int, n: int, n_actions: int = 4):
    """actions i64, rewards f64 in {-1,0,1} (p=.05/.90/.05), terminals
    Bernoulli(0.01)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), STREAM_META]))
    actions = rng.integers(0, n_actions, size=n).astype(np.int64)
    rewards = rng.choice(np.array([-1.0, 0.0, 1.0]), size=n, p=[0.05, 0.90, 0.05])
    terminals = rng.random(n) < 0.01
    return actions, rewards.astype(np.float64), terminals


def warmup_td(seed: int, n: int) -> np.ndarray:
    """|N(0,1)| TD errors used for the one warm-up priority update."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), STREAM_TD]))
    return np.abs(rng.standard_normal(n))
