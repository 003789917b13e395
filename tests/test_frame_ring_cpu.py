"""Host bookkeeping of the frame-deduplicated ring (frame_ring.FrameIndex):
pool ids, reference counts, eviction and exhaustion, checked against a
full-stack model of the same ring (what the reference's ReplayMemory holds,
replay.py:83-102).  A simulated pool applies the uploads exactly as the
device does, so "every live slot rebuilds its planes" proves no live frame
was ever overwritten."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1804_05834_b200.errors import ConfigError
from paper_1804_05834_b200.frame_ring import FrameIndex

STACK = 4


def episodic(rng, n, max_len=7, size=16):
    """(state planes, next planes) of an Atari-like stream: each episode
    starts from one frame repeated STACK times, every step shifts one new
    frame in, the next episode starts fresh."""
    out = []
    while len(out) < n:
        f = rng.integers(0, 256, size, dtype=np.uint8).tobytes()
        stack = [f] * STACK
        for _ in range(int(rng.integers(1, max_len + 1))):
            new = rng.integers(0, 256, size, dtype=np.uint8).tobytes()
            nxt = stack[1:] + [new]
            out.append(stack + nxt)
            stack = nxt
    return out[:n]


def check(ix, pool, model):
    for slot, planes in model.items():
        assert [pool[int(f)] for f in ix.ids[slot]] == planes, slot
    counts = np.bincount(ix.ids[list(model)].ravel(), minlength=ix.frame_capacity) \
        if model else np.zeros(ix.frame_capacity, np.int64)
    assert np.array_equal(counts, ix.refs)
    assert len(ix.free) == int(np.sum(ix.refs == 0))
    assert len(set(ix.free)) == len(ix.free)


@pytest.mark.parametrize("capacity", [1, 2, 5, 64])
def test_stream_rebuilds_every_live_slot(capacity):
    rng = np.random.default_rng(capacity)
    ix = FrameIndex(capacity, 2 * capacity + 4 * STACK, STACK)
    pool, model = {}, {}
    for t, planes in enumerate(episodic(rng, 6 * capacity + 20)):
        slot = t % capacity
        for fid, p in ix.assign(slot, planes):
            pool[fid] = p
        model[slot] = planes
        check(ix, pool, model)
    # an episodic stream costs about one new frame per transition
    assert ix.live_frames <= capacity + 2 * STACK + capacity


def test_dedup_ratio_on_long_episodes():
    rng = np.random.default_rng(3)
    cap = 500
    ix = FrameIndex(cap, 2 * cap + 4 * STACK, STACK)
    for t, planes in enumerate(episodic(rng, 2000, max_len=200)):
        ix.assign(t % cap, planes)
    # full stacks: 8 planes per slot; here ~1 per slot plus episode starts
    assert ix.live_frames < 1.2 * cap


def test_unrelated_transitions_still_correct():
    """No sharing at all (random stacks): 8 new planes per transition, the
    pool must hold them, results stay exact."""
    rng = np.random.default_rng(5)
    cap = 6
    ix = FrameIndex(cap, 8 * cap + 8, STACK)
    pool, model = {}, {}
    for t in range(40):
        planes = [rng.integers(0, 256, 16, dtype=np.uint8).tobytes() for _ in range(2 * STACK)]
        for fid, p in ix.assign(t % cap, planes):
            pool[fid] = p
        model[t % cap] = planes
        check(ix, pool, model)


def test_exhaustion_raises_and_leaves_state_consistent():
    rng = np.random.default_rng(9)
    cap = 4
    ix = FrameIndex(cap, 12, STACK)
    pool, model = {}, {}
    with pytest.raises(ConfigError, match="frame pool exhausted"):
        for t in range(100):
            planes = [rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
                      for _ in range(2 * STACK)]
            for fid, p in ix.assign(t % cap, planes):
                pool[fid] = p
            model[t % cap] = planes
    check(ix, pool, model)


def test_too_small_pool_rejected():
    with pytest.raises(ConfigError):
        FrameIndex(4, 2 * STACK - 1, STACK)
