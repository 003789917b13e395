"""Synthetic input generator (host side): deterministic, distinct streams."""

import numpy as np

from paper_1804_05834_b200 import synth


def test_frames_deterministic_and_distinct():
    a = synth.frames(3, 0, [0, 1, 999_999])
    b = synth.frames(3, 0, [0, 1, 999_999])
    c = synth.frames(3, 1, [0, 1, 999_999])
    assert a.shape == (3, 84, 84, 4) and a.dtype == np.uint8
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    assert not np.array_equal(a[0], a[1])
    # roughly uniform bytes
    assert abs(a.mean() - 127.5) < 2.0


def test_splitmix_known_answer():
    # splitmix64 of 0 (the well-known first output of seed 0)
    assert int(synth.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_metadata_distribution():
    a, r, t = synth.metadata(0, 100_000)
    assert a.min() == 0 and a.max() == 3
    assert set(np.unique(r)) == {-1.0, 0.0, 1.0}
    assert 0.85 < np.mean(r == 0.0) < 0.95
    assert 0.005 < t.mean() < 0.015
