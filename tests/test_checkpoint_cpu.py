"""CYRL checkpoint format (checkpoint.py:1-194 of the reference): byte-level
compatibility in both directions with the live reference (build container),
a committed reference-written file (tests/golden/ref_small.ckpt, made by
tests/golden/make_ckpt_golden.py), and the load-failure taxonomy.  CPU only
(the format layer is host code; the Trainer export/import is in
tests/test_gpu_checkpoint.py)."""

from __future__ import annotations

import dataclasses
import struct
import zlib

import numpy as np
import pytest

from paper_1804_05834_b200 import checkpoint as K
from paper_1804_05834_b200 import errors as E
from paper_1804_05834_b200.config import resolve_config
from tests.conftest import GOLDEN


def sample_ckpt(cfg_cls=None, resolve=resolve_config, Ck=K.Checkpoint):
    rng = np.random.default_rng(0)
    cfg = resolve({"preset": "desk", "seed": 4, "checkpoint_include_memory": True})
    return Ck(
        config=cfg,
        state={"step": 123, "episode": 5, "rng_env": np.random.default_rng(1).bit_generator.state,
               "env_state": {"ball_row": 3, "done": False}, "max_priority": 1.5,
               "needs_reset": False},
        params={"conv1.weight": rng.standard_normal((6, 6, 4, 16)).astype(np.float32),
                "conv1.bias": np.zeros(16, np.float32)},
        target={"conv1.weight": rng.standard_normal((6, 6, 4, 16)).astype(np.float32),
                "conv1.bias": np.ones(16, np.float32)},
        optim={"conv1.weight": rng.random((6, 6, 4, 16)).astype(np.float32),
               "conv1.bias": rng.random(16).astype(np.float32)},
        frames=rng.random((4, 24, 24)).astype(np.float32),
        memory={"states": rng.random((3, 24, 24, 4)).astype(np.float32),
                "actions": np.array([0, 2, 1], dtype=np.int64),
                "rewards": np.array([0.0, -1.0, 1.0]),
                "terminals": np.array([False, True, False]),
                "priorities": rng.random(3)},
    )


def assert_same(a, b):
    assert dataclasses.asdict(a.config) == dataclasses.asdict(b.config)
    assert a.state == b.state
    for sec in ("params", "target", "optim", "memory"):
        da, db = getattr(a, sec), getattr(b, sec)
        assert list(da) == list(db)
        for k in da:
            x, y = np.asarray(da[k]), np.asarray(db[k])
            assert x.shape == y.shape
            assert np.array_equal(x.astype(y.dtype) if y.dtype != bool else x.astype(bool), y), k
    assert np.array_equal(a.frames, b.frames)


def test_round_trip(tmp_path):
    c = sample_ckpt()
    K.save_checkpoint(tmp_path / "a.ckpt", c)
    assert_same(c, K.load_checkpoint(tmp_path / "a.ckpt"))
    c.memory = None
    K.save_checkpoint(tmp_path / "b.ckpt", c)
    assert K.load_checkpoint(tmp_path / "b.ckpt").memory is None


def test_failure_taxonomy(tmp_path):
    p = tmp_path / "a.ckpt"
    K.save_checkpoint(p, sample_ckpt())
    blob = bytearray(p.read_bytes())
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(E.CheckpointMagicError):
        K.load_checkpoint(bad)
    flipped = bytearray(blob)
    flipped[len(blob) // 2] ^= 0x40
    bad.write_bytes(bytes(flipped))
    with pytest.raises(E.CheckpointCRCError):
        K.load_checkpoint(bad)
    body = b"CYRL" + struct.pack("<I", 2) + bytes(blob[8:-4])
    bad.write_bytes(body + struct.pack("<I", zlib.crc32(body)))
    with pytest.raises(E.CheckpointVersionError):
        K.load_checkpoint(bad)
    body = b"CYRL" + struct.pack("<I", 1)            # no sections at all
    bad.write_bytes(body + struct.pack("<I", zlib.crc32(body)))
    with pytest.raises(E.CheckpointError):
        K.load_checkpoint(bad)
    bad.write_bytes(b"CY")
    with pytest.raises(E.CheckpointMagicError):
        K.load_checkpoint(bad)


def test_loads_reference_written_golden_file():
    c = K.load_checkpoint(GOLDEN / "ref_small.ckpt")
    want = np.load(GOLDEN / "ref_small_arrays.npz")
    for sec in ("params", "target", "optim", "memory"):
        for k, v in getattr(c, sec).items():
            assert np.array_equal(v, want[f"{sec}/{k}"]), (sec, k)
    assert np.array_equal(c.frames, want["frames"])
    assert c.config.preset == "desk" and c.config.seed == 4
    assert c.state["step"] == 123


def test_byte_identical_to_live_reference(tmp_path, reference_deepq):
    from deepq import checkpoint as RK
    from deepq.config import resolve_config as ref_resolve
    ours = sample_ckpt()
    ref = sample_ckpt(resolve=ref_resolve, Ck=RK.Checkpoint)
    K.save_checkpoint(tmp_path / "ours.ckpt", ours)
    RK.save_checkpoint(tmp_path / "ref.ckpt", ref)
    assert (tmp_path / "ours.ckpt").read_bytes() == (tmp_path / "ref.ckpt").read_bytes()
    # and each side loads the other's file
    assert_same(ours, K.load_checkpoint(tmp_path / "ref.ckpt"))
    r = RK.load_checkpoint(tmp_path / "ours.ckpt")
    assert r.state == ours.state
    assert dataclasses.asdict(r.config) == dataclasses.asdict(ours.config)
