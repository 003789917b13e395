"""Host side of the acting loop against the reference's own behaviour
(golden fixtures made by tests/golden/make_trainer_golden.py from the
unmodified reference): environment dynamics, preprocessing, frame stacking
and configuration resolution.  CPU only, bit-exact."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1804_05834_b200 import config as C
from paper_1804_05834_b200 import envs as E
from paper_1804_05834_b200.errors import ConfigError

ENV_CASES = [
    ("catch", {}, 11),
    ("catch", {"height": 10, "width": 7, "paddle_width": 2}, 12),
    ("gridworld", {"size": 5, "max_steps": 30}, 13),
    ("tabular", {}, 14),
]


@pytest.mark.parametrize("ci", range(len(ENV_CASES)))
def test_env_sequences_match_reference(golden, ci):
    g = golden("envs")
    name, params, seed = ENV_CASES[ci]
    env = E.make_env(name, rng=np.random.default_rng(seed), **params)
    frames, rewards, terms = [env.reset()], [], []
    for a in g[f"env{ci}_actions"]:
        r = env.step(int(a))
        frames.append(r.observation)
        rewards.append(r.reward)
        terms.append(r.terminal)
        if r.terminal:
            frames.append(env.reset())
    assert np.array_equal(np.stack(frames), g[f"env{ci}_frames"])
    assert np.array_equal(np.array(rewards), g[f"env{ci}_rewards"])
    assert np.array_equal(np.array(terms), g[f"env{ci}_terminals"])


def test_preprocess_frame_bit_exact(golden):
    g = golden("envs")
    i = 0
    while f"pre{i}_in" in g:
        out = E.preprocess_frame(g[f"pre{i}_in"], tuple(int(s) for s in g[f"pre{i}_size"]))
        assert out.dtype == np.float32
        assert np.array_equal(out, g[f"pre{i}_out"]), i
        i += 1
    assert i == 6
    assert np.array_equal(E.preprocess_frame(g["pref_in"], (5, 6)), g["pref_out"])


def test_preprocessor_stack_bit_exact(golden):
    g = golden("envs")
    pre = E.Preprocessor((6, 5), 3)
    seq = g["stack_in"]
    got = [pre.reset(seq[0])] + [pre.push(s) for s in seq[1:]]
    assert np.array_equal(np.stack(got), g["stack_out"])
    st = pre.get_state()
    pre2 = E.Preprocessor((6, 5), 3)
    pre2.set_state(st)
    assert np.array_equal(pre2._stacked(), got[-1])


def test_byte_exact_frames_round_trip_through_u8():
    # a u8 frame at the target size preprocesses to exact f32(k)/255, so the
    # trainer's uint8 ring (rint(x * 255)) stores it bit-for-bit
    f = np.arange(256, dtype=np.uint8).reshape(16, 16)
    x = E.preprocess_frame(f, (16, 16))
    assert E.byte_exact(f, (16, 16))
    assert np.array_equal(np.rint(x * 255.0).astype(np.uint8), f)
    assert np.array_equal(np.float32(np.rint(x * 255.0).astype(np.uint8)) / np.float32(255.0), x)
    assert not E.byte_exact(f, (24, 24))
    assert not E.byte_exact(f.astype(np.float32), (16, 16))


def test_env_errors_and_state_round_trip():
    env = E.Catch(rng=np.random.default_rng(0))
    with pytest.raises(RuntimeError):
        env.step(1)
    env.reset()
    with pytest.raises(ValueError):
        env.step(3)
    env.step(2)
    st = env.get_state()
    other = E.Catch()
    other.set_state(st)
    assert np.array_equal(other._frame(), env._frame())
    with pytest.raises(ValueError):
        E.make_env("pong")
    with pytest.raises(ValueError):
        E.Catch(height=1)


def test_catch_random_policy_catch_rate():
    # ball column independent of the paddle's walk: P(catch) = 8/24 = 1/3
    env = E.Catch(rng=np.random.default_rng(3))
    rng = np.random.default_rng(4)
    total, n = 0.0, 3000
    for _ in range(n):
        env.reset()
        while True:
            r = env.step(int(rng.integers(0, 3)))
            if r.terminal:
                total += r.reward
                break
    assert abs(total / n - (-1.0 / 3.0)) < 0.05


def test_resolve_config_desk_preset_and_validation():
    cfg = C.resolve_config({"preset": "desk", "seed": 3})
    assert (cfg.frame_size, cfg.replay_capacity, cfg.learning_start, cfg.eps_end_step,
            cfg.target_sync, cfg.max_steps, cfg.test_period) == (24, 10_000, 5_000, 50_000,
                                                                  1_000, 200_000, 25_000)
    assert cfg.beta_end_step == 200_000 and cfg.seed == 3
    with pytest.raises(ConfigError):
        C.resolve_config({"gamma": 1.0})
    with pytest.raises(ConfigError):
        C.resolve_config({"learning_start": 8, "batch_size": 32})
    with pytest.raises(ConfigError):
        C.resolve_config({"nope": 1})
    with pytest.raises(ConfigError):
        C.resolve_config({"preset": "huge"})


def test_config_matches_live_reference(reference_deepq):
    from deepq.config import resolve_config as ref_resolve
    import dataclasses
    for over in ({}, {"preset": "desk"}, {"preset": "desk", "env": "gridworld", "seed": 9,
                                          "beta_end_step": 77}):
        a = dataclasses.asdict(C.resolve_config(over))
        b = dataclasses.asdict(ref_resolve(over))
        assert a == b
