"""GPU tests of the acting loop around the device learner (SURVEY.md §8(f)
rank 1), mirroring the reference's pkg/tests/test_trainer.py cases, plus a
trajectory comparison with the reference Trainer's own records
(tests/golden/trainer_catch.npz, made by make_trainer_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def small_cfg(P, **overrides):
    base = {"preset": "desk", "env": "gridworld", "seed": 7, "max_steps": 600,
            "learning_start": 64, "replay_capacity": 512, "target_sync": 100,
            "eps_end_step": 300, "test_period": 250, "test_episodes": 2,
            "max_episode_steps": 40, "beta_end_step": 600}
    base.update(overrides)
    return P.resolve_config(base)


def run_collect(P, cfg):
    sink = P.RecordCollector()
    tr = P.Trainer(cfg, sink=sink)
    tr.run()
    return tr, sink.records


def test_select_action_is_argmax_of_forward(P):
    net = P.build_network("desk", (24, 24, 4), 3, True)
    P.init_params(net, 4)
    rng = np.random.default_rng(0)
    for i in range(20):
        s = (rng.integers(0, 256, size=(24, 24, 4)) / 255.0).astype(np.float32)
        q = net.forward(s[None]).cpu().numpy()[0]
        a = P.select_action(net, s, 0.0, rng)
        assert a == int(np.argmax(q)), (i, q)
    # eps = 1: always the random branch, drawing random() then integers()
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    for _ in range(10):
        a = P.select_action(net, s, 1.0, r1)
        r2.random()
        assert a == int(r2.integers(0, 3))
    with pytest.raises(ValueError):
        P.select_action(net, s, 1.5, r1)


def test_no_learning_before_learning_start(P):
    tr, _ = run_collect(P, small_cfg(P, max_steps=60, learning_start=64))
    assert tr.step == 60 and tr.learn_steps == 0


def test_learn_cadence_after_start(P):
    tr, _ = run_collect(P, small_cfg(P, max_steps=200, learning_start=64, update_period=4))
    assert tr.learn_steps == (200 - 64) // 4 + 1


def test_identical_seeds_identical_records(P):
    cfg = small_cfg(P, env="catch", max_steps=400)
    _, a = run_collect(P, cfg)
    _, b = run_collect(P, cfg)
    assert [r.row() for r in a] == [r.row() for r in b]
    assert len(a) > 0
    _, c = run_collect(P, small_cfg(P, env="catch", max_steps=400, seed=2))
    assert [r.row() for r in a] != [r.row() for r in c]


def test_eval_records_each_test_period(P):
    _, records = run_collect(P, small_cfg(P, env="catch", max_steps=500, test_period=250))
    assert [r.step for r in records if r.eval_mean is not None] == [250, 500]
    steps = [r.step for r in records]
    assert steps == sorted(steps)


def test_truncation_stores_nonterminal(P):
    cfg = small_cfg(P, env="gridworld", max_steps=30, max_episode_steps=10,
                    learning_start=30, batch_size=8)
    sink = P.RecordCollector()
    tr = P.Trainer(cfg, sink=sink)
    tr.env.max_steps = 10_000
    tr.run()
    mem = tr.memory.memory
    assert mem.size == 30
    assert not bool(mem.terminals[:30].any())
    assert len([r for r in sink.records if r.episode_return is not None]) == 3
    # gridworld frames (5x5 -> 24x24 bilinear) are not byte images: f32 ring
    assert mem.states.dtype == torch.float32


def test_terminal_episode_stores_terminal_flag(P):
    tr, _ = run_collect(P, small_cfg(P, env="catch", max_steps=23, learning_start=23,
                                     batch_size=8))
    mem = tr.memory.memory
    t = mem.terminals[:23].cpu().numpy()
    assert t.sum() == 1 and t[22]
    assert mem.states.dtype == torch.uint8           # catch 24x24: byte-exact ring


def test_uniform_memory_when_alpha_zero(P):
    tr = P.Trainer(small_cfg(P, priority_alpha=0.0))
    assert type(tr.memory) is P.ReplayMemory


def test_stored_states_match_preprocessed_frames(P):
    """The staged, batched insert puts exactly the reference's float states
    into the ring (u8 ring: f32(k)/255 <-> k)."""
    cfg = small_cfg(P, env="catch", max_steps=50, learning_start=48, batch_size=8,
                    update_period=4)
    tr = P.Trainer(cfg)
    seen = []
    orig = tr._staged.add

    def spy(state, action, reward, next_state, terminal):
        seen.append((state.copy(), next_state.copy()))
        orig(state, action, reward, next_state, terminal)
    tr._staged.add = spy
    tr.run()
    st = tr.memory.memory.states[:50].cpu().numpy()
    nx = tr.memory.memory.next_states[:50].cpu().numpy()
    for i, (s, n) in enumerate(seen):
        assert np.array_equal(st[i].astype(np.float32) / np.float32(255.0), s)
        assert np.array_equal(nx[i].astype(np.float32) / np.float32(255.0), n)


def test_trajectory_tracks_reference_trainer(P, golden):
    """Same config and seed as the reference run in the golden fixture.
    Until learning starts every decision is the reference's (same substreams,
    same greedy actions): records identical.  Catch episodes have a fixed
    length, so step / episode / epsilon / beta columns stay identical for the
    whole run.  The first learning episode's mean |TD| and loss agree within
    1e-3; later the free-running learner drifts from the reference (ReLU-mask
    flips amplified by RMSprop's first-moment-free step, SURVEY.md Appendix
    A.2: ~1e-6 at step 10, 1e-1 by step 30 for any re-associated fp32
    implementation) and the learning-quality check is the acceptance run
    (tools/catch_acceptance.py)."""
    g = golden("trainer_catch")
    import ast
    over = ast.literal_eval(str(g["overrides"]))
    tr, records = run_collect(P, P.resolve_config(over))
    ref = g["records"]
    assert len(records) == len(ref)
    assert tr.learn_steps == int(g["learn_steps"])
    learn_start = over["learning_start"]
    checked_learning = 0
    for i, (r, want) in enumerate(zip(records, ref)):
        got = [r.step, -1 if r.episode is None else r.episode] + [
            np.nan if v is None else v for v in (r.episode_return, r.epsilon, r.beta,
                                                 r.mean_abs_td, r.loss, r.eval_mean)]
        got = np.array(got, dtype=np.float64)
        assert np.array_equal(got[[0, 1, 3, 4]], want[[0, 1, 3, 4]]), (i, got, want)
        if r.step <= learn_start:
            assert np.array_equal(got, want, equal_nan=True), (i, got, want)
        elif checked_learning < 1 and not np.isnan(want[5]):
            assert got[2] == want[2]
            for c in (5, 6):
                assert abs(got[c] - want[c]) <= 1e-3 * abs(want[c]), (i, c, got[c], want[c])
            checked_learning += 1
    assert checked_learning == 1
