"""GPU tests of checkpoint export/import of the device training state
(SURVEY.md §8(f) rank 2), mirroring the reference's TestResume /
test_abort_writes_checkpoint (pkg/tests/test_trainer.py:102-153): a resumed
run reproduces the uninterrupted one record for record, the replay ring and
sum tree come back bit-exactly, and aborts / zero budgets write files."""

from __future__ import annotations

import dataclasses

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
    base = {"preset": "desk", "env": "catch", "seed": 7, "max_steps": 600,
            "learning_start": 64, "replay_capacity": 512, "target_sync": 100,
            "eps_end_step": 300, "test_period": 250, "test_episodes": 2,
            "max_episode_steps": 40, "beta_end_step": 600}
    base.update(overrides)
    return P.resolve_config(base)


def run_collect(P, cfg, out_dir=None):
    sink = P.RecordCollector()
    tr = P.Trainer(cfg, sink=sink, out_dir=out_dir)
    tr.run()
    return tr, sink.records


@pytest.mark.parametrize("alpha", [0.6, 0.0])
def test_resume_reproduces_uninterrupted_run(P, tmp_path, alpha):
    from paper_1804_05834_b200.checkpoint import load_checkpoint
    full, full_rec = run_collect(P, small_cfg(P, max_steps=400, checkpoint_include_memory=True,
                                              priority_alpha=alpha))
    half_cfg = small_cfg(P, max_steps=200, checkpoint_include_memory=True, priority_alpha=alpha)
    sink_a = P.RecordCollector()
    P.Trainer(half_cfg, sink=sink_a, out_dir=tmp_path).run()
    ck = load_checkpoint(tmp_path / "checkpoint_final.ckpt")
    ck.config = dataclasses.replace(ck.config, max_steps=400)
    sink_b = P.RecordCollector()
    resumed = P.Trainer.from_checkpoint(ck, sink=sink_b)
    resumed.run()
    stitched = [r.row() for r in sink_a.records + sink_b.records]
    assert stitched == [r.row() for r in full_rec]
    assert torch.equal(resumed.online.flat_values, full.online.flat_values)
    assert torch.equal(resumed.optimizer.flat_acc, full.optimizer.flat_acc)


def test_memory_and_tree_round_trip_bit_exact(P, tmp_path):
    from paper_1804_05834_b200.checkpoint import load_checkpoint
    tr = P.Trainer(small_cfg(P, max_steps=300, checkpoint_include_memory=True), out_dir=tmp_path)
    tr.run()
    ck = load_checkpoint(tmp_path / "checkpoint_final.ckpt")
    n = tr.memory.size
    ring = tr.memory.memory
    # on disk: the reference's float32 frames, exactly f32(k)/255
    st = ck.memory["states"]
    assert st.dtype == np.float32 and st.shape == (n, 24, 24, 4)
    assert np.array_equal(st, ring.states[:n].cpu().numpy().astype(np.float32) / np.float32(255.0))
    back = P.Trainer.from_checkpoint(ck)
    r2 = back.memory.memory
    for name in ("states", "next_states", "actions", "rewards", "terminals"):
        assert torch.equal(getattr(r2, name)[:n], getattr(ring, name)[:n]), name
    assert torch.equal(back.memory.tree.nodes, tr.memory.tree.nodes)
    assert back.memory.max_priority == tr.memory.max_priority
    assert (r2.cursor, r2.size) == (ring.cursor, ring.size)
    for (na, a), (nb, b) in zip(tr.online.named_tensors(), back.online.named_tensors()):
        assert na == nb and torch.equal(a.values, b.values)
    for (na, a), (nb, b) in zip(tr.target.named_tensors(), back.target.named_tensors()):
        assert torch.equal(a.values, b.values)


def test_resume_without_memory_restarts_buffer(P, tmp_path):
    from paper_1804_05834_b200.checkpoint import load_checkpoint
    P.Trainer(small_cfg(P, max_steps=150), out_dir=tmp_path).run()
    ck = load_checkpoint(tmp_path / "checkpoint_final.ckpt")
    assert ck.memory is None
    ck.config = dataclasses.replace(ck.config, max_steps=180)
    tr = P.Trainer.from_checkpoint(ck)
    assert tr.step == 150 and tr.memory.size == 0
    tr.run()
    assert tr.step == 180 and tr.memory.size == 30


def test_abort_and_zero_budget_write_checkpoints(P, tmp_path):
    tr, records = run_collect(P, small_cfg(P, max_steps=0), out_dir=tmp_path / "zero")
    assert tr.step == 0 and records == []
    assert (tmp_path / "zero" / "checkpoint_final.ckpt").exists()
    tr = P.Trainer(small_cfg(P, max_steps=100), out_dir=tmp_path / "abort")
    orig = tr.env.step
    calls = {"n": 0}

    def flaky(action):
        calls["n"] += 1
        if calls["n"] > 40:
            raise RuntimeError("emulator crashed")
        return orig(action)
    tr.env.step = flaky
    with pytest.raises(RuntimeError, match="emulator crashed"):
        tr.run()
    assert (tmp_path / "abort" / "checkpoint_abort.ckpt").exists()


def test_periodic_checkpoints(P, tmp_path):
    run_collect(P, small_cfg(P, max_steps=100, checkpoint_period=40), out_dir=tmp_path)
    names = sorted(p.name for p in tmp_path.iterdir())
    assert names == ["checkpoint_40.ckpt", "checkpoint_80.ckpt", "checkpoint_final.ckpt"]


def test_architecture_mismatch(P, tmp_path):
    from paper_1804_05834_b200.checkpoint import load_checkpoint, load_params_into
    from paper_1804_05834_b200.errors import ArchitectureMismatchError
    P.Trainer(small_cfg(P, max_steps=10), out_dir=tmp_path).run()
    ck = load_checkpoint(tmp_path / "checkpoint_final.ckpt")
    plain = P.build_network("desk", (24, 24, 4), 3, False)
    with pytest.raises(ArchitectureMismatchError):
        load_params_into(plain, ck.params)
