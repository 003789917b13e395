"""Frame-deduplicated ring (frame_ring.py, dqn_frame_gather) against the
full-stack ring holding the same transitions (the reference's storage,
replay.py:83-115): sampled bytes and metadata identical, learn_step on it
bit-identical, footprint ~1/8 for an episodic stream."""

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


def episodic(rng, n, shape, max_len=9):
    """Transitions of an Atari-like stream: an episode starts from one frame
    repeated, each step shifts one new frame into the stack."""
    h, w, s = shape
    out = []
    while len(out) < n:
        stack = [rng.integers(0, 256, (h, w), dtype=np.uint8)] * s
        for _ in range(int(rng.integers(1, max_len + 1))):
            nxt = stack[1:] + [rng.integers(0, 256, (h, w), dtype=np.uint8)]
            out.append((np.stack(stack, -1), int(rng.integers(0, 4)),
                        float(rng.choice([-1.0, 0.0, 1.0])), np.stack(nxt, -1),
                        bool(rng.random() < 0.1)))
            stack = nxt
    return out[:n]


def _pair(P, cap, shape, stream, as_float=False):
    from paper_1804_05834_b200.frame_ring import FrameDedupMemory
    full = P.ReplayMemory(cap, shape)
    dedup = FrameDedupMemory(cap, shape)
    for s, a, r, s2, t in stream:
        if as_float:
            s, s2 = s.astype(np.float32) / np.float32(255.0), s2.astype(np.float32) / np.float32(255.0)
        tr = P.Transition(s, a, r, s2, t)
        assert full.store(tr) == dedup.store(tr)
    return full, dedup


@pytest.mark.parametrize("shape", [(84, 84, 4), (10, 10, 4), (10, 10, 3), (9, 7, 4)])
def test_gather_matches_full_stack_ring(P, shape):
    rng = np.random.default_rng(sum(shape))
    cap = 40
    full, dedup = _pair(P, cap, shape, episodic(rng, 3 * cap + 7, shape))
    assert full.size == dedup.size == cap and full.cursor == dedup.cursor
    idx = rng.integers(0, cap, 300)
    a, b = full.sample_uniform(300, np.random.default_rng(1)), dedup.sample_uniform(300, np.random.default_rng(1))
    for f in ("states", "next_states", "actions", "rewards", "terminals", "indices"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    ti = torch.as_tensor(idx, device="cuda")
    out = [torch.empty((300,) + shape, dtype=torch.uint8, device="cuda") for _ in range(2)]
    dedup.gather_into(ti, 300, out[0], out[1], None, None, None)
    assert torch.equal(out[0], full.states[ti]) and torch.equal(out[1], full.next_states[ti])


def test_float_frames_and_footprint(P):
    rng = np.random.default_rng(7)
    shape, cap = (84, 84, 4), 64
    stream = episodic(rng, 2 * cap, shape, max_len=40)
    full, dedup = _pair(P, cap, shape, stream, as_float=True)
    ti = torch.arange(cap, device="cuda")
    s, s2 = torch.empty_like(full.states), torch.empty_like(full.next_states)
    dedup.gather_into(ti, cap, s, s2, None, None, None)
    assert torch.equal(s, full.states) and torch.equal(s2, full.next_states)
    full_bytes = 2 * cap * full.slot_bytes
    assert dedup.resident_bytes < 0.3 * full_bytes, (dedup.resident_bytes, full_bytes)


@pytest.mark.parametrize("fused", [True, False])
def test_learn_step_identical_on_dedup_ring(P, fused, monkeypatch):
    """The learner over PrioritizedReplay(frame_dedup=True) -- the graph's
    batch from dqn_frame_sample_gather (descent + stack assembly in one
    launch) or dqn_tree_sample + dqn_frame_gather -- gives the same TdResults
    and parameters as over the full-stack ring, bit for bit."""
    monkeypatch.setattr(P.agent, "FUSED_SAMPLE", fused)
    rng = np.random.default_rng(11)
    shape, cap = (24, 24, 4), 256
    stream = episodic(rng, 300, shape)
    runs = []
    for dedup in (False, True):
        cfg = P.RunConfig(batch_size=32, double=True, dueling=True, beta_end_step=1000)
        on = P.build_network("desk", shape, 3, True)
        tg = P.build_network("desk", shape, 3, True)
        P.init_params(on, 1)
        P.sync_target(on, tg)
        opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
        mem = P.PrioritizedReplay(cap, shape, P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()),
                                  frame_dedup=dedup)
        for s, a, r, s2, t in stream:
            mem.store(P.Transition(s, a % 3, r, s2, t))
        g = np.random.default_rng(5)
        res = [P.learn_step(on, tg, mem, opt, cfg, 100 + i, g) for i in range(4)]
        runs.append((res, on.flat_values.clone(), mem.tree.nodes.clone()))
    (ra, wa, na), (rb, wb, nb) = runs
    for x, y in zip(ra, rb):
        assert np.array_equal(x.td_errors, y.td_errors) and np.array_equal(x.losses, y.losses)
    assert torch.equal(wa, wb) and torch.equal(na, nb)


def test_store_many_matches_store(P):
    """The batched insert (one upload for the batch, pool ids possibly freed
    and reused inside it) leaves the same sampled bytes as per-transition
    stores and as the full-stack ring."""
    from paper_1804_05834_b200.frame_ring import FrameDedupMemory
    rng = np.random.default_rng(21)
    shape, cap = (84, 84, 4), 16
    stream = episodic(rng, 70, shape, max_len=5)
    full, one = _pair(P, cap, shape, stream)
    many = FrameDedupMemory(cap, shape, frame_capacity=2 * cap + 16)
    for c0 in range(0, len(stream), 23):               # batches that wrap the ring
        chunk = stream[c0:c0 + 23]
        many.store_many([c[0] for c in chunk], [c[1] for c in chunk], [c[2] for c in chunk],
                        [c[3] for c in chunk], [c[4] for c in chunk])
    assert many.cursor == full.cursor and many.size == full.size
    # the full-stack ring's batched insert with batches longer than the ring
    batched = P.ReplayMemory(cap, shape)
    for c0 in range(0, len(stream), 23):
        chunk = stream[c0:c0 + 23]
        batched.store_many(np.stack([c[0] for c in chunk]), [c[1] for c in chunk],
                           [c[2] for c in chunk], np.stack([c[3] for c in chunk]),
                           [c[4] for c in chunk])
    for f in ("states", "next_states", "actions", "rewards", "terminals"):
        assert torch.equal(getattr(batched, f), getattr(full, f)), f
    ti = torch.arange(cap, device="cuda")
    for mem in (one, many):
        s, s2 = torch.empty_like(full.states), torch.empty_like(full.next_states)
        a = torch.empty(cap, dtype=torch.int64, device="cuda")
        r = torch.empty(cap, dtype=torch.float64, device="cuda")
        t = torch.empty(cap, dtype=torch.bool, device="cuda")
        mem.gather_into(ti, cap, s, s2, a, r, t)
        assert torch.equal(s, full.states) and torch.equal(s2, full.next_states)
        assert torch.equal(a, full.actions) and torch.equal(r, full.rewards)
        assert torch.equal(t, full.terminals)


def test_store_many_validates_before_assigning(P):
    """a malformed state in the middle of a batch raises before
    any transition is assigned; later stores still match the full ring."""
    from paper_1804_05834_b200.errors import GeometryError
    from paper_1804_05834_b200.frame_ring import FrameDedupMemory
    rng = np.random.default_rng(3)
    shape, cap = (10, 10, 4), 16
    stream = episodic(rng, 12, shape)
    full, dedup = P.ReplayMemory(cap, shape), FrameDedupMemory(cap, shape)
    cols = list(zip(*stream))
    bad = list(cols[0])
    bad[3] = np.zeros((10, 10, 3), dtype=np.uint8)           # wrong stack depth
    with pytest.raises(GeometryError):
        dedup.store_many(bad, cols[1], cols[2], cols[3], cols[4])
    assert dedup.size == 0 and dedup.cursor == 0 and dedup.index.live_frames == 0
    a = torch.as_tensor(np.asarray(cols[1]), device="cuda")   # device metadata is accepted
    dedup.store_many(cols[0], a, cols[2], cols[3], cols[4])
    full.store_many(np.stack(cols[0]), np.asarray(cols[1]), np.asarray(cols[2]),
                    np.stack(cols[3]), np.asarray(cols[4]))
    ti = torch.arange(12, device="cuda")
    s, s2 = (torch.empty((12,) + shape, dtype=torch.uint8, device="cuda") for _ in range(2))
    dedup.gather_into(ti, 12, s, s2, None, None, None)
    assert torch.equal(s, full.states[:12]) and torch.equal(s2, full.next_states[:12])
    assert torch.equal(dedup.actions[:12], full.actions[:12])


def test_store_many_pool_exhaustion_keeps_the_assigned_prefix(P):
    """when the frame pool runs out part-way through a batch, the
    transitions assigned so far are uploaded and the cursor advances past
    them before ConfigError propagates (device table == host index)."""
    from paper_1804_05834_b200.errors import ConfigError
    from paper_1804_05834_b200.frame_ring import FrameDedupMemory
    rng = np.random.default_rng(4)
    shape, cap = (6, 6, 4), 16
    # independent random stacks: 8 new frames per transition, pool of 3 x 8
    stream = [(rng.integers(0, 256, shape, dtype=np.uint8), 1, 0.5,
               rng.integers(0, 256, shape, dtype=np.uint8), False) for _ in range(5)]
    dedup = FrameDedupMemory(cap, shape, frame_capacity=24)
    cols = list(zip(*stream))
    with pytest.raises(ConfigError):
        dedup.store_many(cols[0], cols[1], cols[2], cols[3], cols[4])
    assert dedup.size == 3 and dedup.cursor == 3
    ti = torch.arange(3, device="cuda")
    s, s2 = (torch.empty((3,) + shape, dtype=torch.uint8, device="cuda") for _ in range(2))
    dedup.gather_into(ti, 3, s, s2, None, None, None)
    assert np.array_equal(s.cpu().numpy(), np.stack(cols[0][:3]))
    assert np.array_equal(s2.cpu().numpy(), np.stack(cols[3][:3]))
    with pytest.raises(NotImplementedError):
        dedup.fill_synthetic(0, 4)


@pytest.mark.parametrize("alpha", [0.6, 0.0])
def test_trainer_on_dedup_ring_matches_full_ring(P, alpha):
    """The Trainer's staged insert through the frame-deduplicated ring: the
    same records and parameters as the full-stack ring (the learner reads
    byte-identical batches)."""
    from tests.test_gpu_checkpoint import small_cfg
    runs = []
    for dedup in (False, True):
        sink = P.RecordCollector()
        tr = P.Trainer(small_cfg(P, max_steps=400, priority_alpha=alpha), sink=sink,
                       frame_dedup=dedup)
        tr.run()
        runs.append(([r.row() for r in sink.records], tr.online.flat_values.clone()))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("src_dedup", [True, False])
def test_resume_on_dedup_ring(P, tmp_path, src_dedup):
    """CYRL memory section from / into the frame-deduplicated ring: a run
    resumed on the dedup ring (from a dedup or a full-ring checkpoint)
    reproduces the uninterrupted run record for record."""
    import dataclasses
    from paper_1804_05834_b200.checkpoint import load_checkpoint
    from tests.test_gpu_checkpoint import small_cfg
    full_sink = P.RecordCollector()
    full = P.Trainer(small_cfg(P, max_steps=400, checkpoint_include_memory=True), sink=full_sink)
    full.run()
    sink_a = P.RecordCollector()
    P.Trainer(small_cfg(P, max_steps=200, checkpoint_include_memory=True), sink=sink_a,
              out_dir=tmp_path, frame_dedup=src_dedup).run()
    ck = load_checkpoint(tmp_path / "checkpoint_final.ckpt")
    ck.config = dataclasses.replace(ck.config, max_steps=400)
    sink_b = P.RecordCollector()
    resumed = P.Trainer.from_checkpoint(ck, sink=sink_b, frame_dedup=True)
    resumed.run()
    assert [r.row() for r in sink_a.records + sink_b.records] == [r.row() for r in full_sink.records]
    assert torch.equal(resumed.online.flat_values, full.online.flat_values)
