"""GPU parity of the replay side against the oracle and the reference's
golden vectors: frame ring fill/gather (bit-exact bytes), sum-tree nodes and
sampled indices (bit-exact), IS weights and alpha-power leaves (ULP bounds)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import deepq_oracle as O
from tests.helpers import ulp_diff

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def test_ring_fill_matches_host_hash_and_gather_is_exact(P):
    from paper_1804_05834_b200 import synth
    mem = P.ReplayMemory(300, (84, 84, 4))
    mem.fill_synthetic(11, 300)
    slots = np.array([0, 7, 299, 150, 7])
    assert np.array_equal(mem.states[slots].cpu().numpy(), synth.frames(11, 0, slots))
    assert np.array_equal(mem.next_states[slots].cpu().numpy(), synth.frames(11, 1, slots))
    b = mem._gather(slots, None, None)
    assert np.array_equal(b.states.cpu().numpy(), synth.frames(11, 0, slots))
    assert np.array_equal(b.next_states.cpu().numpy(), synth.frames(11, 1, slots))
    a, r, t = synth.metadata(11, 300)
    assert np.array_equal(b.actions.cpu().numpy(), a[slots])
    assert np.array_equal(b.rewards.cpu().numpy(), r[slots])
    assert np.array_equal(b.terminals.cpu().numpy(), t[slots])


def test_gather_generic_float_states(P):
    mem = P.ReplayMemory(5, (2, 2, 1), dtype=np.float32)
    for i in range(7):            # wraps: slots hold 5, 6, 2, 3, 4
        s = np.full((2, 2, 1), float(i), np.float32)
        mem.store(P.Transition(s, i % 3, float(i), s + 0.5, i == 4))
    assert mem.size == 5 and mem.cursor == 2
    got = sorted(float(mem.states[i, 0, 0, 0]) for i in range(5))
    assert got == [2.0, 3.0, 4.0, 5.0, 6.0]
    b = mem.sample_uniform(64, np.random.default_rng(0))
    idx = b.indices.cpu().numpy()
    assert np.array_equal(idx, np.random.default_rng(0).integers(0, 5, 64))
    st = b.states.cpu().numpy()[:, 0, 0, 0]
    assert np.array_equal(b.next_states.cpu().numpy()[:, 0, 0, 0], st + 0.5)
    assert np.all(b.weights.cpu().numpy() == 1.0)


def _device_tree(P, nodes: np.ndarray, cap: int):
    t = P.SumTree(cap)
    t.nodes.copy_(torch.as_tensor(nodes, device="cuda"))
    return t


def test_tree_golden_kat_and_random(P, golden):
    g = golden("tree")
    t = P.SumTree(4)
    for i, p in enumerate([1.0, 2.0, 3.0, 4.0]):
        t.set(i, p)
    assert np.array_equal(t.nodes.cpu().numpy(), g["kat_nodes"])
    assert np.array_equal(t.find(g["kat_q"]).cpu().numpy(), g["kat_idx"])
    for r in range(8):
        cap = int(g[f"rand{r}_cap"])
        t = P.SumTree(cap)
        t.set_many(np.arange(cap), g[f"rand{r}_pri"])
        assert np.array_equal(t.nodes.cpu().numpy(), g[f"rand{r}_nodes"])
        assert np.array_equal(t.find(g[f"rand{r}_q"]).cpu().numpy(), g[f"rand{r}_idx"])
    # 4000 sets with duplicates, in batch order: last write wins
    t = P.SumTree(1000)
    t.set_many(g["big_order"], g["big_vals"])
    assert np.array_equal(t.nodes.cpu().numpy(), g["big_nodes"])
    assert np.array_equal(t.find(g["big_q"]).cpu().numpy(), g["big_idx"])


def test_tree_errors(P):
    t = P.SumTree(4)
    with pytest.raises(ValueError):
        t.find([0.5])
    with pytest.raises(IndexError):
        t.set(4, 1.0)
    with pytest.raises(ValueError):
        t.set(0, -1.0)


def _per(P, cap=1000, beta_end=1000):
    cfg = P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1.0, beta_end))
    return P.PrioritizedReplay(cap, (1, 1, 1), cfg)


def test_per_against_reference_golden(P, golden):
    g = golden("per")
    mem = _per(P)
    z = np.zeros((1, 1, 1), np.uint8)
    mem.store_many(np.zeros((700, 1, 1, 1), np.uint8), np.arange(700) % 4, np.zeros(700),
                   np.zeros((700, 1, 1, 1), np.uint8), np.zeros(700, bool))
    mem.update_priorities(np.arange(700), g["td0"])
    nodes = mem.tree.nodes.cpu().numpy()
    base = mem.tree._leaf_base
    # leaves (|td|+eps)^alpha: device pow vs libm pow within 1 ulp
    assert ulp_diff(nodes[base:], g["nodes0"][base:]).max() <= 1
    # internal nodes are a pure function of the leaves: bit-exact given them
    ref = O.HeapTree(1000)
    ref.nodes[:] = nodes
    ref.rebuild()
    assert np.array_equal(ref.nodes, nodes)
    assert mem.max_priority == g["maxp0"]
    # teacher-force the reference tree so the sample comparison is exact
    mem.tree.nodes.copy_(torch.as_tensor(g["nodes0"], device="cuda"))
    for s in range(4):
        k = int(g[f"s{s}_k"])
        u = torch.as_tensor(g[f"s{s}_u"], device="cuda")
        beta = torch.full((1,), float(g[f"s{s}_beta"]), dtype=torch.float64, device="cuda")
        idx = torch.empty(k, dtype=torch.int64, device="cuda")
        prob = torch.empty(k, dtype=torch.float64, device="cuda")
        w = torch.empty(k, dtype=torch.float64, device="cuda")
        mem.sample_indices(u, k, beta, idx, prob, w, mem.tree._flags)
        assert np.array_equal(idx.cpu().numpy(), g[f"s{s}_idx"])
        assert np.array_equal(prob.cpu().numpy(), g[f"s{s}_prob"])
        assert ulp_diff(w.cpu().numpy(), g[f"s{s}_w"]).max() <= 4
        assert w.cpu().numpy().max() == 1.0
        mem.update_priorities(g[f"s{s}_upd_idx"], np.abs(g[f"s{s}_td"]))
        got = mem.tree.nodes.cpu().numpy()
        assert ulp_diff(got[base:], g[f"s{s}_nodes"][base:]).max() <= 1
        assert mem.max_priority == g[f"s{s}_maxp"]
        mem.tree.nodes.copy_(torch.as_tensor(g[f"s{s}_nodes"], device="cuda"))
    slot = mem.store(P.Transition(z, 1, 0.0, z, False))
    assert slot == g["store_slot"]
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got, g["store_nodes"]).max() <= 1
    mem.tree.nodes.copy_(torch.as_tensor(g["store_nodes"], device="cuda"))
    # out-of-range index mid-batch: earlier leaves written, then IndexError
    with pytest.raises(IndexError):
        mem.update_priorities(np.array([3, 5, 999, 7]), np.array([9.0, 8.0, 7.0, 6.0]))
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got, g["partial_after"]).max() <= 1
    assert mem.max_priority == g["partial_maxp"]


def test_sampler_at_1m_leaves_bit_exact(P):
    """1M-leaf tree (depth 20): device descent == oracle descent on the same
    nodes for 32 stratified and 1M random queries."""
    n = 1_000_000
    mem = P.PrioritizedReplay(n, (1, 1, 1))
    mem.memory._set_size(n)
    rng = np.random.default_rng(123)
    leaves = rng.random(n) ** 3 + 1e-6
    mem.tree.load_leaves(leaves)
    nodes = mem.tree.nodes.cpu().numpy()
    ref = O.HeapTree(n)
    ref.nodes[ref.base:ref.base + n] = leaves
    ref.rebuild()
    assert np.array_equal(ref.nodes, nodes)
    for k in (32, 4096):
        u = rng.random(k)
        b = mem.sample(k, 0.4, np.random.default_rng(5))
        ui = np.random.default_rng(5).random(k)
        idx, prob, w = O.per_indices(ref, n, k, 0.4, ui)
        assert np.array_equal(b.indices.cpu().numpy(), idx)
        assert np.array_equal(b.probabilities.cpu().numpy(), prob)
        assert ulp_diff(b.weights.cpu().numpy(), w).max() <= 4
        del u
    q = rng.random(n) * ref.total
    assert np.array_equal(mem.tree.find(q).cpu().numpy(), ref.descend(q))


def test_update_duplicates_last_wins_large_batch(P):
    n = 5000
    mem = _per(P, cap=n)
    mem.memory._set_size(n)
    mem.tree.load_leaves(np.ones(n))
    rng = np.random.default_rng(7)
    idx = rng.integers(0, n, size=3000)          # > 1024: several chunks, duplicates
    td = rng.random(3000) * 4
    mem.update_priorities(idx, td)
    ref = O.PerReplay(n, (1, 1, 1), 0.6, 0.01)
    ref.ring.size = n
    ref.tree.nodes[ref.tree.base:ref.tree.base + n] = 1.0
    ref.tree.rebuild()
    ref.update_priorities(idx, td)
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got[ref.tree.base:], ref.tree.nodes[ref.tree.base:]).max() <= 1
    chk = O.HeapTree(n)
    chk.nodes[:] = got
    chk.rebuild()
    assert np.array_equal(chk.nodes, got)
    assert mem.max_priority == ref.max_priority


def _bulk_case(P, n, k, seed):
    mem = _per(P, cap=n)
    mem.memory._set_size(n)
    mem.tree.load_leaves(np.ones(n))
    ref = O.PerReplay(n, (1, 1, 1), 0.6, 0.01)
    ref.ring.size = n
    ref.tree.nodes[ref.tree.base:ref.tree.base + n] = 1.0
    ref.tree.rebuild()
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, n, size=k)             # >= 4096: the multi-CTA bulk path
    td = rng.random(k) * 4
    return mem, ref, idx, td


def test_update_bulk_path_bit_exact_with_duplicates(P):
    mem, ref, idx, td = _bulk_case(P, n=50_000, k=40_000, seed=8)
    mem.update_priorities(idx, td)
    ref.update_priorities(idx, td)
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got[ref.tree.base:], ref.tree.nodes[ref.tree.base:]).max() <= 1
    chk = O.HeapTree(50_000)
    chk.nodes[:] = got
    chk.rebuild()
    assert np.array_equal(chk.nodes, got)            # every ancestor = sum of children
    assert mem.max_priority == ref.max_priority
    # a second bulk call reuses the scratch (winner table back at rest)
    idx2 = np.random.default_rng(9).integers(0, 50_000, size=8192)
    td2 = np.random.default_rng(10).random(8192)
    mem.update_priorities(idx2, td2)
    ref.update_priorities(idx2, td2)
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got[ref.tree.base:], ref.tree.nodes[ref.tree.base:]).max() <= 1


def test_update_bulk_path_partial_update_then_index_error(P):
    mem, ref, idx, td = _bulk_case(P, n=20_000, k=12_000, seed=11)
    idx[9000] = 20_000                                # out of range mid-batch
    max_before = mem.max_priority
    with pytest.raises(IndexError):
        mem.update_priorities(idx, td)
    with pytest.raises(IndexError):
        ref.update_priorities(idx, td)                # the reference writes [0, 9000) first
    got = mem.tree.nodes.cpu().numpy()
    assert ulp_diff(got[ref.tree.base:], ref.tree.nodes[ref.tree.base:]).max() <= 1
    assert mem.max_priority == max_before             # untouched on the raising call


@pytest.mark.parametrize("cap", [1000, 300_000, 1 << 20])
def test_sample_gather_equals_sample_then_gather(cap):
    """dqn_sample_gather (warp descent, eight levels per round trip, fused
    with the frame gather) against dqn_tree_sample + dqn_ring_gather at tree
    depths 10, 19 and 20: identical indices, probabilities, weights, bytes."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    from paper_1804_05834_b200 import _lib
    mem = P.PrioritizedReplay(cap, (16,), P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1, 10)))
    ring = mem.memory
    rng = np.random.default_rng(cap)
    ring.states.copy_(torch.as_tensor(rng.integers(0, 256, (cap, 16), dtype=np.uint8)))
    ring.next_states.copy_(torch.as_tensor(rng.integers(0, 256, (cap, 16), dtype=np.uint8)))
    ring.actions.copy_(torch.as_tensor(rng.integers(0, 4, cap)))
    ring.rewards.copy_(torch.as_tensor(rng.standard_normal(cap)))
    ring._set_size(cap)
    leaves = rng.random(cap) ** 3
    leaves[rng.integers(0, cap, cap // 10)] = 0.0
    mem.tree.load_leaves(leaves)
    k = 32
    u = torch.as_tensor(np.concatenate([rng.random(k), [0.55]]), device="cuda")
    outs = []
    for fused in (True, False):
        idx = torch.zeros(k, dtype=torch.int64, device="cuda")
        prob = torch.zeros(k, dtype=torch.float64, device="cuda")
        w = torch.zeros(k, dtype=torch.float64, device="cuda")
        x = torch.zeros((2 * k, 16), dtype=torch.uint8, device="cuda")
        a = torch.zeros(k, dtype=torch.int64, device="cuda")
        r = torch.zeros(k, dtype=torch.float64, device="cuda")
        t = torch.zeros(k, dtype=torch.bool, device="cuda")
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        st = _lib.stream_ptr()
        if fused:
            _lib.call("dqn_sample_gather", st, mem.tree.nodes.data_ptr(), mem.tree.depth,
                      ring._size_dev.data_ptr(), u.data_ptr(), k, u[k:].data_ptr(),
                      idx.data_ptr(), prob.data_ptr(), w.data_ptr(), fl.data_ptr(),
                      ring.states.data_ptr(), ring.next_states.data_ptr(), ring.slot_bytes,
                      ring.actions.data_ptr(), ring.rewards.data_ptr(), ring.terminals.data_ptr(),
                      x.data_ptr(), x[k:].data_ptr(), a.data_ptr(), r.data_ptr(), t.data_ptr())
        else:
            mem.sample_indices(u[:k], k, u[k:], idx, prob, w, fl)
            ring.gather_into(idx, k, x[:k], x[k:], a, r, t)
        torch.cuda.synchronize()
        assert fl.item() == 0
        outs.append((idx, prob, w, x, a, r, t))
    for p_, q_ in zip(*outs):
        assert torch.equal(p_, q_)
    assert mem.tree.depth >= 10
