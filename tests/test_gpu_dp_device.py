"""The device data-parallel learner (dp.DeviceDataParallelLearner,
csrc/dp.cu).  One GPU is available, so:

* world size 1 over NCCL must reproduce ``learn_step`` bit for bit (same
  queries, descent, weights, update), with the whole global update captured
  as one CUDA graph, collectives included;
* the multi-shard steps are checked kernel by kernel against the host
  restatement in dp.py (``stratified_queries``, ``is_weights``, owner-side
  ``update_priorities``) on several shards that live on this one GPU --
  routing over N shard totals, owner descent into the (index, leaf) table,
  IS weights over the union, the peer-ring gather through a table of ring
  pointers, and the owned-strata compaction + masked priority update.
No kernel here waits on another rank.
"""

from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    import paper_1804_05834_b200 as P
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield P


def _learner(P, seed=7, cap=256, shareable=False):
    cfg = P.RunConfig(double=True, dueling=True, batch_size=32, beta_end_step=1000,
                      priority_alpha=0.6)
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 1)
    P.init_params(tg, 2)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()),
                              shareable=shareable)
    mem.fill_synthetic(seed, cap)
    return on, tg, mem, opt, cfg


def test_device_dp_world1_equals_learn_step(P):
    from paper_1804_05834_b200 import dp
    on, tg, mem, opt, cfg = _learner(P)
    on2, tg2, mem2, opt2, cfg2 = _learner(P, shareable=True)
    learner = dp.DeviceDataParallelLearner(on2, tg2, mem2, opt2, cfg2)
    rng_a, rng_b = np.random.default_rng(5), np.random.default_rng(5)
    for s in range(5):                         # eager, capture, then graph replays
        res = P.learn_step(on, tg, mem, opt, cfg, 100 + s, rng_a)
        plan = next(p for p in P.agent._PLANS.values() if p.online is on)
        r = learner.step(rng_b.random(32), mem2.beta(100 + s))
        assert np.array_equal(r.indices, plan.idx.cpu().numpy())
        assert np.array_equal(r.weights, plan.w.cpu().numpy())
        assert np.array_equal(r.td_errors, res.td_errors)
    assert learner.graph_exec is not None
    assert torch.equal(on.flat_values, on2.flat_values)
    assert torch.equal(opt.flat_acc, opt2.flat_acc)
    assert torch.equal(mem.tree.nodes, mem2.tree.nodes)
    assert mem.max_priority == mem2.max_priority
    learner.close()


def _trees(P, n, cap, seed):
    rng = np.random.default_rng(seed)
    trees = []
    for r in range(n):
        t = P.SumTree(cap)
        pri = rng.random(cap) * (r + 1) * 3.0
        if r == 1:
            pri[:] = 0.0                      # an empty shard is skipped by routing
        t.load_leaves(pri)
        trees.append(t)
    return trees


def test_route_descend_weights_match_host_restatement(P):
    from paper_1804_05834_b200 import _lib, dp
    N, k, cap = 4, 32, 1000
    K = N * k
    trees = _trees(P, N, cap, 3)
    sizes = [cap, cap, 700, 999]
    maxp = [1.5, 2.0, 0.5, 3.25]
    info = torch.tensor([[t.total, s, m] for t, s, m in zip(trees, sizes, maxp)],
                        dtype=torch.float64, device="cuda").reshape(-1)
    u = np.random.default_rng(9).random(K)
    ud = torch.as_tensor(u, device="cuda")
    owner = torch.zeros(K, dtype=torch.int64, device="cuda")
    ql = torch.zeros(K, dtype=torch.float64, device="cuda")
    sums = torch.zeros(3, dtype=torch.float64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    _lib.call("dqn_dp_route", st, info.data_ptr(), N, ud.data_ptr(), K, owner.data_ptr(),
              ql.data_ptr(), sums.data_ptr(), flags.data_ptr(), None, 0, 0, None)
    totals = np.array([t.total for t in trees])
    want_owner, want_q, T = dp.stratified_queries(totals, K, u)
    assert np.array_equal(owner.cpu().numpy(), want_owner)
    assert np.array_equal(ql.cpu().numpy(), want_q)
    assert sums.cpu().numpy().tolist() == [T, float(sum(sizes)), max(maxp)]
    assert 1 not in set(want_owner.tolist())
    # each "rank" descends its own queries; the SUM of the tables is the table
    table = torch.zeros(2 * K, dtype=torch.float64, device="cuda")
    part = torch.zeros(2 * K, dtype=torch.float64, device="cuda")
    for r, t in enumerate(trees):
        _lib.call("dqn_dp_descend", st, t.nodes.data_ptr(), t.depth, owner.data_ptr(),
                  ql.data_ptr(), K, r, part.data_ptr())
        table += part
    tab = table.cpu().numpy().reshape(K, 2)
    # the fused route + descent gives each rank its part of the same table
    fused = torch.zeros(2 * K, dtype=torch.float64, device="cuda")
    for r, t in enumerate(trees):
        _lib.call("dqn_dp_route", st, info.data_ptr(), N, ud.data_ptr(), K, owner.data_ptr(),
                  ql.data_ptr(), sums.data_ptr(), flags.data_ptr(), t.nodes.data_ptr(), t.depth,
                  r, part.data_ptr())
        fused += part
    assert torch.equal(fused, table)
    for r, t in enumerate(trees):
        m = want_owner == r
        if m.any():
            idx = t.find(want_q[m]).cpu().numpy()
            assert np.array_equal(tab[m, 0].astype(np.int64), idx)
            assert np.array_equal(tab[m, 1], t.leaves().cpu().numpy()[idx])
    # IS weights over the union (numpy pow vs device pow: <= 1 ulp)
    beta = torch.full((1,), 0.55, dtype=torch.float64, device="cuda")
    lidx = torch.zeros(K, dtype=torch.int64, device="cuda")
    w_all = torch.zeros(K, dtype=torch.float64, device="cuda")
    w_mine = torch.zeros(k, dtype=torch.float64, device="cuda")
    for rank in range(N):
        _lib.call("dqn_dp_weights", st, table.data_ptr(), sums.data_ptr(), beta.data_ptr(), K, k,
                  rank, lidx.data_ptr(), w_all.data_ptr(), w_mine.data_ptr())
        _, want_w = dp.is_weights(tab[:, 1], T, sum(sizes), 0.55)
        np.testing.assert_array_max_ulp(w_all.cpu().numpy(), want_w, maxulp=2)
        assert np.array_equal(w_mine.cpu().numpy(), w_all.cpu().numpy()[rank * k:(rank + 1) * k])
        assert np.array_equal(lidx.cpu().numpy(), tab[:, 0].astype(np.int64))


def test_peer_ring_gather_from_several_shards(P):
    from paper_1804_05834_b200 import _lib
    from paper_1804_05834_b200.dp import _PeerRing, _RING_FIELDS
    N, k, cap = 3, 8, 50
    K = N * k
    rings = []
    for r in range(N):
        m = P.ReplayMemory(cap, (84, 84, 4), shareable=(r == 0))
        m.fill_synthetic(20 + r, cap)
        rings.append(m)
    S = _PeerRing.struct()
    tab = (S * N)(*[S(*[getattr(m, f).data_ptr() for f in _RING_FIELDS]) for m in rings])
    dtab = torch.frombuffer(bytearray(bytes(tab)), dtype=torch.uint8).to("cuda")
    rng = np.random.default_rng(4)
    owner = rng.integers(0, N, K)
    local = rng.integers(0, cap, K)
    od = torch.as_tensor(owner, device="cuda")
    table = torch.zeros(2 * K, dtype=torch.float64, device="cuda")
    table[0::2] = torch.as_tensor(local.astype(np.float64), device="cuda")
    table[1::2] = 1.0
    sums = torch.tensor([float(K), 100.0, 0.0], dtype=torch.float64, device="cuda")
    beta = torch.full((1,), 0.5, dtype=torch.float64, device="cuda")
    for rank in range(N):
        x = torch.zeros((2 * k, 84, 84, 4), dtype=torch.uint8, device="cuda")
        a = torch.zeros(k, dtype=torch.int64, device="cuda")
        rw = torch.zeros(k, dtype=torch.float64, device="cuda")
        t = torch.zeros(k, dtype=torch.bool, device="cuda")
        lidx = torch.zeros(K, dtype=torch.int64, device="cuda")
        w_all = torch.zeros(K, dtype=torch.float64, device="cuda")
        w_mine = torch.zeros(k, dtype=torch.float64, device="cuda")
        _lib.call("dqn_dp_gather", _lib.stream_ptr(), dtab.data_ptr(), od.data_ptr(),
                  table.data_ptr(), k, rank, rings[0].slot_bytes, x.data_ptr(), a.data_ptr(),
                  rw.data_ptr(), t.data_ptr(), sums.data_ptr(), beta.data_ptr(), K,
                  lidx.data_ptr(), w_all.data_ptr(), w_mine.data_ptr())
        assert np.array_equal(lidx.cpu().numpy(), local)
        assert torch.all(w_all == 1.0) and torch.all(w_mine == 1.0)   # equal leaves
        for b in range(k):
            j = rank * k + b
            m, i = rings[owner[j]], int(local[j])
            assert torch.equal(x[b], m.states[i]) and torch.equal(x[k + b], m.next_states[i])
            assert a[b].item() == m.actions[i].item() and rw[b].item() == m.rewards[i].item()
            assert t[b].item() == m.terminals[i].item()


def test_owned_strata_update_matches_host_update_priorities(P):
    from paper_1804_05834_b200 import _lib
    N, k, cap = 4, 32, 300
    K = N * k
    rng = np.random.default_rng(6)
    owner = rng.integers(0, N, K)
    local = rng.integers(0, cap, K)
    local[5] = local[9]                          # duplicates: last write wins in batch order
    owner[5] = owner[9]
    td = rng.standard_normal(K)
    st = _lib.stream_ptr()
    od, ld, tdd = (torch.as_tensor(v, device="cuda") for v in (owner, local, td))
    for rank in range(N):
        mem = P.PrioritizedReplay(cap, (4,), P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1, 10)),
                                  dtype=np.float32)
        mem.memory._set_size(cap)
        ref = P.PrioritizedReplay(cap, (4,), P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1, 10)),
                                  dtype=np.float32)
        ref.memory._set_size(cap)
        base = rng.random(cap)
        mem.tree.load_leaves(base)
        ref.tree.load_leaves(base)
        idx_c = torch.zeros(K, dtype=torch.int64, device="cuda")
        td_c = torch.zeros(K, dtype=torch.float64, device="cuda")
        n_c = torch.zeros(1, dtype=torch.int32, device="cuda")
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("dqn_dp_owned", st, od.data_ptr(), ld.data_ptr(), tdd.data_ptr(), K, rank, 0.01,
                  idx_c.data_ptr(), td_c.data_ptr(), n_c.data_ptr(), mem._max_p.data_ptr(),
                  fl.data_ptr(), None)
        _lib.call("dqn_tree_update_n", st, mem.tree.nodes.data_ptr(), mem.tree.depth,
                  mem.memory._size_dev.data_ptr(), idx_c.data_ptr(), td_c.data_ptr(), K,
                  n_c.data_ptr(), 0.6, 0.01, None, fl.data_ptr())
        m = owner == rank
        assert n_c.item() == int(m.sum())
        ref.update_priorities(local[m], td[m])        # owner's call, global batch order
        assert torch.equal(mem.tree.nodes, ref.tree.nodes)
        assert mem.max_priority == max(1.0, float((np.abs(td) + 0.01).max()))
        assert fl.item() == 0


class _Hub:
    """Host-side collectives for ranks that are threads of this process: each
    rank synchronises its stream, posts its buffer, and copies the combined
    result once every rank has posted.  Kernels never wait on another rank."""

    def __init__(self, n):
        import threading
        self.n = n
        self.lock = threading.Lock()
        self.barriers = {}
        self.slots = {}

    def barrier(self, name):
        import threading
        with self.lock:
            if name not in self.barriers:
                self.barriers[name] = threading.Barrier(self.n)
            return self.barriers[name]


class _EmuComm:
    def __init__(self, hub, rank, name):
        self.hub, self.rank, self.name = hub, rank, name

    def _exchange(self, t):
        torch.cuda.current_stream().synchronize()
        self.hub.slots[(self.name, self.rank)] = t.detach().clone()
        b = self.hub.barrier(self.name)
        b.wait()
        vals = [self.hub.slots[(self.name, r)] for r in range(self.hub.n)]
        b.wait()
        return vals

    def all_gather(self, send, recv, stream):
        recv.copy_(torch.cat([v.reshape(-1) for v in self._exchange(send)]))
        torch.cuda.current_stream().synchronize()

    def all_reduce(self, t, op, stream, out=None):
        from paper_1804_05834_b200 import nccl
        vals = self._exchange(t)
        acc = vals[0].clone()
        for v in vals[1:]:
            acc = acc + v if op == nccl.NCCL_SUM else torch.maximum(acc, v)
        (t if out is None else out).copy_(acc)
        torch.cuda.current_stream().synchronize()

    def close(self):
        pass


def test_emulated_world2_equals_global_batch_update(P, monkeypatch):
    """Two ranks as threads on this GPU, collectives emulated on the host:
    both ranks agree on the sampled strata, weights and TD errors; the summed
    per-rank gradients equal the gradient of ONE batch-64 update over the
    same transitions and weights (the loss is a sum); each shard's tree gets
    exactly its owned strata in global batch order; max_priority becomes the
    global running max on every shard."""
    import threading
    from paper_1804_05834_b200 import agent, dp
    from tests.helpers import rel_norm
    monkeypatch.setattr(agent, "USE_GRAPH", False)
    N, k, cap = 2, 32, 200
    K = N * k
    hub = _Hub(N)
    shards, nets, learners = [], [], []
    for r in range(N):
        on, tg, mem, opt, cfg = _learner(P, seed=40 + r, cap=cap)
        shards.append(mem)
        nets.append((on, tg, opt, cfg))
    mp0 = [m.max_priority for m in shards]
    before = [m.tree.nodes.clone() for m in shards]
    for r in range(N):
        names = iter(["main", "td"])
        on, tg, opt, cfg = nets[r]
        opt.enqueue_apply = lambda flags: None          # keep the reduced gradients
        learners.append(dp.DeviceDataParallelLearner(
            on, tg, shards[r], opt, cfg,
            _emulated=(r, N, lambda r=r, names=names: _EmuComm(hub, r, next(names)), shards)))
    u = np.random.default_rng(11).random(K)
    out, errs = [None] * N, []

    def run(r):
        try:
            out[r] = learners[r].step(u, 0.7)
        except Exception as e:          # pragma: no cover - surfaced below
            errs.append(e)
    th = [threading.Thread(target=run, args=(r,)) for r in range(N)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    a, b = out
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.owner, b.owner)
    assert np.array_equal(a.weights, b.weights) and np.array_equal(a.td_errors, b.td_errors)
    assert set(a.owner.tolist()) == {0, 1}
    g = [n[0].flat_grads.clone() for n in nets]
    assert torch.equal(g[0], g[1])
    # the same transitions and weights through one batch-64 update
    cfg64 = P.RunConfig(double=True, dueling=True, batch_size=K, beta_end_step=1000)
    on64 = P.build_network("atari", (84, 84, 4), 4, True)
    tg64 = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on64, 1)
    P.init_params(tg64, 2)
    opt64 = P.RmsProp(on64)
    plan = agent._StepPlan(on64, tg64, shards[0], opt64, cfg64)
    local = a.indices // N
    for j in range(K):
        m = shards[int(a.owner[j])].memory
        plan.x[j].copy_(m.states[local[j]])
        plan.x[K + j].copy_(m.next_states[local[j]])
        plan.a[j] = m.actions[local[j]]
        plan.r[j] = m.rewards[local[j]]
        plan.t[j] = m.terminals[local[j]]
    plan.w.copy_(torch.as_tensor(a.weights))
    plan.enqueue_learn(priorities=False)
    torch.cuda.synchronize()
    td64 = plan.d_out[K:2 * K].cpu().numpy()
    assert rel_norm(a.td_errors, td64) < 1e-5
    assert rel_norm(g[0].cpu().numpy(), on64.flat_grads.cpu().numpy()) < 1e-5
    # owner-side priority updates in global batch order
    for r in range(N):
        ref = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1, 10)))
        ref.memory._set_size(cap)
        ref.tree.nodes.copy_(before[r])
        m = a.owner == r
        ref.update_priorities(local[m], a.td_errors[m])
        assert torch.equal(shards[r].tree.nodes, ref.tree.nodes)
    want_max = max(max(mp0), float((np.abs(a.td_errors) + 0.01).max()))
    assert [s.max_priority for s in shards] == [want_max] * N
