"""Data-parallel learner (cfg5) on CPU: world_size-2 gloo processes run the
sharded protocol of paper_1804_05834_b200/dp.py with an oracle compute
backend; the result must equal a single-process restatement written here
independently: N oracle sum-tree shards + the global stratification rule +
one learner at the global batch K = k * N (the reference's own cfg5
comparator).  Indices and IS weights bit-exact, TD errors
and weights norm-wise."""

from __future__ import annotations

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import deepq_oracle as O

WORLD = 2
K_PER = 8
CAP = 64
SHAPE = (6, 6, 2)
TRUNK = [("conv", 2, 2, 2), ("relu",), ("fc", 8), ("relu",)]
ALPHA, EPS = 0.6, 0.01
STEPS = 3


def global_data():
    rng = np.random.default_rng(2024)
    S = rng.random((CAP,) + SHAPE).astype(np.float32)
    S2 = rng.random((CAP,) + SHAPE).astype(np.float32)
    A = rng.integers(0, 3, CAP).astype(np.int64)
    R = rng.choice([-1.0, 0.0, 1.0], CAP)
    T = rng.random(CAP) < 0.2
    TD = np.abs(rng.standard_normal(CAP)) * 2
    return S, S2, A, R, T, TD


def make_shard(rank, world):
    S, S2, A, R, T, TD = global_data()
    glob = np.arange(rank, CAP, world)
    mem = O.PerReplay(len(glob), SHAPE, ALPHA, EPS, float_states=True)
    for g in glob:
        mem.store(S[g], A[g], R[g], S2[g], T[g])
    mem.update_priorities(np.arange(len(glob)), TD[glob])
    return mem


def make_net(seed=5):
    on = O.QNet(TRUNK, SHAPE, 3, True)
    tg = O.QNet(TRUNK, SHAPE, 3, True)
    on.init(seed)
    tg.init(seed + 1)
    return on, tg, O.RmsPropState(on)


class OracleBackend:
    """dp.Backend over the CPU oracle (test infrastructure)."""

    def __init__(self, rank, world):
        self.mem = make_shard(rank, world)
        self.on, self.tg, self.opt = make_net()
        self.names = list(self.on.grads)
        self.cfg = O.LearnCfg(batch_size=K_PER)

    def shard_total(self):
        return self.mem.tree.total

    def shard_size(self):
        return self.mem.size

    def max_priority(self):
        return self.mem.max_priority

    def descend(self, q_local):
        idx = self.mem.tree.descend(q_local)
        return idx, self.mem.tree.leaves()[idx].copy()

    def pack(self, idx):
        ring = self.mem.ring
        return {"s": torch.as_tensor(ring.states[idx]), "s2": torch.as_tensor(ring.next_states[idx]),
                "a": torch.as_tensor(ring.actions[idx]), "r": torch.as_tensor(ring.rewards[idx]),
                "t": torch.as_tensor(ring.terminals[idx].astype(np.uint8))}

    def learn(self, batch, weights):
        b = O.Batch(batch["s"].numpy(), batch["a"].numpy(), batch["r"].numpy().copy(),
                    batch["s2"].numpy(), batch["t"].numpy().astype(bool), None, None,
                    np.asarray(weights))
        self.on.zero_grads()
        out = O.learn_on_batch(self.on, self.tg, b, self.cfg)
        self._flat = torch.as_tensor(np.concatenate([self.on.grads[n].ravel() for n in self.names]))
        return out["td_errors"]

    def grads(self):
        return self._flat

    def apply_update(self, idx, td, max_p):
        self.mem.update_priorities(idx, td)
        self.mem.max_priority = max_p

    def optimizer_step(self):
        off = 0
        flat = self._flat.numpy()
        for n in self.names:
            g = self.on.grads[n]
            g[...] = flat[off:off + g.size].reshape(g.shape)
            off += g.size
        self.opt.step()


def worker(rank, world, port, out):
    from paper_1804_05834_b200 import dp
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    be = OracleBackend(rank, world)
    learner = dp.DataParallelLearner(be, K_PER, ALPHA, EPS, "cpu")
    rng = np.random.default_rng(99)
    res = []
    for step in range(STEPS):
        r = learner.step(rng.random(K_PER * world), 0.4 + 0.1 * step)
        res.append((r.indices, r.weights, r.td_errors))
    out[rank] = {"res": res, "params": {k: v.copy() for k, v in be.on.params.items()},
                 "leaves": be.mem.tree.leaves().copy(), "maxp": be.mem.max_priority}
    dist.barrier()
    dist.destroy_process_group()


def restatement(world):
    """Single process: N shards, global stratified sampling, batch K."""
    shards = [make_shard(r, world) for r in range(world)]
    on, tg, opt = make_net()
    K = K_PER * world
    rng = np.random.default_rng(99)
    max_p = max(m.max_priority for m in shards)
    res = []
    for step in range(STEPS):
        u, beta = rng.random(K), 0.4 + 0.1 * step
        totals = [m.tree.total for m in shards]
        T = 0.0
        for t in totals:
            T = T + t
        q = np.minimum(np.maximum((np.arange(K) + u) * (T / K), 1e-300), np.nextafter(T, 0))
        owner, loc, leaf = [], [], []
        for qj in q:
            base = 0.0
            for r, t in enumerate(totals):
                if qj <= base + t or r == world - 1:
                    i = int(shards[r].tree.descend([qj - base])[0])
                    owner.append(r)
                    loc.append(i)
                    leaf.append(shards[r].tree.leaves()[i])
                    break
                base = base + t
        owner, loc, leaf = np.array(owner), np.array(loc), np.array(leaf)
        prob = leaf / T
        w = np.power(sum(m.size for m in shards) * prob, -beta)
        w = w / w.max()
        rings = [m.ring for m in shards]
        b = O.Batch(np.stack([rings[o].states[i] for o, i in zip(owner, loc)]),
                    np.array([rings[o].actions[i] for o, i in zip(owner, loc)]),
                    np.array([rings[o].rewards[i] for o, i in zip(owner, loc)]),
                    np.stack([rings[o].next_states[i] for o, i in zip(owner, loc)]),
                    np.array([rings[o].terminals[i] for o, i in zip(owner, loc)]),
                    None, prob, w)
        on.zero_grads()
        out = O.learn_on_batch(on, tg, b, O.LearnCfg(batch_size=K))
        td = out["td_errors"]
        max_p = max(max_p, float((np.abs(td) + EPS).max()))
        for r in range(world):
            sel = owner == r
            if sel.any():
                shards[r].update_priorities(loc[sel], np.abs(td[sel]))
            shards[r].max_priority = max_p
        opt.step()
        res.append((loc * world + owner, w, td))
    return res, on, shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def dp_run():
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(worker, args=(WORLD, _free_port(), out), nprocs=WORLD, join=True,
                       start_method="spawn")
    return dict(out)


def test_ranks_agree_and_match_restatement(dp_run):
    ref, on, shards = restatement(WORLD)
    for r in range(WORLD):
        got = dp_run[r]
        for (gi, gw, gt), (ri, rw, rt) in zip(got["res"], ref):
            assert np.array_equal(gi, ri)                 # sampled transitions: bit-exact
            assert np.array_equal(gw, rw)                 # IS weights: same numpy ops
            assert np.max(np.abs(gt - rt)) <= 1e-6 * max(1.0, np.max(np.abs(rt)))
        for k, v in got["params"].items():
            assert np.linalg.norm(v - on.params[k]) <= 1e-5 * max(1e-12, np.linalg.norm(on.params[k])), k
        leaves = got["leaves"]
        # leaves are (|delta|+eps)^alpha of fp32-network deltas (batch k vs K rows)
        assert np.allclose(leaves, shards[r].tree.leaves(), rtol=1e-6, atol=0)
        assert got["maxp"] == pytest.approx(shards[r].max_priority, rel=1e-12)
    # both ranks applied identical updates
    for k in dp_run[0]["params"]:
        assert np.array_equal(dp_run[0]["params"][k], dp_run[1]["params"][k])


def test_sharding_math_units():
    from paper_1804_05834_b200 import dp
    rank, loc = dp.shard_of(np.arange(10), 4)
    assert list(rank) == [0, 1, 2, 3, 0, 1, 2, 3, 0, 1]
    assert np.array_equal(dp.global_slot(rank, loc, 4), np.arange(10))
    owner, ql, T = dp.stratified_queries(np.array([1.0, 0.0, 3.0]), 8, np.full(8, 0.5))
    assert T == 4.0 and set(owner) <= {0, 2} and np.all(ql > 0)
    plan = dp.exchange_plan(np.array([0, 1, 1, 0, 1, 1, 0, 0]), 1, 2, 4)
    # rank 1 owns strata 1,2 (learned by rank 0) and 4,5 (its own); it learns
    # strata 4..7 whose owners are 1,1,0,0
    assert plan.send_counts == [2, 2] and plan.recv_counts == [2, 2]
    assert plan.recv_order.tolist() == [2, 3, 0, 1]
    assert sorted(plan.recv_order.tolist()) == [0, 1, 2, 3]
