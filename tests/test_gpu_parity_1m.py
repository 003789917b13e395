"""Full one-update parity at the true 1M capacity (cfg2-cfg4: a 56 GB uint8
ring in HBM), against a virtual-ring oracle: the
oracle's ring generates the sampled transitions' frames lazily from the same
splitmix64 counter hash the device fill uses (synth.py), so the oracle
update runs at 1M without the reference's 226 GB float32 ring.  Reference:
replay.py:104-124,215-241, agent.py:91-132.

Checked per config: sampled indices bit-exact; targets, TD errors, losses
<= 1e-5; every weight tensor and the RMSprop accumulators <= 1e-3
(north_star; observed ~1e-6); for PER the tree after the priority update
(leaves <= 1e-5 norm-wise, internal nodes exact given the leaves) and the
max priority.
"""

from __future__ import annotations

import gc

import numpy as np
import pytest

from oracle import deepq_oracle as O
from paper_1804_05834_b200 import synth
from tests.helpers import ATARI, follow_device_relu_kinks, rel_norm

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N = 1_000_000
SEED = 3


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


@pytest.fixture(autouse=True)
def _free_rings(P):
    """Each case holds a 56 GB ring: drop every cached learner plan (they
    reference their memories) before and after, even when a case fails."""
    def clear():
        P.agent._PLANS.clear()
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    clear()
    yield
    clear()


class VirtualRing(O.Ring):
    """Oracle ring of ``n`` synthetic transitions whose frames are produced on
    demand (same bytes as the device's dqn_ring_fill_hash); metadata arrays
    are materialised (24 MB at 1M)."""

    def __init__(self, n: int, seed: int):
        self.capacity, self.state_shape = n, ATARI
        self.seed = seed
        self.actions, self.rewards, self.terminals = synth.metadata(seed, n)
        self.cursor, self.size = 0, n

    def gather(self, idx, prob, w):
        idx = np.asarray(idx, dtype=np.int64)
        s = synth.frames(self.seed, 0, idx)
        s2 = synth.frames(self.seed, 1, idx)
        return O.Batch(self.lift(s), self.actions[idx], self.rewards[idx].copy(),
                       self.lift(s2), self.terminals[idx], idx, prob, w)


CFGS = {
    "cfg2": dict(dueling=False, double=True, per=False),
    "cfg3": dict(dueling=False, double=True, per=True),
    "cfg4": dict(dueling=True, double=True, per=True),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_one_update_at_1m(P, name):
    kw = CFGS[name]
    cfg = P.RunConfig(double=kw["double"], dueling=kw["dueling"], batch_size=32,
                      beta_end_step=50_000_000, priority_alpha=0.6 if kw["per"] else 0.0)
    on = P.build_network("atari", ATARI, 4, kw["dueling"])
    tg = P.build_network("atari", ATARI, 4, kw["dueling"])
    P.init_params(on, 1)
    P.init_params(tg, 2)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    if kw["per"]:
        mem = P.PrioritizedReplay(N, ATARI, P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    else:
        mem = P.ReplayMemory(N, ATARI)
    mem.fill_synthetic(SEED, N)

    o_on = O.QNet(O.ATARI_TRUNK, ATARI, 4, kw["dueling"])
    o_tg = O.QNet(O.ATARI_TRUNK, ATARI, 4, kw["dueling"])
    o_on.init(1)
    o_tg.init(2)
    o_opt = O.RmsPropState(o_on)
    ring = VirtualRing(N, SEED)
    if kw["per"]:
        o_mem = O.PerReplay.__new__(O.PerReplay)
        o_mem.ring = ring
        o_mem.tree = O.HeapTree(N)
        o_mem.tree.nodes[:] = mem.tree.nodes.cpu().numpy()      # identical starting tree
        o_mem.alpha, o_mem.eps = 0.6, 0.01
        o_mem.beta_sched = (0.4, 1.0, 50_000_000)
        o_mem.max_priority = float(mem.max_priority)
    else:
        o_mem = ring
    o_cfg = O.LearnCfg(double=kw["double"])

    # the ring bytes themselves at a few slots (device fill == host hash)
    probe = np.array([0, 1, 4093, 500_000, N - 1])
    got = torch.empty((len(probe),) + ATARI, dtype=torch.uint8, device="cuda")
    mem_ring = mem.memory if kw["per"] else mem
    got.copy_(mem_ring.states[torch.as_tensor(probe, device="cuda")])
    assert np.array_equal(got.cpu().numpy(), synth.frames(SEED, 0, probe))

    step = 1000
    res = P.learn_step(on, tg, mem, opt, cfg, step, np.random.default_rng(77))
    plan = next(p for p in P.agent._PLANS.values() if p.online is on)
    # ReLU kinks within fp32 rounding resolved as the device did (helpers)
    kinks = follow_device_relu_kinks(o_on, [a.cpu().numpy() for a in plan.on_bind.act])
    ores = O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, step, rng=np.random.default_rng(77))
    if kinks:
        print(f"{name}: ReLU kinks resolved as on the device: {kinks}")

    assert np.array_equal(plan.last_indices().cpu().numpy(), ores["batch"].indices)
    assert rel_norm(res.targets, ores["targets"]) < 1e-5
    assert rel_norm(res.td_errors, ores["td_errors"]) < 1e-5
    assert rel_norm(res.losses, ores["losses"]) < 1e-5
    worst = 0.0
    for n, t in on.named_tensors():
        d = rel_norm(t.values.cpu().numpy(), o_on.params[n])
        worst = max(worst, d)
        assert d < 1e-3, (n, d)
        a = rel_norm(opt.acc[n].cpu().numpy(), o_opt.acc[n])
        assert a < 1e-3, (n, a)
    if kw["per"]:
        nodes = mem.tree.nodes.cpu().numpy()
        assert rel_norm(nodes, o_mem.tree.nodes) < 1e-5
        chk = O.HeapTree(N)
        chk.nodes[:] = nodes
        chk.rebuild()
        assert np.array_equal(chk.nodes, nodes)
        touched = np.unique(ores["batch"].indices) + o_mem.tree.base
        assert rel_norm(nodes[touched], o_mem.tree.nodes[touched]) < 1e-5
        assert abs(mem.max_priority - o_mem.max_priority) <= 1e-12 * o_mem.max_priority
    print(f"{name} @1M: worst weight rel-norm {worst:.2e}, "
          f"TD rel {rel_norm(res.td_errors, ores['td_errors']):.2e}")
