"""Pin the CPU oracle to the reference: golden fixtures made by the
unmodified reference (tests/golden/make_golden.py), plus a live comparison
when /root/reference is mounted.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import deepq_oracle as O
from tests.helpers import oracle_learner, rel_norm

# fp32 BLAS results differ in the last bits across CPUs (OpenBLAS kernel
# choice); network-derived fields are compared norm-wise at this tolerance.
NET_TOL = 1e-4


def test_tree_kat_and_random(golden):
    g = golden("tree")
    t = O.HeapTree(4)
    for i, p in enumerate([1.0, 2.0, 3.0, 4.0]):
        t.put(i, p)
    assert np.array_equal(t.nodes, g["kat_nodes"])
    assert np.array_equal(t.descend(g["kat_q"]), g["kat_idx"])
    assert t.descend([6.5])[0] == 3
    for r in range(8):
        cap = int(g[f"rand{r}_cap"])
        t = O.HeapTree(cap)
        for i, p in enumerate(g[f"rand{r}_pri"]):
            t.put(i, float(p))
        assert np.array_equal(t.nodes, g[f"rand{r}_nodes"])
        assert np.array_equal(t.descend(g[f"rand{r}_q"]), g[f"rand{r}_idx"])


def test_tree_rebuild_equals_sequential_sets(golden):
    g = golden("tree")
    t = O.HeapTree(1000)
    for i, v in zip(g["big_order"], g["big_vals"]):
        t.put(int(i), float(v))
    assert np.array_equal(t.nodes, g["big_nodes"])
    t2 = O.HeapTree(1000)
    last = {}
    for i, v in zip(g["big_order"], g["big_vals"]):
        last[int(i)] = float(v)
    for i, v in last.items():
        t2.nodes[t2.base + i] = v
    t2.rebuild()
    assert np.array_equal(t2.nodes, g["big_nodes"])     # order-free, bit-exact
    assert np.array_equal(t2.descend(g["big_q"]), g["big_idx"])


def test_per_sample_update_store_partial(golden):
    g = golden("per")
    mem = O.PerReplay(1000, (1, 1, 1), 0.6, 0.01, (0.4, 1.0, 1000))
    z = np.zeros((1, 1, 1), np.uint8)
    for i in range(700):
        mem.store(z, i % 4, 0.0, z, False)
    mem.update_priorities(np.arange(700), g["td0"])
    assert np.array_equal(mem.tree.nodes, g["nodes0"])
    assert mem.max_priority == g["maxp0"]
    for s in range(4):
        k = int(g[f"s{s}_k"])
        idx, prob, w = O.per_indices(mem.tree, mem.size, k, float(g[f"s{s}_beta"]), g[f"s{s}_u"])
        assert np.array_equal(idx, g[f"s{s}_idx"])
        assert np.array_equal(prob, g[f"s{s}_prob"])
        # numpy's vectorised pow may differ from another CPU's by 1 ulp
        assert np.max(np.abs(w - g[f"s{s}_w"]) / g[f"s{s}_w"]) < 1e-15
        mem.update_priorities(g[f"s{s}_upd_idx"], np.abs(g[f"s{s}_td"]))
        assert np.array_equal(mem.tree.nodes, g[f"s{s}_nodes"])
        assert mem.max_priority == g[f"s{s}_maxp"]
    slot = mem.store(z, 1, 0.0, z, False)
    assert slot == g["store_slot"]
    assert np.array_equal(mem.tree.nodes, g["store_nodes"])
    with pytest.raises(IndexError):
        mem.update_priorities(np.array([3, 5, 999, 7]), np.array([9.0, 8.0, 7.0, 6.0]))
    assert np.array_equal(mem.tree.nodes, g["partial_after"])
    assert mem.max_priority == g["partial_maxp"]


def _tiny_oracle():
    trunk = [("conv", 2, 2, 2), ("relu",), ("fc", 8), ("relu",)]
    return O.QNet(trunk, (6, 6, 2), 3, True)


def test_rmsprop_bit_exact(golden):
    g = golden("rmsprop")
    net = _tiny_oracle()
    net.init(5)
    for k in net.params:
        assert np.array_equal(net.params[k], g[f"w0_{k}"]), k
    opt = O.RmsPropState(net)
    for step in range(5):
        for k in net.grads:
            net.grads[k][...] = g[f"g{step}_{k}"]
        opt.step()
    for k in net.params:
        assert np.array_equal(net.params[k], g[f"w_{k}"]), k
        assert np.array_equal(opt.acc[k], g[f"acc_{k}"]), k


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg4", "cfg4h"])
def test_learner_matches_reference_golden(golden, name):
    g = golden(f"learn_{name}")
    dueling, double, per, huber, steps, cap, seed = (int(v) for v in g["meta"])
    online, target, mem, opt, cfg = oracle_learner(bool(dueling), bool(double), bool(per),
                                                   bool(huber), cap, seed)
    if per:
        assert np.array_equal(mem.tree.nodes, g["nodes_before"])
    for st in range(steps):
        rng = np.random.default_rng(1000 + st)
        res = O.learn_step(online, target, mem, opt, cfg, 100 + 4 * st, rng=rng)
        assert rel_norm(res["targets"], g[f"st{st}_targets"]) < NET_TOL
        assert rel_norm(res["td_errors"], g[f"st{st}_td"]) < NET_TOL
        assert rel_norm(res["losses"], g[f"st{st}_losses"]) < NET_TOL
        if st == 0:
            assert rel_norm(res["q"], g["q0"]) < NET_TOL
            assert rel_norm(res["out_grad"], g["outgrad0"]) < NET_TOL
            for k, v in online.params.items():
                assert rel_norm(v.ravel()[::997], g[f"w1_{k}"]) < NET_TOL, k
        if per:
            assert rel_norm(mem.tree.nodes, g[f"st{st}_nodes"]) < 1e-9
    for k, v in online.params.items():
        assert rel_norm(v.ravel()[::997], g[f"wN_{k}"]) < 1e-3, k


def test_oracle_vs_live_reference_one_step(reference_deepq):
    """Direct comparison with the live reference on a fresh case (container
    only): bit-exact indices, norm-wise network fields."""
    deepq = reference_deepq
    from deepq.config import RunConfig
    from deepq.replay import PrioritizedReplay, PriorityConfig
    from tests.golden.make_golden import fill_reference_memory

    cfg = RunConfig(double=True, dueling=True, batch_size=32, beta_end_step=500)
    on = deepq.build_network("atari", (84, 84, 4), 4, True)
    tg = deepq.build_network("atari", (84, 84, 4), 4, True)
    deepq.init_params(on, 11)
    deepq.init_params(tg, 12)
    opt = deepq.RmsProp(on)
    mem = PrioritizedReplay(48, (84, 84, 4), PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    fill_reference_memory(mem, 48, 3, True)
    res = deepq.learn_step(on, tg, mem, opt, cfg, 33, np.random.default_rng(9))

    o_on, o_tg, o_mem, o_opt, o_cfg = oracle_learner(True, True, True, cap=48, seed=3,
                                                     beta_end=500, online_seed=11,
                                                     target_seed=12)
    ores = O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, 33, rng=np.random.default_rng(9))
    assert rel_norm(ores["td_errors"], res.td_errors) < 1e-6
    for n, t in on.named_tensors():
        assert rel_norm(o_on.params[n], t.values) < 1e-6, n
