"""Generate the golden fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``deepq`` from /root/reference/pkg/src read-only and writes small
``.npz`` fixtures next to this file.  The fixtures pin the CPU oracle
(oracle/deepq_oracle.py) on machines where the reference is absent (the GPU
box).  Network-valued fields are fp32 BLAS results and may differ in the last
bits across CPUs; the tests compare them with a norm-wise tolerance, while
tree / index / RMSprop fields are compared bit-exactly.
"""

from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

import deepq  # noqa: E402
from deepq.config import RunConfig  # noqa: E402
from deepq.layers import LayerSpec  # noqa: E402
from deepq.network import build_network, init_params  # noqa: E402
from deepq.optim import RmsProp, sync_target  # noqa: E402
from deepq.replay import (PrioritizedReplay, PriorityConfig, ReplayMemory,  # noqa: E402
                          SumTree, Transition)
from deepq.schedules import LinearSchedule  # noqa: E402

_spec = importlib.util.spec_from_file_location("synth", REPO / "paper_1804_05834_b200" / "synth.py")
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)

SUB = 997  # subsample stride for large weight tensors


def tree_cases():
    out = {}
    t = SumTree(4)
    for i, p in enumerate([1.0, 2.0, 3.0, 4.0]):
        t.set(i, p)
    q = np.array([6.5, 0.01, 0.5, 1.0, 1.001, 2.999, 3.0, 3.5, 6.0, 9.99, 10.0, 0.0, 11.0])
    out["kat_nodes"] = t.nodes.copy()
    out["kat_q"] = q
    out["kat_idx"] = t.find(q)
    rng = np.random.default_rng(3)
    for r in range(8):
        n = int(rng.integers(1, 40))
        pri = rng.random(n) * 10.0
        t = SumTree(n)
        for i, p in enumerate(pri):
            t.set(i, float(p))
        qs = rng.random(64) * t.total
        out[f"rand{r}_cap"] = np.int64(n)
        out[f"rand{r}_pri"] = pri
        out[f"rand{r}_nodes"] = t.nodes.copy()
        out[f"rand{r}_q"] = qs
        out[f"rand{r}_idx"] = t.find(qs)
    # big tree: 1000 leaves built by set() in a shuffled order with duplicates
    t = SumTree(1000)
    rng = np.random.default_rng(30)
    order = rng.integers(0, 1000, size=4000)
    vals = rng.random(4000) * 3.0
    for i, v in zip(order, vals):
        t.set(int(i), float(v))
    out["big_order"] = order
    out["big_vals"] = vals
    out["big_nodes"] = t.nodes.copy()
    qs = rng.random(4096) * t.total
    out["big_q"] = qs
    out["big_idx"] = t.find(qs)
    np.savez_compressed(HERE / "tree.npz", **out)


def per_cases():
    out = {}
    cap = 1000
    cfg = PriorityConfig(0.6, 0.01, LinearSchedule(0.4, 1.0, 1000))
    mem = PrioritizedReplay(cap, (1, 1, 1), cfg)
    for i in range(700):                      # partially full: size != capacity
        mem.store(Transition(np.zeros((1, 1, 1), np.float32), i % 4, 0.0,
                             np.zeros((1, 1, 1), np.float32), False))
    td0 = np.abs(np.random.default_rng(40).standard_normal(700)) * 2.0
    mem.update_priorities(np.arange(700), td0)
    out["td0"] = td0
    out["nodes0"] = mem.tree.nodes.copy()
    out["maxp0"] = np.float64(mem.max_priority)
    for s in range(4):
        k = [32, 32, 7, 256][s]
        beta = mem.beta(100 * s + 17)
        rng = np.random.default_rng(100 + s)
        u = np.random.default_rng(100 + s).random(k)
        b = mem.sample(k, beta, rng)
        out[f"s{s}_k"] = np.int64(k)
        out[f"s{s}_beta"] = np.float64(beta)
        out[f"s{s}_u"] = u
        out[f"s{s}_idx"] = b.indices.copy()
        out[f"s{s}_prob"] = b.probabilities
        out[f"s{s}_w"] = b.weights
        td = np.random.default_rng(200 + s).standard_normal(k) * (s + 1)
        if s == 1:          # duplicate indices: last write wins
            b.indices[5] = b.indices[3]
            b.indices[9] = b.indices[3]
            td[9] = 0.0
        out[f"s{s}_upd_idx"] = b.indices.copy()
        out[f"s{s}_td"] = td
        mem.update_priorities(b.indices, np.abs(td))
        out[f"s{s}_nodes"] = mem.tree.nodes.copy()
        out[f"s{s}_maxp"] = np.float64(mem.max_priority)
    # store after updates: new leaf = max_priority ** alpha
    slot = mem.store(Transition(np.zeros((1, 1, 1), np.float32), 1, 0.0,
                                np.zeros((1, 1, 1), np.float32), False))
    out["store_slot"] = np.int64(slot)
    out["store_nodes"] = mem.tree.nodes.copy()
    # partial update: out-of-range index in the middle
    nodes_before = mem.tree.nodes.copy()
    try:
        mem.update_priorities(np.array([3, 5, 999, 7]), np.array([9.0, 8.0, 7.0, 6.0]))
        raise AssertionError("expected IndexError")
    except IndexError:
        pass
    out["partial_before"] = nodes_before
    out["partial_after"] = mem.tree.nodes.copy()
    out["partial_maxp"] = np.float64(mem.max_priority)
    np.savez_compressed(HERE / "per.npz", **out)


def tiny_net(dtype=np.float32, dueling=True):
    trunk = [LayerSpec("convolution", {"filters": 2, "filter_h": 2, "filter_w": 2,
                                       "stride_h": 2, "stride_w": 2}),
             LayerSpec.relu(), LayerSpec.linear(8), LayerSpec.relu()]
    return build_network(trunk, (6, 6, 2), 3, dueling, dtype=dtype)


def rmsprop_case():
    out = {}
    net = tiny_net()
    init_params(net, 5)
    opt = RmsProp(net, 0.000625, 0.95, 1e-6)
    rng = np.random.default_rng(50)
    for step in range(5):
        for name, t in net.named_tensors():
            scale = 10.0 ** rng.integers(-8, 1)
            t.grad[...] = (rng.standard_normal(t.shape) * scale).astype(np.float32)
            out[f"g{step}_{name}"] = t.grad.copy()
        opt.step()
    for name, t in net.named_tensors():
        out[f"w_{name}"] = t.values.copy()
        out[f"acc_{name}"] = opt.acc[name].copy()
    init_params(net, 5)
    for name, t in net.named_tensors():
        out[f"w0_{name}"] = t.values.copy()
    np.savez_compressed(HERE / "rmsprop.npz", **out)


def fill_reference_memory(mem_obj, n, seed, prioritized):
    ring = mem_obj.memory if prioritized else mem_obj
    slots = np.arange(n)
    s = synth.frames(seed, 0, slots)
    s2 = synth.frames(seed, 1, slots)
    a, r, t = synth.metadata(seed, n)
    for i in range(n):
        tr = Transition((s[i].astype(np.float64) / 255.0).astype(np.float32), int(a[i]),
                        float(r[i]), (s2[i].astype(np.float64) / 255.0).astype(np.float32),
                        bool(t[i]))
        mem_obj.store(tr)
    if prioritized:
        mem_obj.update_priorities(np.arange(n), synth.warmup_td(seed, n))
    return ring


def learner_case(name, dueling, double, per, huber=False, steps=3, cap=64, seed=7):
    out = {}
    cfg = RunConfig(double=double, dueling=dueling, huber=huber, batch_size=32,
                    priority_alpha=0.6 if per else 0.0, beta_end_step=1000)
    online = build_network("atari", (84, 84, 4), 4, dueling)
    target = build_network("atari", (84, 84, 4), 4, dueling)
    init_params(online, 1)
    init_params(target, 2)
    opt = RmsProp(online, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    if per:
        pc = PriorityConfig(0.6, 0.01, cfg.beta_schedule())
        mem = PrioritizedReplay(cap, (84, 84, 4), pc)
        fill_reference_memory(mem, cap, seed, True)
        out["nodes_before"] = mem.tree.nodes.copy()
    else:
        mem = ReplayMemory(cap, (84, 84, 4))
        fill_reference_memory(mem, cap, seed, False)
    for st in range(steps):
        rng = np.random.default_rng(1000 + st)
        step = 100 + 4 * st
        res = deepq.learn_step(online, target, mem, opt, cfg, step, rng)
        out[f"st{st}_targets"] = res.targets
        out[f"st{st}_td"] = res.td_errors
        out[f"st{st}_losses"] = res.losses
        if st == 0:
            out["q0"] = online.y.values.copy()
            out["outgrad0"] = online.y.grad.copy()
            for n_, t_ in online.named_tensors():
                out[f"w1_{n_}"] = t_.values.ravel()[::SUB].copy()
                out[f"w1norm_{n_}"] = np.float64(np.linalg.norm(t_.values.astype(np.float64)))
        if per:
            out[f"st{st}_nodes"] = mem.tree.nodes.copy()
            out[f"st{st}_maxp"] = np.float64(mem.max_priority)
    for n_, t_ in online.named_tensors():
        out[f"wN_{n_}"] = t_.values.ravel()[::SUB].copy()
        out[f"wNnorm_{n_}"] = np.float64(np.linalg.norm(t_.values.astype(np.float64)))
    out["meta"] = np.array([dueling, double, per, huber, steps, cap, seed], dtype=np.int64)
    np.savez_compressed(HERE / f"learn_{name}.npz", **out)


if __name__ == "__main__":
    tree_cases()
    per_cases()
    rmsprop_case()
    learner_case("cfg1", dueling=False, double=False, per=False)
    learner_case("cfg3", dueling=False, double=True, per=True)
    learner_case("cfg4", dueling=True, double=True, per=True)
    learner_case("cfg4h", dueling=True, double=True, per=True, huber=True, steps=2)
    print("golden fixtures written to", HERE)
