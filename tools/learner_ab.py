"""Diagnostic: the cfg4 learner's device update rate (bench.py's device loop:
pre-drawn PER uniforms in HBM, one graph launch per update) under several
settings of a library-side override, interleaved A/B/A/B so clock and
placement drift average out.

    python tools/learner_ab.py --ct=-1,0,2:3,0:2:192,0:2:128:0  # conv_tc cluster[:stages[:fill[:dgrad[:dgrad fill]]]]
                                                 # (-1 = generic engine, 0 = auto)
Settings are applied before each (re)capture: launch configurations are baked
into the graph.  Uses the trace build by default (the overrides exist only
there; with DQN_B200_LIB pointing at the product library the overrides are
skipped and only Python-side switches apply); its
tcgen05-engine time marks slow the engine kernels a little, so confirm an
engine-side winner with two product builds and bench.py.
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("DQN_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, agent  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ct", default="-1,0")
    ap.add_argument("--cap", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    settings = a.ct.split(",")

    prio = {"v": None}

    def _set(name, *vals):
        fn = getattr(_lib.lib, name, None)       # trace-build entry points only
        if fn is not None:
            fn(*vals)

    def apply(v):
        _set("dqn_c1_set", 1)
        _set("dqn_lt_set_cluster", 4, 16)
        _set("dqn_tc_set_cluster_splitk", 1)
        _set("dqn_w1_set_cluster_max", 4)
        _set("dqn_tc_set_dgrad_cap", 16)
        _set("dqn_tc_set_wgrad_cap", 8)
        agent.WEIGHTS_BESIDE = True
        if v == "w8fused":                     # IS weights as the fused sample launch's extra CTA row
            agent.WEIGHTS_BESIDE = False
            v = "0"
        if v.startswith("wcap="):              # fp32 conv wgrad split cap
            _set("dqn_tc_set_wgrad_cap", int(v[5:]))
            v = "0"
        _set("dqn_ct_set_fill_small", 64)
        _set("dqn_ct_set_ts", 3)
        _set("dqn_ct_set_dts", 3)
        _set("dqn_ltd_set_min_batch", 64)
        _set("dqn_ltd_set_fill", 128)
        if v.startswith("ltdmin="):            # fc1 dgrad on lin_tc above this batch[/fill]
            mb_, _, fl_ = v[7:].partition("/")
            _set("dqn_ltd_set_min_batch", int(mb_))
            _set("dqn_ltd_set_fill", int(fl_ or 128))
            v = "0"
        if v.startswith("dts="):               # conv_tc dgrad with A lo in TMEM, stages
            _set("dqn_ct_set_dts", int(v[4:]))
            v = "0"
        if v.startswith("ts="):                # conv_tc forward with A lo in TMEM, stages
            _set("dqn_ct_set_ts", int(v[3:]))
            v = "0"
        _set("dqn_rms_set_cap", 148 * 8)
        if v.startswith("rms="):               # optimizer grid cap
            _set("dqn_rms_set_cap", int(v[4:]))
            v = "0"
        if v.startswith("fs="):                # conv_tc fill: fs=<batch <= 32>[/<above>]
            fs_, _, fb_ = v[3:].partition("/")
            _set("dqn_ct_set_fill_small", int(fs_))
            v = "0:2:" + (fb_ or "128")
        if v.startswith("dcap="):              # linear dgrad split cap
            _set("dqn_tc_set_dgrad_cap", int(v[5:]))
            v = "0"
        if v.startswith("w1cl="):              # conv1 wgrad: largest cluster
            _set("dqn_w1_set_cluster_max", int(v[5:]))
            v = "0"
        if v == "nocks":                       # engine split-K through global partials only
            _set("dqn_tc_set_cluster_splitk", 0)
            v = "0"
        if v.startswith("lt="):                # fc1 forward cluster sizes: lt=<b<=32>/<b>32>
            a_, b_ = v[3:].split("/")
            _set("dqn_lt_set_cluster", int(a_), int(b_))
            v = "0"
        if v.startswith("c1="):                # conv1 forward kernel on (1) / engine (0)
            _set("dqn_c1_set", int(v[3:]))
            v = "0"
        elif v.startswith("p"):                # stream priorities: p<main>,<side>,<tree>
            prio["v"] = [int(x) for x in v[1:].split("/")]
            v = "0"
        else:
            prio["v"] = None
        cl, _, rest = v.partition(":")
        st, _, rest = rest.partition(":")
        fill, _, rest = rest.partition(":")
        dg, _, dfill = rest.partition(":")
        _set("dqn_ct_set_dgrad", int(dg or 1))
        _set("dqn_ct_set_dfill", int(dfill or 256))
        _set("dqn_ct_set_cluster", int(cl))
        _set("dqn_ct_set_stages", int(st or 2))
        _set("dqn_ct_set_fill", int(fill or 128))
    cfg = P.RunConfig(batch_size=32, double=True, dueling=True, priority_alpha=0.6,
                      beta_end_step=50_000_000)
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    mem = P.PrioritizedReplay(a.cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    mem.fill_synthetic(1, a.cap)
    rng = np.random.default_rng(2)
    for s in range(4):
        P.learn_step(on, tg, mem, opt, cfg, 50_000 + s, rng)
    k = 32
    draws = np.empty((a.steps, k + 1))
    for s in range(a.steps):
        draws[s, :k] = rng.random(k)
        draws[s, k] = mem.beta(50_200 + s)
    d_draws = torch.as_tensor(draws, device="cuda")
    slot = torch.zeros_like(d_draws[0])
    graphs = {}
    for v in settings:
        apply(v)
        P.agent._PLANS.clear()
        P.learn_step(on, tg, mem, opt, cfg, 50_100, rng)       # a plan of this setting
        plan = agent._plan_for(on, tg, mem, opt, cfg)
        if prio["v"] is not None:
            pm, ps, pt = prio["v"]
            plan.capture_stream = torch.cuda.Stream(priority=pm)
            plan.side = torch.cuda.Stream(priority=ps)
            plan.tree_stream = torch.cuda.Stream(priority=pt)
        saved = plan.h_in
        plan.h_in = slot
        graphs[v] = (plan, agent.capture_graph(lambda: plan.enqueue(io=False), plan.capture_stream))
        plan.h_in = saved
    apply("0")
    sp = torch.cuda.current_stream().cuda_stream
    res = {v: [] for v in settings}
    for _ in range(a.rounds):
        for v in settings:
            g = graphs[v][1][1]
            for s in range(20):
                slot.copy_(d_draws[s], non_blocking=True)
                g.launch(sp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in range(a.steps):
                slot.copy_(d_draws[s], non_blocking=True)
                g.launch(sp)
            e1.record()
            torch.cuda.synchronize()
            res[v].append(a.steps / (e0.elapsed_time(e1) / 1e3))
    for v in settings:
        print(f"{v:>8}: " + " ".join(f"{x:7.0f}" for x in res[v]) +
              f"  | median {np.median(res[v]):7.0f} updates/s", flush=True)


if __name__ == "__main__":
    main()
