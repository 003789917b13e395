"""Diagnostic: one learner update at 1M capacity against the oracle
(tests/test_gpu_parity_1m.py's setup), every tensor's relative error printed,
under several conv_tc overrides (-1 engine, 0 conv_tc, -2 conv_tc for the
stride-2 layer only, -3 stride-1 only) and with / without the CUDA graph."""
import gc
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("DQN_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from oracle import deepq_oracle as O  # noqa: E402
from paper_1804_05834_b200 import _lib, agent  # noqa: E402
from tests.helpers import ATARI, rel_norm  # noqa: E402
from tests.test_gpu_parity_1m import CFGS, N, SEED, VirtualRing  # noqa: E402


def run(name, graph):
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
        o_mem.tree.nodes[:] = mem.tree.nodes.cpu().numpy()
        o_mem.alpha, o_mem.eps = 0.6, 0.01
        o_mem.beta_sched = (0.4, 1.0, 50_000_000)
        o_mem.max_priority = float(mem.max_priority)
    else:
        o_mem = ring
    o_cfg = O.LearnCfg(double=kw["double"])
    agent.USE_GRAPH = graph
    res = P.learn_step(on, tg, mem, opt, cfg, 1000, np.random.default_rng(77))
    agent.USE_GRAPH = True
    ores = O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, 1000, rng=np.random.default_rng(77))
    out = [f"td {rel_norm(res.td_errors, ores['td_errors']):.1e}"]
    for n, t in on.named_tensors():
        out.append(f"{n} {rel_norm(t.values.cpu().numpy(), o_on.params[n]):.1e}")
    return " ".join(out)


modes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "-1,0,-2,-3").split(",")]
names = (sys.argv[2] if len(sys.argv) > 2 else "cfg2,cfg3").split(",")
graphs = [g == "1" for g in (sys.argv[3] if len(sys.argv) > 3 else "0").split(",")]
for mode in modes:
    for name in names:
        for graph in graphs:
            _lib.lib.dqn_ct_set_cluster(mode)
            P.agent._PLANS.clear()
            print(f"mode {mode:2d} {name} graph={graph}: {run(name, graph)}", flush=True)
            gc.collect()
            torch.cuda.empty_cache()
