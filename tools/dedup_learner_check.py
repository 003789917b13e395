"""Diagnostic: the learner's gathered batch on a frame-deduplicated ring vs
a manual gather of the same indices."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200.agent import _plan_for  # noqa: E402
from tests.test_gpu_frame_ring import episodic  # noqa: E402

shape, cap = (24, 24, 4), 256
stream = episodic(np.random.default_rng(11), 300, shape)
cfg = P.RunConfig(batch_size=32, double=True, dueling=True, beta_end_step=1000)
on = P.build_network("desk", shape, 3, True)
tg = P.build_network("desk", shape, 3, True)
P.init_params(on, 1)
P.sync_target(on, tg)
opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
mem = P.PrioritizedReplay(cap, shape, P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()), frame_dedup=True)
for s, a, r, s2, t in stream:
    mem.store(P.Transition(s, a % 3, r, s2, t))
g = np.random.default_rng(5)
for step in range(3):
    P.learn_step(on, tg, mem, opt, cfg, 100 + step, g)
    plan = _plan_for(on, tg, mem, opt, cfg)
    torch.cuda.synchronize()
    k = plan.k
    idx = plan.last_indices().clone()
    b = mem.memory._gather(idx, None, None)
    print(step, "graph", plan.graph_exec is not None,
          "states", torch.equal(plan.x[:k], b.states), "next", torch.equal(plan.x[k:], b.next_states),
          "a", torch.equal(plan.a, b.actions), "r", torch.equal(plan.r, b.rewards),
          "t", torch.equal(plan.t, b.terminals), "x dtype", plan.x.dtype, plan.x.shape, plan.x.is_contiguous())
    if not torch.equal(plan.x[:k], b.states):
        rows = [j for j in range(k) if not torch.equal(plan.x[j], b.states[j])]
        print("  bad rows", rows[:10], "idx", idx[rows[:5]].tolist())
