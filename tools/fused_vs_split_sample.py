"""Diagnostic: learn_step's sampled indices / TD errors with the fused
sample+gather kernel vs dqn_tree_sample + gather (DQN_B200_FUSED_SAMPLE=0 is
read at plan build, so both run in one process via two plans)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from tests.test_gpu_frame_ring import episodic  # noqa: E402

shape, cap = (24, 24, 4), 256
stream = episodic(np.random.default_rng(11), 300, shape)
out = {}
for name, dedup, fused in (("full_fused", False, "1"), ("full_split", False, "0"), ("dedup", True, "1")):
    os.environ["DQN_B200_FUSED_SAMPLE"] = fused
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
    from paper_1804_05834_b200.agent import _plan_for
    idxs, tds = [], []
    for i in range(4):
        res = P.learn_step(on, tg, mem, opt, cfg, 100 + i, g)
        plan = _plan_for(on, tg, mem, opt, cfg)
        idxs.append(plan.last_indices().cpu().numpy().copy())
        tds.append(res.td_errors.copy())
    out[name] = (np.concatenate(idxs), np.concatenate(tds), plan.fused_sample)
    for i in range(4):
        print(name, i, "idx", idxs[i][:6], "td", tds[i][:3], "maxp", mem.max_priority)
print("full fused vs split idx equal", np.array_equal(out["full_fused"][0], out["full_split"][0]),
      "td equal", np.array_equal(out["full_fused"][1], out["full_split"][1]))
print("full split vs dedup idx equal", np.array_equal(out["full_split"][0], out["dedup"][0]),
      "td equal", np.array_equal(out["full_split"][1], out["dedup"][1]))
# the stand-alone gather on this stream, and the learner's gathered batch
from paper_1804_05834_b200.frame_ring import FrameDedupMemory  # noqa: E402
full = P.ReplayMemory(cap, shape)
dd = FrameDedupMemory(cap, shape)
for s, a, r, s2, t in stream:
    full.store(P.Transition(s, a % 3, r, s2, t))
    dd.store(P.Transition(s, a % 3, r, s2, t))
ti = torch.arange(cap, device="cuda")
x1, x2 = torch.empty_like(full.states), torch.empty_like(full.states)
dd.gather_into(ti, cap, x1, x2, None, None, None)
bad = [(i) for i in range(cap) if not (torch.equal(x1[i], full.states[i]) and torch.equal(x2[i], full.next_states[i]))]
print("standalone mismatching slots", len(bad), bad[:10], "live frames", dd.index.live_frames)
if bad:
    i = bad[0]
    print("ids", dd.index.ids[i], "cursor", dd.cursor)
    for which, (a, b) in enumerate(((x1[i], full.states[i]), (x2[i], full.next_states[i]))):
        print(which, [bool(torch.equal(a[..., s], b[..., s])) for s in range(4)])
