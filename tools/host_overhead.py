"""Diagnostic: host overhead of the public learn_step call vs the bare graph
replay (cfg4, B = 32, 100k ring)."""
import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import agent  # noqa: E402

cfg = P.RunConfig(batch_size=32, beta_end_step=50_000_000)
on = P.build_network("atari", (84, 84, 4), 4, True)
tg = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(on, 1)
P.sync_target(on, tg)
opt = P.RmsProp(on)
mem = P.PrioritizedReplay(100_000, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
mem.fill_synthetic(1, 100_000)
rng = np.random.default_rng(0)
for s in range(20):
    P.learn_step(on, tg, mem, opt, cfg, s, rng)
torch.cuda.synchronize()
plan = agent._plan_for(on, tg, mem, opt, cfg)
N = 2000
t0 = time.perf_counter()
for s in range(N):
    P.learn_step(on, tg, mem, opt, cfg, 100 + s, rng)
t1 = time.perf_counter()
print(f"learn_step e2e: {(t1 - t0) / N * 1e6:.1f} us/update")
st = torch.cuda.current_stream()
t0 = time.perf_counter()
for s in range(N):
    plan.graph_exec.launch(torch.cuda.current_stream().cuda_stream)
    st.synchronize()
t1 = time.perf_counter()
print(f"graph.replay + sync: {(t1 - t0) / N * 1e6:.1f} us/update")
t0 = time.perf_counter()
for s in range(N):
    plan.graph_exec.launch(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"graph.replay back-to-back: {(t1 - t0) / N * 1e6:.1f} us/update")
pr = cProfile.Profile()
pr.enable()
for s in range(500):
    P.learn_step(on, tg, mem, opt, cfg, 5000 + s, rng)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
