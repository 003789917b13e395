"""One cfg4 learner update (B=32) between cudaProfilerStart/Stop, for
    ncu --profile-from-start off ... python tools/profile_step.py
Eager launches (no CUDA graph) so every kernel of the step is profiled.
The ring is 100k transitions (kernel costs do not depend on capacity except
the sum-tree depth: 17 levels here vs 20 at 1M)."""
import os
import sys
from pathlib import Path

os.environ.setdefault("DQN_B200_GRAPH", "0")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402

cap = int(os.environ.get("CAP", "100000"))
cfg = P.RunConfig(batch_size=32, beta_end_step=50_000_000)
on = P.build_network("atari", (84, 84, 4), 4, True)
tg = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(on, 1)
P.sync_target(on, tg)
opt = P.RmsProp(on)
mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
mem.fill_synthetic(1, cap)
rng = np.random.default_rng(0)
for s in range(5):
    P.learn_step(on, tg, mem, opt, cfg, 1000 + s, rng)
torch.cuda.synchronize()
torch.cuda.profiler.start()
P.learn_step(on, tg, mem, opt, cfg, 2000, rng)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one learn_step")
