"""Diagnostic: where the host time of the acting loop goes (desk preset,
Catch, 20k env steps after learning starts), cProfile sorted by tottime."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1804_05834_b200 as P  # noqa: E402

cfg = P.resolve_config({"preset": "desk", "env": "catch", "seed": 1, "max_steps": 26_000,
                        "learning_start": 5_000, "test_period": 1_000_000})
tr = P.Trainer(cfg)
while tr.step < 6_000:
    tr._one_step()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
while tr.step < cfg.max_steps:
    tr._one_step()
pr.disable()
dt = time.perf_counter() - t0
print(f"{(cfg.max_steps - 6_000) / dt:.0f} env steps/s ({dt / (cfg.max_steps - 6_000) * 1e6:.0f} us/step, "
      f"profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(22)

# the batch-1 act alone (no learner work queued)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1804_05834_b200 import trainer as T  # noqa: E402
a = T._actor(tr.online)
st = np.random.default_rng(0).random(tr.online.input_shape).astype(np.float32)
for _ in range(50):
    a.q_values(st)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    a.q_values(st)
print(f"act alone: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us per greedy action")
