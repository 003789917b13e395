"""Soak / race check: two identical cfg4 learners (100k ring) stepped in
lockstep for N updates through learn_step; every 500 updates their TD
errors, parameters, optimizer state and sum trees must be bit-identical,
and no step may fail.  usage: python tools/soak.py [updates]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
cfg = P.RunConfig(batch_size=32, beta_end_step=50_000_000)
L = []
for _ in range(2):
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on)
    mem = P.PrioritizedReplay(100_000, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    mem.fill_synthetic(3, 100_000)
    L.append((on, tg, mem, opt, np.random.default_rng(9)))
t0 = time.perf_counter()
for s in range(N):
    tds = []
    for on, tg, mem, opt, rng in L:
        tds.append(P.learn_step(on, tg, mem, opt, cfg, 1000 + s, rng).td_errors)
        if (s + 1) % 2500 == 0:
            P.sync_target(on, tg)
    assert np.array_equal(tds[0], tds[1]), f"TD errors diverged at update {s}"
    if (s + 1) % 500 == 0:
        (a, _, ma, oa, _), (b, _, mb, ob, _) = L
        assert torch.equal(a.flat_values, b.flat_values), f"weights diverged at {s}"
        assert torch.equal(oa.flat_acc, ob.flat_acc), f"optimizer state diverged at {s}"
        assert torch.equal(ma.tree.nodes, mb.tree.nodes), f"trees diverged at {s}"
        assert np.isfinite(tds[0]).all()
print(f"soak OK: {N} lockstep updates x 2 learners in {time.perf_counter() - t0:.1f} s, "
      f"bit-identical throughout")
