"""Sum-tree sampling / update at 1M leaves (the SURVEY §8(d) sampler
microbenchmark) on its own, for ncu captures and A/B runs; checks the
sampled indices against the CPU oracle's descent (bit-exact).

    python tools/tree_bench.py [k]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from oracle import deepq_oracle as O  # noqa: E402

cap = 1 << 20
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
mem = P.PrioritizedReplay(cap, (1, 1, 4), P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1.0, 100)))
leaves = np.random.default_rng(0).random(cap) ** 3 + 1e-3
mem.tree.load_leaves(leaves)
mem.memory._set_size(cap)
u = torch.as_tensor(np.random.default_rng(1).random(k), device="cuda")
beta = torch.full((1,), 0.4, dtype=torch.float64, device="cuda")
qi = torch.empty(k, dtype=torch.int64, device="cuda")
qp = torch.empty(k, dtype=torch.float64, device="cuda")
qw = torch.empty(k, dtype=torch.float64, device="cuda")
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    mem.sample_indices(u, k, beta, qi, qp, qw, fl)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mem.sample_indices(u, k, beta, qi, qp, qw, fl)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
ref = O.HeapTree(cap)
ref.nodes[:] = mem.tree.nodes.cpu().numpy()
idx, prob, w = O.per_indices(ref, cap, k, 0.4, u.cpu().numpy())
exact = bool(np.array_equal(qi.cpu().numpy(), idx)) and bool(np.array_equal(qp.cpu().numpy(), prob))
wmax = float(np.max(np.abs(qw.cpu().numpy() - w) / w))
print(f"tree_sample k={k}: {us:.1f} us, {k * 200 / (us * 1e-6) / 1e9:.0f} GB/s algorithmic "
      f"(200 B/query), indices+P bit-exact {exact}, IS weight max rel {wmax:.1e}")
