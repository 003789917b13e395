"""Batch-1/3 forwards vs the same rows of a batch-64 forward (used by
tests/test_gpu_network.py).
Prints "OK <max rel err>" or raises."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from tests.helpers import rel_norm  # noqa: E402

worst = 0.0
for arch, shape, u8 in (("atari", (84, 84, 4), True), ("atari", (84, 84, 4), False),
                        ("desk", (24, 24, 4), False)):
    net = P.build_network(arch, shape, 4, True)
    P.init_params(net, 2)
    xs = np.random.default_rng(1).integers(0, 256, size=(64,) + shape, dtype=np.uint8)
    x = xs if u8 else (xs / 255.0).astype(np.float32)
    big = net.forward(x).cpu().numpy().copy()
    for rows in (1, 3):
        err = rel_norm(net.forward(x[:rows]).cpu().numpy(), big[:rows])
        assert err < 1e-5, (arch, u8, rows, err)
        worst = max(worst, err)
print(f"OK {worst:.2e}")
