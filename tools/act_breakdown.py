"""Diagnostic: where a batch-1 act (select_action) spends its time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import trainer as T  # noqa: E402

for arch, shape in (("desk", (24, 24, 4)), ("atari", (84, 84, 4))):
    net = P.build_network(arch, shape, 3, True)
    P.init_params(net, 1)
    a = T._actor(net)
    st = np.random.default_rng(0).random(shape).astype(np.float32)
    for _ in range(50):
        a.q_values(st)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        a.q_values(st)
    t_act = (time.perf_counter() - t0) / n * 1e6
    # device time of the act graph alone, back to back
    g = a.graph
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        type(g).__mro__[1].replay(g)
    e1.record()
    torch.cuda.synchronize()
    t_dev = e0.elapsed_time(e1) / n * 1e3
    # a bare launch + sync round trip
    t0 = time.perf_counter()
    for _ in range(n):
        torch.cuda.synchronize()
    t_sync = (time.perf_counter() - t0) / n * 1e6
    print(f"{arch}: act {t_act:.1f} us, graph device time {t_dev:.1f} us, bare sync {t_sync:.1f} us")


def dev_us(fn, reps=20, replays=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * replays) * 1e3


for arch, shape in (("desk", (24, 24, 4)), ("atari", (84, 84, 4))):
    net = P.build_network(arch, shape, 3, True)
    P.init_params(net, 1)
    a = T._actor(net)
    print(f"{arch}: H2D state {dev_us(lambda: a.d_x.copy_(a.h_x, non_blocking=True)):.1f} us, "
          f"D2H q {dev_us(lambda: a.h_q.copy_(a.bind.act[-1][:a.nA], non_blocking=True)):.1f} us, "
          f"forward {dev_us(lambda: net.forward_into(a.d_x, a.bind, flags=a.flags)):.1f} us")
    for l in range(len(net._units)):
        print(f"   layer {l} {net._units[l]['name']}: {dev_us(lambda: net.layer_into(a.bind, l, 0, a.flags)):.1f} us")
