"""Diagnostic: device time of the learner's non-GEMM kernels in isolation
(CUDA events, back-to-back launches, 1M-leaf tree / 100k ring)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import agent  # noqa: E402


def timeit(fn, reps=20, replays=50):
    """Device time per call: `reps` calls captured in one CUDA graph."""
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


cap = int(os.environ.get("CAP", "1000000"))
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
    P.learn_step(on, tg, mem, opt, cfg, s, rng)
pl = agent._plan_for(on, tg, mem, opt, cfg)
k = pl.k
print(f"tree_sample   {timeit(lambda: mem.sample_indices(pl.d_in[:k], k, pl.d_in[k:], pl.idx, pl.prob, pl.w, pl.flags)):7.2f} us")
print(f"ring_gather   {timeit(lambda: pl.ring.gather_into(pl.idx, k, pl.x[:k], pl.x[k:], pl.a, pl.r, pl.t)):7.2f} us")
print(f"tree_update   {timeit(lambda: mem.update_priorities_dev(pl.idx, pl.d_out[k:2 * k], k, pl.flags)):7.2f} us")
print(f"rms_apply     {timeit(lambda: opt.enqueue_apply(pl.flags)):7.2f} us")
pl.run(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    pl.run(True)
e1.record()
torch.cuda.synchronize()
print(f"whole update  {e0.elapsed_time(e1) / 200 * 1e3:7.2f} us (graph replay)")

# the fused head (K1: both Q heads + TD block, K2: head backward + wgrad)
import ctypes as C  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402


def head():
    out = pl.d_out
    _lib.call("dqn_head_td", _lib.stream_ptr(), C.byref(on.desc_for(pl.x)), on.flat_values.data_ptr(),
              on.flat_grads.data_ptr(), C.byref(pl.on_bind.struct), C.byref(pl.on_view.struct),
              C.byref(tg.desc_for(pl.x)), tg.flat_values.data_ptr(), C.byref(pl.tg_bind.struct),
              pl.a.data_ptr(), pl.r.data_ptr(), pl.t.data_ptr(), pl.w.data_ptr(), pl.gamma,
              pl.flags_td, out[:k].data_ptr(), out[k:2 * k].data_ptr(), out[2 * k:3 * k].data_ptr(),
              out[3 * k:].data_ptr(), pl.head_work.data_ptr(), pl.flags.data_ptr(), None)


print(f"head_td (K1+K2) {timeit(head):7.2f} us")
print(f"rms_apply+sync {timeit(lambda: (opt.enqueue_apply(pl.flags), P.sync_target(on, tg))):7.2f} us")
print(f"empty kernel   {timeit(lambda: _lib.call('dqn_sync_target', _lib.stream_ptr(), tg.flat_values.data_ptr(), on.flat_values.data_ptr(), 0)):7.2f} us")

# conv1 weight gradient from the frames (the update's last GEMM)
us = timeit(lambda: pl.online.layer_into(pl.on_view, 0, 2, pl.flags))
print(f"conv1 wgrad    {us:7.2f} us")
