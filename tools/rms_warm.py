"""Diagnostic: RMSprop apply over the Atari net with L2 warm (back-to-back
launches, 27 MB of w / g / acc stay resident) vs after an L2 flush."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
opt = P.RmsProp(net)
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(20):
    net.flat_grads.normal_(0, 1e-3)
    opt.enqueue_apply(fl)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for mode in ("warm", "flushed"):
    ts = []
    for _ in range(20):
        if mode == "flushed":
            flush.fill_(1)
        e[0].record()
        opt.enqueue_apply(fl)
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]) * 1e3)
    ts.sort()
    print(f"rms_apply {mode}: median {ts[len(ts) // 2]:.2f} us, min {ts[0]:.2f} us")
