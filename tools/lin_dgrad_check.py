"""Diagnostic: fc1 dgrad (dqn_net_layer phase 1) vs a torch fp32 reference,
repeated launches, to separate a wrong result from a nondeterministic one."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
B = 32
torch.manual_seed(0)
x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
bind = net.binding(B)
net.forward_into(x, bind)
fc1 = next(i for i, u in enumerate(net._units) if u["kind"] == _lib.LAYER_LINEAR)
g = torch.Generator(device="cuda").manual_seed(0)
bind.dact[fc1].copy_(torch.randn(bind.dact[fc1].shape, device="cuda", generator=g) * 0.01)
W = dict(net.named_tensors())["fc1.weight"].values            # [3136, 512]
dy = bind.dact[fc1][:B * 512].view(B, 512)
mask = bind.act[fc1 - 1][:B * 3136].view(B, 3136)
ref = (dy.double() @ W.double().t()) * (mask > 0)
outs = []
for rep in range(4):
    bind.dact[fc1 - 1].zero_()
    net.layer_into(bind, fc1, 1)
    torch.cuda.synchronize()
    outs.append(bind.dact[fc1 - 1][:B * 3136].view(B, 3136).clone())
err = [float((o.double() - ref).norm() / ref.norm()) for o in outs]
same = all(torch.equal(outs[0], o) for o in outs[1:])
print(f"BN=32 rel err {max(err):.3e} deterministic {same}")
bad = (outs[0].double() - ref).abs() > 1e-4 * ref.abs().max()
if bad.any():
    rows, cols = torch.nonzero(bad, as_tuple=True)
    print("bad rows", sorted(set(rows.tolist()))[:10], "cols", sorted(set((cols // 32).tolist()))[:20],
          "count", int(bad.sum()))
if os.environ.get("LIN_DGRAD_DUMP"):
    torch.save(outs[0].cpu(), os.environ["LIN_DGRAD_DUMP"])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(20):
    net.layer_into(bind, fc1, 1)
e0.record()
for _ in range(200):
    net.layer_into(bind, fc1, 1)
e1.record()
torch.cuda.synchronize()
print(f"fc1 dgrad {e0.elapsed_time(e1) / 200 * 1000:.2f} us/launch (incl. host launch overhead)")
