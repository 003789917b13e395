"""Diagnostic (trace build): conv2 / conv3 forward error against an fp64
convolution, generic engine vs conv_tc.cu, batch 64."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("DQN_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, synth  # noqa: E402
on = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(on, 5)
B = 64
x8 = torch.as_tensor(synth.frames(4, 1, np.arange(B) * 7 + 3), device="cuda")
tens = dict(on.named_tensors())
shapes = [tuple(u["out_shape"]) for u in on._units]
for mode, ts in ((-1, 0), (0, 0), (0, 2), (0, 3), (0, 4)):
    _lib.lib.dqn_ct_set_cluster(mode)
    _lib.lib.dqn_ct_set_ts(ts)
    on.forward(x8)
    bind = on.binding(B)
    out = []
    for l, (name, fh, st) in enumerate([("conv2", 4, 2), ("conv3", 3, 1)], start=1):
        h, w, c = shapes[l - 1]; oh, ow, n = shapes[l]
        xin = bind.act[l - 1][: B * h * w * c].view(B, h, w, c).double().permute(0, 3, 1, 2)
        W = tens[f"{name}.weight"].values.double().reshape(fh, fh, c, n).permute(3, 2, 0, 1)
        ref = F.conv2d(xin, W, tens[f"{name}.bias"].values.double(), stride=st).permute(0, 2, 3, 1)
        ref = F.relu(ref)
        got = bind.act[l][: B * oh * ow * n].view(B, oh, ow, n).double()
        out.append(f"{name} rel {float((got-ref).norm()/ref.norm()):.3e} max {float((got-ref).abs().max()/ref.abs().max()):.3e}")
    print("engine" if mode < 0 else f"conv_tc ts={ts}", " | ".join(out))
