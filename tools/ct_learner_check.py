"""Diagnostic: after one eager cfg2 learner update, the conv2 / conv3
activations of both networks' forward bindings against an fp64 convolution
of the same inputs."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("DQN_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, agent  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
per = len(sys.argv) > 2 and sys.argv[2] == "per"
_lib.lib.dqn_ct_set_cluster(mode)
cfg = P.RunConfig(double=True, dueling=False, batch_size=32, beta_end_step=50_000_000,
                  priority_alpha=0.6 if per else 0.0)
on = P.build_network("atari", (84, 84, 4), 4, False)
tg = P.build_network("atari", (84, 84, 4), 4, False)
P.init_params(on, 1)
P.init_params(tg, 2)
opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
N = 100_000
mem = (P.PrioritizedReplay(N, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
       if per else P.ReplayMemory(N, (84, 84, 4)))
mem.fill_synthetic(5, N)
agent.USE_GRAPH = False
P.learn_step(on, tg, mem, opt, cfg, 1000, np.random.default_rng(77))
torch.cuda.synchronize()
plan = agent._plan_for(on, tg, mem, opt, cfg)
for label, net, bind in (("online", on, plan.on_bind), ("target", tg, plan.tg_bind)):
    B = bind.batch
    tens = dict(net.named_tensors())
    shapes = [tuple(u["out_shape"]) for u in net._units]
    out = []
    for l, (name, fh, st) in enumerate([("conv2", 4, 2), ("conv3", 3, 1)], start=1):
        h, w, c = shapes[l - 1]
        oh, ow, n = shapes[l]
        xin = bind.act[l - 1][: B * h * w * c].view(B, h, w, c).double().permute(0, 3, 1, 2)
        W = tens[f"{name}.weight"].values.double().reshape(fh, fh, c, n).permute(3, 2, 0, 1)
        ref = F.relu(F.conv2d(xin, W, tens[f"{name}.bias"].values.double(), stride=st))
        ref = ref.permute(0, 2, 3, 1)
        got = bind.act[l][: B * oh * ow * n].view(B, oh, ow, n).double()
        d = (got - ref).abs().amax(dim=(1, 2, 3))
        bad = torch.nonzero(d > 1e-4 * float(ref.abs().max())).flatten().tolist()
        out.append(f"{name} rel {float((got - ref).norm() / ref.norm()):.2e} bad images {bad[:10]}")
    print(f"mode {mode} {'per' if per else 'uniform'} {label} B={B}: " + " | ".join(out), flush=True)
