"""Diagnostic: conv2 / conv3 dgrad (dqn_net_layer phase 1, tcgen05 engine) vs
an fp64 torch reference, over repeated launches; LIN_DGRAD_DUMP-style dump
(CONV_DGRAD_DUMP) so the TMA and register B paths can be compared bit for bit."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
dumps = {}
worst = 0.0
for B in (32, 5, 64):
    torch.manual_seed(B)
    x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
    bind = net.binding(B)
    net.forward_into(x, bind)
    for i, u in enumerate(net._units):
        if u["kind"] != _lib.LAYER_CONV or i == 0:
            continue
        fh, fw, sh, sw = u["geo"]
        ih, iw, ic = u["in_shape"]
        oh, ow, oc = u["out_shape"]
        W = dict(net.named_tensors())[u["name"] + ".weight"].values.reshape(fh, fw, ic, oc)
        g = torch.Generator(device="cuda").manual_seed(i)
        bind.dact[i].copy_(torch.randn(bind.dact[i].shape, device="cuda", generator=g) * 0.01)
        dy = bind.dact[i][:B * oh * ow * oc].view(B, oh, ow, oc)
        mask = bind.act[i - 1][:B * ih * iw * ic].view(B, ih, iw, ic)
        ref = torch.nn.grad.conv2d_input((B, ic, ih, iw), W.double().permute(3, 2, 0, 1),
                                         dy.double().permute(0, 3, 1, 2), stride=(sh, sw))
        ref = ref.permute(0, 2, 3, 1) * (mask > 0)
        outs = []
        for rep in range(3):
            bind.dact[i - 1].zero_()
            net.layer_into(bind, i, 1)
            torch.cuda.synchronize()
            outs.append(bind.dact[i - 1][:B * ih * iw * ic].view(B, ih, iw, ic).clone())
        err = max(float((o.double() - ref).norm() / ref.norm()) for o in outs)
        same = all(torch.equal(outs[0], o) for o in outs[1:])
        worst = max(worst, err if same else 1.0)
        dumps[f"{u['name']}_B{B}"] = outs[0].cpu()
        print(f"{u['name']} B={B} rel err {err:.3e} deterministic {same}")
print(f"WORST {worst:.3e}")
if os.environ.get("CONV_DGRAD_DUMP"):
    torch.save(dumps, os.environ["CONV_DGRAD_DUMP"])
