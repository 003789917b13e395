"""Diagnostic: every layer phase of the Atari net through the tcgen05 engine
vs the SIMT kernels on identical inputs (relative norm errors)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, synth  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


def main(batch=32, dueling=True):
    torch.cuda.set_device(0)
    net = P.build_network("atari", (84, 84, 4), 4, dueling)
    P.init_params(net, 1)
    g = torch.Generator(device="cuda").manual_seed(0)
    for _, t in net.named_tensors():
        if t.values.dim() == 1:
            t.values.copy_(torch.randn(t.shape, device="cuda", generator=g) * 0.01)
    x = torch.as_tensor(synth.frames(3, 0, np.arange(batch)), device="cuda")
    b = net.binding(batch)
    b.x = x
    b.struct.x = x.data_ptr()
    for u in range(len(net._units)):
        b.dact[u].copy_(torch.randn(b.dact[u].shape, device="cuda", generator=g))
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    d_simt = _lib.NetDesc.from_buffer_copy(net._desc_u8)
    d_simt.algo = 1
    d_tc = _lib.NetDesc.from_buffer_copy(net._desc_u8)
    # forward chain once with SIMT to populate activations
    _lib.call("dqn_net_forward", st, C.byref(d_simt), net.flat_values.data_ptr(), C.byref(b.struct), flags.data_ptr())
    worst = 0.0
    for li, u in enumerate(net._units):
        for phase in (0, 1, 2):
            if phase == 1 and li == 0:
                continue
            outs = []
            for d in (d_simt, d_tc):
                if phase == 0:
                    keep = b.act[li].clone()
                    _lib.call("dqn_net_layer", st, C.byref(d), net.flat_values.data_ptr(),
                              net.flat_grads.data_ptr(), C.byref(b.struct), li, 0, flags.data_ptr())
                    outs.append(b.act[li].clone())
                    b.act[li].copy_(keep)
                elif phase == 1:
                    keep = b.dact[li - 1].clone()
                    _lib.call("dqn_net_layer", st, C.byref(d), net.flat_values.data_ptr(),
                              net.flat_grads.data_ptr(), C.byref(b.struct), li, 1, flags.data_ptr())
                    outs.append(b.dact[li - 1].clone())
                    b.dact[li - 1].copy_(keep)
                else:
                    net.flat_grads.zero_()
                    _lib.call("dqn_net_layer", st, C.byref(d), net.flat_values.data_ptr(),
                              net.flat_grads.data_ptr(), C.byref(b.struct), li, 2, flags.data_ptr())
                    outs.append(net.flat_grads.clone())
            torch.cuda.synchronize()
            e = rel(outs[1], outs[0])
            worst = max(worst, e)
            print(f"{u['name']:5s} {['fwd', 'dgrad', 'wgrad'][phase]:5s} rel={e:.3e} "
                  f"norm={float(outs[0].double().norm()):.4e}", flush=True)
    print("WORST", worst)
    return worst


if __name__ == "__main__":
    for swap in (0,):
        print("== mn descriptor swap", swap)

        main()
