"""Diagnostic (trace build): fc1 forward at large batch, lin_tc with several
K-split cluster sizes against the generic engine."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("DQN_B200_LIB", str(ROOT / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for B in (256, 1024, 4096):
    b = net.binding(B)
    x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
    net.forward_into(x, b)
    torch.cuda.synchronize()
    res = []
    for mb, cl in ((64, 1), (1 << 20, 0), (1 << 20, 1), (1 << 20, 2), (1 << 20, 4), (1 << 20, 8)):
        _lib.lib.dqn_lt_set_large(mb, cl)
        args = (C.byref(net.desc_for(x)), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
                C.byref(b.struct), 3, 0, flags.data_ptr())
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):
                _lib.call("dqn_net_layer", s.cuda_stream, *args)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(5):
                    _lib.call("dqn_net_layer", s.cuda_stream, *args)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        res.append(f"{'engine' if mb == 64 else (f'lin_tc cl{cl}' if cl else 'lin_tc auto')} {us:.1f} us "
                   f"({2 * B * 3136 * 512 / us / 1e6:.1f} TF/s)")
    _lib.lib.dqn_lt_set_large(1 << 20, 0)
    print(f"B={B} fc1 fwd: " + " | ".join(res), flush=True)
    res = []
    q = net.forward(x)
    net.backward(torch.ones_like(q))
    for mb in (1 << 20, 64):
        _lib.lib.dqn_ltd_set_min_batch(mb)
        args = (C.byref(net.desc_for(x)), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
                C.byref(net._cur.struct), 3, 1, flags.data_ptr())
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):
                _lib.call("dqn_net_layer", s.cuda_stream, *args)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(5):
                    _lib.call("dqn_net_layer", s.cuda_stream, *args)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        res.append(f"{'engine' if mb > 4096 else 'lin_tc'} {us:.1f} us "
                   f"({2 * B * 3136 * 512 / us / 1e6:.1f} TF/s)")
    _lib.lib.dqn_ltd_set_min_batch(64)
    print(f"B={B} fc1 dgrad: " + " | ".join(res), flush=True)
