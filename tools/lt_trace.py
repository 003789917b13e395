"""Diagnostic: per-CTA phase marks of the fc1 weight-streaming kernel
(csrc/lin_tc.cu, trace build): fwd and dgrad at batch 32 / 64."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
os.environ["DQN_B200_LIB"] = str(ROOT / "paper_1804_05834_b200" / "libdqn_b200_trace.so")
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
for B in (32, 64):
    b = net.binding(B)
    x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
    net.forward_into(x, b)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    for phase in (0,):
        args = (_lib.stream_ptr(), C.byref(net.desc_for(x)), net.flat_values.data_ptr(),
                net.flat_grads.data_ptr(), C.byref(b.struct), 3, phase, flags.data_ptr())
        for _ in range(3):
            _lib.call("dqn_net_layer", *args)
        torch.cuda.synchronize()
        _lib.call("dqn_net_layer", *args)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (1024 * 6))()
        _lib.lib.dqn_lt_trace(buf)
        t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 6).astype(np.int64)
        t = t[t[:, 0] > 0]
        t = t[t[:, 0] >= t[:, 0].max() - 10**6]           # this launch
        t0 = t[:, 0].min()
        names = ["entry", "pdl", "conv0", "mma_done", "staged", "reduced"]
        print(f"B={B} {'fwd' if phase == 0 else 'dgrad'}: {len(t)} CTAs, span {(t[:, 5].max() - t0) / 1e3:.2f} us | "
              + " ".join(f"{n} {((t[:, i] - t0) / 1e3).mean():.2f}/{((t[:, i] - t0) / 1e3).max():.2f}"
                         for i, n in enumerate(names)))
