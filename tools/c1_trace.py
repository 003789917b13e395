"""Diagnostic (trace build): per-CTA phase marks of the conv1 forward kernel
(csrc/conv1_tc.cu) at batch 32 / 64 / 4096 (first 1024 CTAs)."""
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
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for B in (32, 64, 4096):
    b = net.binding(B)
    x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
    net.forward_into(x, b)
    args = (_lib.stream_ptr(), C.byref(net.desc_for(x)), net.flat_values.data_ptr(),
            net.flat_grads.data_ptr(), C.byref(b.struct), 0, 0, flags.data_ptr())
    for _ in range(3):
        _lib.call("dqn_net_layer", *args)
    torch.cuda.synchronize()
    _lib.call("dqn_net_layer", *args)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (1024 * 5))()
    _lib.lib.dqn_c1_trace(buf)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 5).astype(np.int64)
    t = t[t[:, 0] > 0]
    t = t[t[:, 0] >= t[:, 0].max() - 10**6]
    t0 = t[:, 0].min()
    names = ["entry", "pdl", "loaded", "mma_done", "stored"]
    print(f"B={B}: {len(t)} CTAs, span {(t[:, 4].max() - t0) / 1e3:.2f} us | "
          + " ".join(f"{n} {((t[:, i] - t0) / 1e3).mean():.2f}/{((t[:, i] - t0) / 1e3).max():.2f}"
                     for i, n in enumerate(names))
          + f" | per-CTA loaded->done {((t[:, 3] - t[:, 2]) / 1e3).mean():.2f} done->stored "
          f"{((t[:, 4] - t[:, 3]) / 1e3).mean():.2f} entry->loaded {((t[:, 2] - t[:, 0]) / 1e3).mean():.2f}",
          flush=True)
