"""Diagnostic: conv2 / conv3 forward launch times, conv_tc.cu at
several cluster sizes against the generic engine (tc_gemm.cuh FwdPol), each
a CUDA graph of 20 back-to-back launches of one layer.

    python tools/ct_bench.py
"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("DQN_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
REPS = 20
for B in (32, 64, 4096):
    b = net.binding(B)
    x = torch.randint(0, 256, (B, 84, 84, 4), dtype=torch.uint8, device="cuda")
    net.forward_into(x, b)
    torch.cuda.synchronize()
    for layer, name, phase in ((0, "conv1", 0), (1, "conv2", 0), (2, "conv3", 0), (1, "conv2.dgrad", 1),
                               (2, "conv3.dgrad", 1)):
        res = []
        for cl, stg in ((-1, 2), (0, 2), (0, 12), (0, 13), (0, 14)):
            _lib.lib.dqn_ct_set_cluster(cl)
            _lib.lib.dqn_ct_set_stages(stg if stg < 10 else 2)
            _lib.lib.dqn_ct_set_ts(stg - 10 if stg >= 10 else 0)
            _lib.lib.dqn_ct_set_dgrad(0 if cl < 0 else 1)
            _lib.lib.dqn_c1_set(0 if cl < 0 else 1)
            if layer == 0 and cl > 0:
                continue
            if phase == 1 and stg not in (2, 13, 14):
                continue
            _lib.lib.dqn_ct_set_dts(stg - 10 if (phase == 1 and stg >= 10) else 0)
            args = (C.byref(net.desc_for(x)), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
                    C.byref(b.struct), layer, phase, flags.data_ptr())
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    _lib.call("dqn_net_layer", s.cuda_stream, *args)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(REPS):
                        _lib.call("dqn_net_layer", s.cuda_stream, *args)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * REPS)
            res.append(f"{'engine' if cl < 0 else ('auto' if cl == 0 else f'cl{cl}')}/{stg} {us:.2f}")
        _lib.lib.dqn_ct_set_cluster(0)
        _lib.lib.dqn_ct_set_dgrad(1)
        _lib.lib.dqn_ct_set_ts(3)
        _lib.lib.dqn_ct_set_dts(3)
        _lib.lib.dqn_c1_set(1)
        print(f"B={B} {name}: " + " | ".join(res), flush=True)
