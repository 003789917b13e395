"""Diagnostic: per-CTA timeline of every tcgen05 layer phase of the Atari net.

Loads the trace build (make -C paper_1804_05834_b200/csrc trace), runs each
layer phase alone and prints, per launch: CTAs, SMs, the span from the first
CTA entry to the last exit, and the mean/max of each CTA phase (setup =
TMEM alloc + operand init + raw prologue, kloop = k-blocks, epi = TMEM ->
partial/final stores, fix = split-K fixup + dealloc), plus the host-side
event time of the same launch.
"""
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
from paper_1804_05834_b200 import _lib, synth  # noqa: E402


def read_trace():
    buf = (C.c_ulonglong * (8192 * 30))()
    n = _lib.lib.dqn_tc_trace(buf, 8192)
    return np.frombuffer(buf, dtype=np.uint64, count=30 * n).reshape(n, 30).astype(np.int64)


def main(skip=0):
    torch.cuda.set_device(0)
    _lib.lib.dqn_tc_skip(skip)
    print(f"== skip mask {skip} (1 no MMA, 2 no loads, 4 no piece stores)")
    _lib.lib.dqn_tc_trace.argtypes = [C.c_void_p, C.c_int]
    _lib.lib.dqn_tc_trace.restype = C.c_int
    net = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(net, 1)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = _lib.stream_ptr()
    g = torch.Generator(device="cuda").manual_seed(0)
    for batch in (64, 32):
        b = net.binding(batch)
        x = torch.as_tensor(synth.frames(3, 0, np.arange(batch)), device="cuda")
        b.x = x
        b.struct.x = x.data_ptr()
        for u in range(len(net._units)):
            b.dact[u].copy_(torch.randn(b.dact[u].shape, device="cuda", generator=g))
        desc = _lib.NetDesc.from_buffer_copy(net._desc_u8)
        _lib.call("dqn_net_forward", st, C.byref(desc), net.flat_values.data_ptr(),
                  C.byref(b.struct), flags.data_ptr())
        for li, u in enumerate(net._units):
            for phase in ((0,) if batch == 64 else (1, 2)):
                if phase == 1 and li == 0:
                    continue
                args = (st, C.byref(desc), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
                        C.byref(b.struct), li, phase, flags.data_ptr())
                for _ in range(3):
                    _lib.call("dqn_net_layer", *args)
                torch.cuda.synchronize()
                read_trace()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.call("dqn_net_layer", *args)
                e1.record()
                torch.cuda.synchronize()
                t = read_trace()
                name = f"{u['name']}.{['fwd', 'dgrad', 'wgrad'][phase]} b{batch}"
                ev = e0.elapsed_time(e1) * 1e3
                if len(t) == 0:
                    print(f"{name:18s} (no tcgen05 launch) event {ev:6.1f} us")
                    continue
                t0 = t[:, 2].min()
                span = (t[:, 6].max() - t0) / 1e3
                ph = np.diff(t[:, 2:7], axis=1) / 1e3       # setup, kloop, epi, fix
                start = (t[:, 2] - t0) / 1e3
                print(f"{name:18s} ctas {len(t):4d} sms {len(set(t[:, 1])):3d} nk {t[:, 7].min()}-{t[:, 7].max()} "
                      f"span {span:6.1f} event {ev:6.1f} | start max {start.max():5.1f} | "
                      + " ".join(f"{k} {ph[:, i].mean():5.1f}/{ph[:, i].max():5.1f}"
                                 for i, k in enumerate(("setup", "kloop", "epi", "fix"))))
                rel = lambda c: (t[:, c] - t[:, 3]) / 1e3          # noqa: E731  (from setup end)
                print(f"{'':18s} from setup end: first store {rel(8).mean():5.2f}  first full {rel(9).mean():5.2f}"
                      f"  last mma issued {rel(10).mean():5.2f}  done {rel(4).mean():5.2f}")
                # group 0 thread 0, k-blocks 0/2/4/6: enter put, empty ok, arrived, MMAs issued
                tk = t[:, 12:28].reshape(-1, 4, 4)
                parts = []
                for j in range(4):
                    ok = tk[:, j, 0] > 0
                    if not ok.any():
                        break
                    e = (tk[ok, j, :] - t[ok, 3][:, None]) / 1e3
                    parts.append(f"kb{2 * j}: " + "/".join(f"{e[:, c].mean():.2f}" for c in range(4)))
                print(f"{'':18s} " + "  ".join(parts))
                al = (t[:, 28] - t[:, 2]) / 1e3
                ps = (t[:, 29] - t[:, 2]) / 1e3
                print(f"{'':18s} setup split: tmem alloc done {al.mean():.2f}  pre-sync {ps.mean():.2f}  "
                      f"after pdl_wait {((t[:, 3] - t[:, 2]) / 1e3).mean():.2f} (us from entry)")
    net.flat_grads.zero_()


if __name__ == "__main__":
    for m in (sys.argv[1:] or ["0"]):
        main(int(m))
