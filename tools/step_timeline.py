"""Diagnostic: timeline of the tcgen05 GEMMs inside one CUDA-graph learner
update (cfg4, B = 32), from the trace build's per-CTA %globaltimer records.

    make -C paper_1804_05834_b200/csrc trace && python tools/step_timeline.py

Each line is one GEMM launch (graph node): CTAs, k-blocks per CTA, first CTA
entry and last CTA exit relative to the first entry of the update, and the
mean/max of the CTA phases (setup, k-loop, epilogue, split-K fixup).  Gaps
between GEMMs on a stream are the non-GEMM kernels (tree, gather, head, TD,
optimizer) and launch latency.
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
from paper_1804_05834_b200 import _lib  # noqa: E402


def read_trace():
    buf = (C.c_ulonglong * (8192 * 30))()
    n = _lib.lib.dqn_tc_trace(buf, 8192)
    return np.frombuffer(buf, dtype=np.uint64, count=30 * n).reshape(n, 30).astype(np.int64)


def main():
    _lib.lib.dqn_tc_trace.argtypes = [C.c_void_p, C.c_int]
    _lib.lib.dqn_tc_trace.restype = C.c_int
    cap = int(os.environ.get("CAP", "100000"))
    cfg = P.RunConfig(batch_size=32, beta_end_step=50_000_000)
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on)
    mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    mem.fill_synthetic(1, cap)
    rng = np.random.default_rng(0)
    for s in range(6):
        P.learn_step(on, tg, mem, opt, cfg, 1000 + s, rng)
    torch.cuda.synchronize()
    for rep in range(2):
        read_trace()
        P.learn_step(on, tg, mem, opt, cfg, 2000 + rep, rng)
        torch.cuda.synchronize()
        t = read_trace()
        t0 = t[:, 2].min()
        print(f"== update {rep}: {len(t)} CTA records, GEMM span {(t[:, 6].max() - t0) / 1e3:.1f} us")
        rows = []
        for lid in np.unique(t[:, 11]):
            r = t[t[:, 11] == lid]
            ph = np.diff(r[:, 2:7], axis=1) / 1e3
            rows.append(((r[:, 2].min() - t0) / 1e3, (r[:, 6].max() - t0) / 1e3, lid, len(r),
                         r[:, 7].min(), r[:, 7].max(), ph))
        for start, end, lid, n, k0, k1, ph in sorted(rows):
            print(f"  id {lid:4d} ctas {n:4d} nk {k0:2d}-{k1:2d}  {start:7.1f} -> {end:7.1f} "
                  f"({end - start:5.1f} us) | "
                  + " ".join(f"{k} {ph[:, i].mean():4.1f}/{ph[:, i].max():4.1f}"
                             for i, k in enumerate(("setup", "kloop", "epi", "fix"))))


if __name__ == "__main__":
    main()
