"""Diagnostic: kernel timeline of the learner's CUDA-graph update as it really
runs (concurrent streams, PDL overlap), from CUPTI activity records through
torch.profiler -- not serialised like ncu.

    python tools/graph_timeline.py [--cap N] [--reps R] [--json out.json]

Prints, for the last of R graph-replayed cfg4 updates, every kernel's start,
end and duration relative to the update's first kernel, its stream, and the
update's span.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_05834_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default="")
    ap.add_argument("--split-sample", action="store_true",
                    help="descent and frame gather as two launches (agent.FUSED_SAMPLE = False)")
    a = ap.parse_args()
    if a.split_sample:
        P.agent.FUSED_SAMPLE = False
    cfg = P.RunConfig(batch_size=32, beta_end_step=50_000_000)
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on)
    mem = P.PrioritizedReplay(a.cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    mem.fill_synthetic(1, a.cap)
    rng = np.random.default_rng(0)
    for s in range(8):
        P.learn_step(on, tg, mem, opt, cfg, 1000 + s, rng)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for s in range(a.reps):
            P.learn_step(on, tg, mem, opt, cfg, 2000 + s, rng)
            torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() >= 0]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", -1))
                 for e in ev if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()),
                key=lambda r: r[0])
    # split into updates at gaps > 20 us
    ups, cur = [], [ks[0]]
    for r in ks[1:]:
        if r[0] - max(x[1] for x in cur) > 20:
            ups.append(cur)
            cur = [r]
        else:
            cur.append(r)
    ups.append(cur)
    last = ups[-1]
    t0 = last[0][0]
    span = max(r[1] for r in last) - t0
    print(f"updates seen: {len(ups)}; spans (us): {[round(max(r[1] for r in u) - u[0][0], 1) for u in ups]}")
    print(f"last update: {len(last)} kernels, span {span:.1f} us")
    rows = []
    for s, e, n, st in last:
        nm = n.replace("void ", "").replace("dqn::", "").replace("(anonymous namespace)::", "")
        nm = nm.replace("tc::", "").replace("<unnamed>::", "")[:90]
        rows.append({"start": s - t0, "end": e - t0, "us": e - s, "stream": st, "name": nm})
        print(f"  {s - t0:7.1f} -> {e - t0:7.1f} ({e - s:5.1f} us) s{st:<4} {nm}")
    if a.json:
        Path(a.json).write_text(json.dumps({"span_us": span, "spans": [max(r[1] for r in u) - u[0][0] for u in ups],
                                            "kernels": rows}, indent=1))


if __name__ == "__main__":
    main()
