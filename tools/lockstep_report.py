"""Teacher-forced lockstep report: per step, the
worst per-tensor weight rel-norm error of the device learner vs the CPU
oracle, plus a free-running drift curve.  Run under both kernel families:
    python tools/lockstep_report.py            # tcgen05 trunk
    DQN_B200_ALGO=simt python tools/lockstep_report.py
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import deepq_oracle as O  # noqa: E402
from tests.helpers import oracle_learner, rel_norm  # noqa: E402
from tests.test_gpu_learner import CASES, device_learner, teacher_force  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402


def run(name, steps, free=False):
    kw = CASES[name]
    on, tg, mem, opt, cfg = device_learner(P, **kw)
    o_on, o_tg, o_mem, o_opt, o_cfg = oracle_learner(**kw)
    teacher_force(P, on, tg, mem, opt, o_on, o_tg, o_mem, o_opt)
    rows = []
    for st in range(steps):
        if not free:
            teacher_force(P, on, tg, mem, opt, o_on, o_tg, o_mem, o_opt)
        res = P.learn_step(on, tg, mem, opt, cfg, 100 + 4 * st, np.random.default_rng(500 + st))
        ores = O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, 100 + 4 * st,
                            rng=np.random.default_rng(500 + st))
        errs = {n: rel_norm(t.values.cpu().numpy(), o_on.params[n]) for n, t in on.named_tensors()}
        worst = max(errs, key=errs.get)
        rows.append((st, rel_norm(res.td_errors, ores["td_errors"]), worst, errs[worst]))
    return rows


if __name__ == "__main__":
    algo = os.environ.get("DQN_B200_ALGO", "tc")
    for name in ("cfg4", "cfg4_huber"):
        rows = run(name, 12)
        print(f"[{algo}] {name} lockstep: " + " ".join(f"{r[3]:.1e}({r[2].split('.')[0]}.{r[2].split('.')[1][0]})" for r in rows))
    rows = run("cfg4", 30, free=True)
    print(f"[{algo}] cfg4 free-running drift (worst tensor): " +
          " ".join(f"{r[0]}:{r[3]:.1e}" for r in rows if r[0] in (0, 1, 2, 5, 10, 20, 29)))
