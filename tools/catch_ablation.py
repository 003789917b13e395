"""The reference's ablation criterion (pkg/tests/test_acceptance.py:276-309,
"criterion 09", soft) on the device learner: the four benchmark variants
(cli.py:30-35: double DQN, dueling, prioritized, dueling + prioritized) on
Catch, desk preset, 60,000 env steps, evaluation every 10,000, seeds 1-5;
steps to the first evaluation >= 0.8 per run; pass = the prioritized
variants' median <= the uniform variants' median.

usage: python tools/catch_ablation.py [out_dir]
"""
import csv
import json
import math
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1804_05834_b200 as P  # noqa: E402

VARIANTS = [("double DQN", False, 0.0), ("dueling double DQN", True, 0.0),
            ("double DQN with prioritized replay", False, 0.6),
            ("dueling double DQN with prioritized replay", True, 0.6)]


def main():
    out = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "ablation")
    res = {"criterion": "test_acceptance.py:276-309 (soft)", "runs": []}
    steps = {v[0]: [] for v in VARIANTS}
    t0 = time.perf_counter()
    for seed in (1, 2, 3, 4, 5):
        for label, dueling, alpha in VARIANTS:
            cfg = P.resolve_config({"preset": "desk", "env": "catch", "seed": seed,
                                    "dueling": dueling, "priority_alpha": alpha,
                                    "max_steps": 60_000, "test_period": 10_000,
                                    "beta_end_step": 60_000})
            d = out / f"{label.replace(' ', '_')}_s{seed}"
            d.mkdir(parents=True, exist_ok=True)
            with P.MetricsWriter(d / "metrics.csv") as sink:
                P.Trainer(cfg, sink=sink).run()
            rows = list(csv.reader(open(d / "metrics.csv", newline="")))
            evals = [(int(r[0]), float(r[7])) for r in rows[1:] if r[7]]
            hit = next((s for s, m in evals if m >= 0.8), math.inf)
            steps[label].append(hit)
            res["runs"].append({"variant": label, "seed": seed, "evals": evals,
                                "steps_to_0.8": None if hit == math.inf else hit})
            print(json.dumps(res["runs"][-1]), flush=True)
    pri = statistics.median(v for k, vs in steps.items() if "prioritized" in k for v in vs)
    uni = statistics.median(v for k, vs in steps.items() if "prioritized" not in k for v in vs)
    res["median_steps_to_0.8"] = {k: statistics.median(v) for k, v in steps.items()}
    res["prioritized_median"], res["uniform_median"] = pri, uni
    res["pass"] = pri <= uni
    res["elapsed_s"] = round(time.perf_counter() - t0, 1)
    (out / "summary.json").write_text(json.dumps(res, indent=1, default=str))
    print(json.dumps({k: res[k] for k in ("median_steps_to_0.8", "prioritized_median",
                                          "uniform_median", "pass", "elapsed_s")}, default=str))


if __name__ == "__main__":
    main()
