"""The reference's end-to-end learning criterion (pkg/tests/test_acceptance.py
:253-273, "criterion 08") on the device learner: desk preset, Catch, dueling,
priority alpha 0.6, 200,000 env steps per seed, seeds 1-5; pass = final
evaluation mean >= 0.9 for at least 4 of 5 seeds and every seed under 1800 s.

Each seed writes <out>/seed<N>/metrics.csv (the reference's CSV layout) and
the summary goes to <out>/summary.json.

usage: python tools/catch_acceptance.py [out_dir] [seeds=1,2,3,4,5] [max_steps]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1804_05834_b200 as P  # noqa: E402


def main():
    out = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "catch")
    seeds = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,4,5").split(",")]
    over = {"preset": "desk", "env": "catch", "dueling": True, "priority_alpha": 0.6}
    if len(sys.argv) > 3:
        over["max_steps"] = int(sys.argv[3])
    summary = {"criterion": "test_acceptance.py:253-273 (desk preset, catch, 200k steps, "
                            ">= 4/5 seeds final eval >= 0.9, each < 1800 s)", "seeds": []}
    for seed in seeds:
        cfg = P.resolve_config({**over, "seed": seed})
        d = out / f"seed{seed}"
        d.mkdir(parents=True, exist_ok=True)
        t0 = time.perf_counter()
        with P.MetricsWriter(d / "metrics.csv") as sink:
            tr = P.Trainer(cfg, sink=sink)
            tr.run()
        el = time.perf_counter() - t0
        evals = []
        import csv
        with open(d / "metrics.csv", newline="") as fh:
            rows = list(csv.reader(fh))
        evals = [(int(r[0]), float(r[7])) for r in rows[1:] if r[7]]
        rec = {"seed": seed, "elapsed_s": round(el, 1), "learn_steps": tr.learn_steps,
               "episodes": tr.episode, "evals": evals,
               "final_eval": evals[-1][1] if evals else None,
               "env_steps_per_s": round(cfg.max_steps / el, 1)}
        summary["seeds"].append(rec)
        print(json.dumps(rec), flush=True)
    finals = [s["final_eval"] for s in summary["seeds"]]
    summary["good"] = sum(1 for f in finals if f is not None and f >= 0.9)
    summary["max_elapsed_s"] = max(s["elapsed_s"] for s in summary["seeds"])
    # the criterion is defined over the five seeds 1-5
    summary["pass"] = (bool(summary["good"] >= 4 and summary["max_elapsed_s"] < 1800.0)
                       if sorted(seeds) == [1, 2, 3, 4, 5] else None)
    (out / "summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: summary[k] for k in ("good", "max_elapsed_s", "pass")}))


if __name__ == "__main__":
    main()
