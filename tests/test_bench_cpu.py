"""bench.py contract checks that need no GPU: the reference (CPU) arm never
imports the package or loads libdqn_b200.so, both arms build the same
``config`` object, and ``--gpus N`` on a box with fewer GPUs refuses."""

import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def test_reference_arm_loads_no_library_of_ours():
    code = (
        "import sys, bench\n"
        "on, tg, mem, opt, lcfg, O = bench.cpu_learner('cfg1', 8)\n"
        "import numpy as np\n"
        "O.learn_step(on, tg, mem, opt, lcfg, 10, rng=np.random.default_rng(0))\n"
        "mods = [m for m in sys.modules if m.startswith('paper_1804_05834_b200')]\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(len(mods), 'libdqn_b200' in maps)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split()[-2:] == ["0", "False"], out.stdout


def test_both_arms_share_the_config_object():
    sys.path.insert(0, str(REPO))
    import bench
    a = bench.bench_config("cfg4", 1_000_000, 32, 1, "single")
    assert a["global_batch"] == 32 and a["parallelism"] == "single GPU"
    d = bench.bench_config("cfg4", 1_000_000, 32, 8, "dp")
    assert d["global_batch"] == 256 and d["parallelism"] == "dp8"

    class A:
        mode = "auto"
    assert bench.resolve_mode(A, 1) == "single" and bench.resolve_mode(A, 8) == "dp"


def test_gpus_more_than_visible_fails_loudly():
    import torch
    have = torch.cuda.device_count()
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(max(2, have + 1)), "--steps", "3"],
                         cwd=REPO, capture_output=True, text=True, timeout=300)
    assert out.returncode != 0
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "refusing" in line["error"]
