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


def test_reference_arm_under_torchrun_world2():
    """The driver launches `--impl reference` like our arm (torchrun, N ranks):
    rank 0 alone prints the cfg5 comparator line (global batch 32 N in one
    process, value in batch-32 updates/s), the other ranks exit 0."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1",
                          f"--master-port={port}", "bench.py", "--impl", "reference", "--gpus", "2",
                          "--steps", "3", "--warmup", "3"],
                         cwd=REPO, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["global_batch"] == 64 and d["config"]["parallelism"] == "dp2"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
