"""A small checkpoint written by the UNMODIFIED reference
(deepq/checkpoint.py save_checkpoint), plus its arrays as .npz, so the CYRL
loader is pinned where the reference is absent:

    python tests/golden/make_ckpt_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))

from deepq import checkpoint as RK  # noqa: E402
from deepq.config import resolve_config  # noqa: E402

from tests.test_checkpoint_cpu import sample_ckpt  # noqa: E402

if __name__ == "__main__":
    c = sample_ckpt(resolve=resolve_config, Ck=RK.Checkpoint)
    RK.save_checkpoint(HERE / "ref_small.ckpt", c)
    arrays = {"frames": c.frames}
    for sec in ("params", "target", "optim", "memory"):
        for k, v in getattr(c, sec).items():
            arrays[f"{sec}/{k}"] = np.asarray(v)
    np.savez_compressed(HERE / "ref_small_arrays.npz", **arrays)
