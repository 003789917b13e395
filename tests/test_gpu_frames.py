"""GPU tests of the device frame pipeline (dqn_preprocess_frames,
frames.py): bit-exact against the reference's own
preprocess_frame / Preprocessor outputs (tests/golden/envs.npz, made by
make_trainer_golden.py from the unmodified reference) and against the host
restatement on larger random batches."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_05834_b200 import frames as F
    return F


def test_reference_golden_frames_bit_exact(F, golden):
    g = golden("envs")
    for i in range(6):
        f = g[f"pre{i}_in"]
        size = tuple(int(s) for s in g[f"pre{i}_size"])
        got = F.preprocess_frames(f[None], size).cpu().numpy()[0]
        assert np.array_equal(got, g[f"pre{i}_out"]), i


def test_reference_golden_stack_bit_exact(F, golden):
    g = golden("envs")
    pre = F.DevicePreprocessor((6, 5), 3)
    seq = g["stack_in"]
    got = [pre.reset(seq[0]).cpu().numpy()] + [pre.push(s).cpu().numpy() for s in seq[1:]]
    assert np.array_equal(np.stack(got), g["stack_out"])


@pytest.mark.parametrize("shape,size", [((16, 210, 160, 3), (84, 84)), ((5, 10, 7), (24, 24)),
                                        ((3, 24, 24), (24, 24)), ((4, 40, 30, 1), (17, 23)),
                                        ((2, 8, 8, 3), (24, 24)), ((2, 1, 5), (24, 24))])
def test_batches_match_host_restatement(F, shape, size):
    from paper_1804_05834_b200.envs import preprocess_frame
    rng = np.random.default_rng(sum(shape))
    x = rng.integers(0, 256, size=shape, dtype=np.uint8)
    got = F.preprocess_frames(torch.as_tensor(x, device="cuda"), size).cpu().numpy()
    want = np.stack([preprocess_frame(f, size) for f in x])
    assert got.dtype == np.float32 and np.array_equal(got, want)


def test_bad_frames_rejected(F):
    with pytest.raises(ValueError):
        F.preprocess_frames(np.zeros((2, 4, 4, 2), dtype=np.uint8), (3, 3))
    with pytest.raises(ValueError):
        F.preprocess_frames(np.zeros((2, 4, 4), dtype=np.float32), (3, 3))
