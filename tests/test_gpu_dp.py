"""Data-parallel learner on the GPU backend (NCCL).  Only one GPU is
available in this run, so the multi-rank protocol is covered by the gloo
test (tests/test_dp_gloo.py); here world size 1 must reproduce the
single-GPU ``learn_step`` (same queries, clip and descent; IS weights from
numpy pow instead of device pow, so TD errors agree to ~1e-12)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    import paper_1804_05834_b200 as P
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield P


def _learner(P, seed=7, cap=256):
    from tests.test_gpu_learner import device_learner
    return device_learner(P, dueling=True, double=True, per=True, cap=cap, seed=seed)


def test_dp_world1_equals_learn_step(P):
    from paper_1804_05834_b200 import dp
    on, tg, mem, opt, cfg = _learner(P)
    on2, tg2, mem2, opt2, cfg2 = _learner(P)
    be = dp.DeviceBackend(on2, tg2, mem2, opt2, cfg2)
    learner = dp.DataParallelLearner(be, 32, 0.6, 0.01, "cuda")
    rng_a, rng_b = np.random.default_rng(5), np.random.default_rng(5)
    for s in range(4):
        res = P.learn_step(on, tg, mem, opt, cfg, 100 + s, rng_a)
        plan = next(p for p in P.agent._PLANS.values() if p.online is on)
        r = learner.step(rng_b.random(32), mem2.beta(100 + s))
        assert np.array_equal(r.indices, plan.idx.cpu().numpy())
        assert np.allclose(r.weights, plan.w.cpu().numpy(), rtol=1e-14, atol=0)
        assert np.allclose(r.td_errors, res.td_errors, rtol=1e-9, atol=1e-12)
    d = (on.flat_values - on2.flat_values).abs().max().item()
    assert d <= 1e-6
    assert np.allclose(mem.tree.nodes.cpu().numpy(), mem2.tree.nodes.cpu().numpy(), rtol=1e-9)
