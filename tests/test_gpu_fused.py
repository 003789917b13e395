"""GPU tests of the learner's fused launches against their unfused forms:

* dqn_head_td (both Q heads + TD block + head backward + head wgrad) vs the
  per-layer head kernels + dqn_td_loss (agent.py:58-73, 91-132);
* the apply-only optimizer (dqn_rmsprop_apply, gradients flagged by their
  producers) vs dqn_rmsprop_step, and its abort on a non-finite gradient
  raised inside a learner update;
* the two-phase head vs the last-CTA-ticket head, the fused sample+gather
  vs two launches.
"""

from __future__ import annotations


import numpy as np
import pytest

from tests.helpers import rel_norm

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def learner(P, dueling, double, per, huber=False, cap=64):
    cfg = P.RunConfig(double=double, dueling=dueling, huber=huber, batch_size=32,
                      beta_end_step=1000, priority_alpha=0.6 if per else 0.0)
    on = P.build_network("atari", (84, 84, 4), 4, dueling)
    tg = P.build_network("atari", (84, 84, 4), 4, dueling)
    P.init_params(on, 1)
    P.init_params(tg, 2)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    if per:
        mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    else:
        mem = P.ReplayMemory(cap, (84, 84, 4))
    mem.fill_synthetic(7, cap)
    return on, tg, mem, opt, cfg


CASES = {
    "cfg1": dict(dueling=False, double=False, per=False),
    "cfg3": dict(dueling=False, double=True, per=True),
    "cfg4": dict(dueling=True, double=True, per=True),
    "cfg4_huber": dict(dueling=True, double=True, per=True, huber=True),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fused_head_matches_per_layer_head(P, name, monkeypatch):
    runs = []
    for fused in ("1", "0"):
        monkeypatch.setattr(P.agent, "FUSED_HEAD", fused == "1")
        on, tg, mem, opt, cfg = learner(P, **CASES[name])
        rng = np.random.default_rng(3)
        res = [P.learn_step(on, tg, mem, opt, cfg, 10, rng)]
        runs.append((res, on.flat_values.cpu().numpy().copy()))
    (fa, wa), (fb, wb) = runs
    for ra, rb in zip(fa, fb):
        # the Q heads reduce in a different (fixed) order; TD block identical
        assert rel_norm(ra.td_errors, rb.td_errors) < 1e-5
        assert rel_norm(ra.targets, rb.targets) < 1e-5
        assert rel_norm(ra.losses, rb.losses) < 1e-5
    # one update from identical state (RMSprop amplifies re-ordering over steps)
    assert rel_norm(wa, wb) < 1e-5


def test_rmsprop_apply_equals_step_on_finite_gradients(P):
    a = P.build_network("desk", (24, 24, 4), 3, True)
    b = P.build_network("desk", (24, 24, 4), 3, True)
    P.init_params(a, 0)
    P.init_params(b, 0)
    oa, ob = P.RmsProp(a), P.RmsProp(b)
    g = torch.Generator(device="cuda").manual_seed(5)
    for _ in range(3):
        grad = torch.randn(a.flat_grads.shape, device="cuda", generator=g) * 1e-2
        a.flat_grads.copy_(grad)
        b.flat_grads.copy_(grad)
        oa.step()
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        ob.enqueue_apply(flags)
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
    assert torch.equal(a.flat_values, b.flat_values)
    assert torch.equal(oa.flat_acc, ob.flat_acc)
    assert torch.all(b.flat_grads == 0)


def test_learner_aborts_on_gradient_overflow(P):
    """Finite Q-values but rewards so large that the head's weight gradient
    overflows fp32: the producing launch flags it, the apply-only optimizer
    skips the update, learn_step raises (optim.py:38-40 semantics)."""
    on, tg, mem, opt, cfg = learner(P, dueling=True, double=True, per=True)
    mem.memory.rewards.fill_(1e38)
    before, acc = on.flat_values.clone(), opt.flat_acc.clone()
    with pytest.raises(P.NonFiniteError):
        P.learn_step(on, tg, mem, opt, cfg, 10, np.random.default_rng(0))
    assert torch.equal(before, on.flat_values)
    assert torch.equal(acc, opt.flat_acc)


@pytest.mark.parametrize("name", ["cfg4", "cfg4_huber", "cfg1"])
def test_head_two_phase_matches_last_cta_form(P, name, monkeypatch):
    """The two-phase head (Q heads, then every CTA recomputes the TD block)
    against the last-CTA-ticket form: same formulas, sums in another fixed
    order (1e-5, as the fused vs per-layer head)."""
    runs = []
    for two in ("1", "0"):
        monkeypatch.setattr(P.agent, "HEAD_TWO_PHASE", two == "1")
        on, tg, mem, opt, cfg = learner(P, **CASES[name])
        res = P.learn_step(on, tg, mem, opt, cfg, 10, np.random.default_rng(3))
        runs.append((res, on.flat_values.clone()))
    (ra, wa), (rb, wb) = runs
    for f in ("targets", "td_errors", "losses"):
        assert rel_norm(getattr(ra, f), getattr(rb, f)) < 1e-5, f
    assert rel_norm(wa.cpu().numpy(), wb.cpu().numpy()) < 1e-5


def test_fused_sample_gather_matches_two_launches(P, monkeypatch):
    """dqn_sample_gather (descent + IS weights + frame gather in one launch)
    against dqn_tree_sample + dqn_ring_gather: identical indices, weights,
    gathered batch and update."""
    runs = []
    for fused in ("1", "0"):
        monkeypatch.setattr(P.agent, "FUSED_SAMPLE", fused == "1")
        on, tg, mem, opt, cfg = learner(P, **CASES["cfg4"])
        rng = np.random.default_rng(8)
        res = [P.learn_step(on, tg, mem, opt, cfg, 10 + s, rng) for s in range(3)]
        plan = next(p for p in P.agent._PLANS.values() if p.online is on)
        assert plan.fused_sample == (fused == "1")
        runs.append((res, plan.idx.clone(), plan.w.clone(), plan.x.clone(), plan.a.clone(),
                     on.flat_values.clone(), mem.tree.nodes.clone()))
    a, b = runs
    for ra, rb in zip(a[0], b[0]):
        assert np.array_equal(ra.td_errors, rb.td_errors)
    for ta, tb in zip(a[1:], b[1:]):
        assert torch.equal(ta, tb)


def test_fused_sample_gather_zero_total_raises(P):
    on, tg, mem, opt, cfg = learner(P, **CASES["cfg4"])
    mem.tree.load_leaves(np.zeros(mem.capacity))
    with pytest.raises(ValueError):
        P.learn_step(on, tg, mem, opt, cfg, 10, np.random.default_rng(0))
