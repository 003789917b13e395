"""The reference's own acceptance / unit cases for the learner path, run on
the device implementation (same parameters and bars as the reference's
tests; the reference files are not imported -- they do not travel to the GPU
box):

* criterion 03, prioritized-sampling fidelity (pkg/tests/test_acceptance.py:123-157);
* criterion 04, sum-tree consistency after 1e5 random operations (:160-178);
* criterion 05, the importance-weight contract (:181-203);
* criterion 07, the dueling identity (:232-250);
* learn_step's output-gradient convention, loss = 1/2 w delta^2, and a single
  transition's |delta| shrinking monotonically (pkg/tests/test_agent.py:262-294).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def _blank_memory(P, n, alpha):
    cfg = P.PriorityConfig(alpha, 0.01, P.LinearSchedule(0.4, 1.0, 100))
    mem = P.PrioritizedReplay(n, (1, 1, 1), cfg, dtype=np.float32)
    blank = np.zeros((1, 1, 1), dtype=np.float32)
    for _ in range(n):
        mem.store(P.Transition(blank, 0, 0.0, blank, False))
    return mem, cfg


def _frequency_run(P, raw, alpha, draws, rng):
    n = len(raw)
    mem, cfg = _blank_memory(P, n, alpha)
    mem.update_priorities(np.arange(n), raw - cfg.epsilon)    # stored raw priority = raw
    counts = np.zeros(n)
    per_call = 100_000
    for _ in range(draws // per_call):
        batch = mem.sample(per_call, beta=0.4, rng=rng)
        counts += np.bincount(batch.indices.cpu().numpy(), minlength=n)
    exact = raw ** alpha / np.sum(raw ** alpha)
    return counts / draws, exact


def test_criterion03_prioritized_sampling_fidelity(P):
    rng = np.random.default_rng(7)
    for alpha in (0.6, 1.0):
        for _ in range(20):
            raw = rng.uniform(0.05, 5.0, size=64)
            freq, exact = _frequency_run(P, raw, alpha, 1_000_000, rng)
            assert float(np.abs(freq - exact).sum()) < 0.02, alpha
    raw = rng.uniform(0.05, 5.0, size=64)
    freq, _ = _frequency_run(P, raw, 0.0, 1_000_000, rng)
    assert np.max(np.abs(freq - 1.0 / 64)) < 0.01


def test_criterion04_sum_tree_consistency(P):
    rng = np.random.default_rng(11)
    cfg = P.PriorityConfig(0.6, 0.01, P.LinearSchedule(0.4, 1.0, 100))
    mem = P.PrioritizedReplay(512, (1, 1, 1), cfg, dtype=np.float32)
    blank = np.zeros((1, 1, 1), dtype=np.float32)
    for _ in range(100_000):
        if mem.size == 0 or rng.random() < 0.4:            # stores evict once full
            mem.store(P.Transition(blank, 0, 0.0, blank, False))
        else:
            idx = rng.integers(0, mem.size, size=8)
            mem.update_priorities(idx, rng.random(8) * 10.0)
    nodes = mem.tree.nodes.cpu().numpy()
    internal = np.arange(1, mem.tree._leaf_base)
    child_sums = nodes[2 * internal] + nodes[2 * internal + 1]
    # the reference's bar is rel 1e-6; every node here is exactly left + right
    assert np.array_equal(nodes[internal], child_sums)
    assert mem.tree.total == pytest.approx(float(mem.tree.leaves().sum()), rel=1e-9)


def test_criterion05_importance_weight_contract(P):
    rng = np.random.default_rng(13)
    mem, _ = _blank_memory(P, 64, 0.6)
    mem.update_priorities(np.arange(64), rng.uniform(0.0, 4.0, 64))
    for _ in range(50):
        w = mem.sample(32, beta=rng.uniform(0.1, 1.0), rng=rng).weights.cpu().numpy()
        assert w.max() == 1.0
        assert np.all((w > 0.0) & (w <= 1.0))
    assert np.all(mem.sample(32, beta=0.0, rng=rng).weights.cpu().numpy() == 1.0)
    uniform, _ = _blank_memory(P, 64, 0.6)
    for beta in (0.0, 0.4, 0.7, 1.0):
        assert np.all(uniform.sample(32, beta=beta, rng=rng).weights.cpu().numpy() == 1.0)
    sched = P.resolve_config().beta_schedule()
    assert sched.value(0) == 0.4 and sched.value(100_000_000) == 1.0


def _tiny_trunk(P):
    return [P.LayerSpec("convolution", {"filters": 2, "filter_h": 2, "filter_w": 2,
                                        "stride_h": 2, "stride_w": 2}),
            P.LayerSpec.relu(), P.LayerSpec.linear(8), P.LayerSpec.relu()]


def test_criterion07_dueling_identity(P):
    net = P.build_network(_tiny_trunk(P), (6, 6, 2), 3, True)
    P.init_params(net, 3)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((100, 6, 6, 2)).astype(np.float32)
    t = dict(net.named_tensors())
    q = net.forward(x).double()
    h = net._cur.act[-2][:100 * 8].view(100, 8).double()          # head input
    v = h @ t["duel.value.weight"].values.double() + t["duel.value.bias"].values.double()
    # the advantage is mean-centred: Q - V sums to zero over the actions
    assert float((q - v).sum(dim=1).abs().max()) < 1e-5
    # a constant advantage across actions collapses Q to V
    t["duel.advantage.weight"].values.copy_(
        torch.as_tensor(rng.standard_normal((8, 1)), device="cuda").float().expand(8, 3))
    t["duel.advantage.bias"].values.fill_(0.37)
    q = net.forward(x).double()
    h = net._cur.act[-2][:100 * 8].view(100, 8).double()
    v = h @ t["duel.value.weight"].values.double() + t["duel.value.bias"].values.double()
    assert float((q - v).abs().max()) < 1e-5


def _pair(P, lr=0.000625, batch=8, cap=64, alpha=0.6):
    cfg = P.RunConfig(batch_size=batch, learning_rate=lr, double=True, dueling=True,
                      priority_alpha=alpha, beta_end_step=1000)
    on = P.build_network(_tiny_trunk(P), (6, 6, 2), 3, True)
    tg = P.build_network(_tiny_trunk(P), (6, 6, 2), 3, True)
    P.init_params(on, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    mem = P.PrioritizedReplay(cap, (6, 6, 2), P.PriorityConfig(alpha, 0.01, cfg.beta_schedule()),
                              dtype=np.float32)
    return on, tg, mem, opt, cfg


def _fill(P, mem, n, seed=0):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        s = rng.random((6, 6, 2)).astype(np.float32)
        s2 = rng.random((6, 6, 2)).astype(np.float32)
        mem.store(P.Transition(s, int(rng.integers(0, 3)), float(rng.standard_normal()), s2,
                               bool(rng.random() < 0.2)))


def test_output_gradient_convention(P):
    """d(1/2 w delta^2)/dQ(s, a) = -w delta on the sampled action, 0 elsewhere;
    priorities are uniform before the first update, so w = 1."""
    on, tg, mem, opt, cfg = _pair(P)
    _fill(P, mem, 16)
    res = P.learn_step(on, tg, mem, opt, cfg, 50, np.random.default_rng(1))
    yg = on.y.grad.cpu().numpy().astype(np.float64)
    assert np.count_nonzero(yg) <= cfg.batch_size
    sampled = np.argmax(np.abs(yg), axis=1)
    np.testing.assert_allclose(yg[np.arange(cfg.batch_size), sampled], -res.td_errors, rtol=1e-6)
    z = yg.copy()
    z[np.arange(cfg.batch_size), sampled] = 0.0
    assert np.all(z == 0.0)
    np.testing.assert_allclose(res.losses, 0.5 * res.td_errors ** 2, rtol=1e-12)


def test_single_transition_delta_shrinks_monotonically(P):
    # the reference's setup_pair (test_agent.py:227-241): plain head, online
    # init seed 0, target synced from it, uniform replay, DQN target, lr 1e-3
    cfg = P.RunConfig(batch_size=4, gamma=0.99, double=False, learning_start=4,
                      learning_rate=0.001, priority_alpha=0.0)
    on = P.build_network(_tiny_trunk(P), (6, 6, 2), 3, False)
    tg = P.build_network(_tiny_trunk(P), (6, 6, 2), 3, False)
    P.init_params(on, 0)
    P.init_params(tg, 1)
    P.sync_target(on, tg)
    opt = P.RmsProp(on, 0.001)
    mem = P.ReplayMemory(64, (6, 6, 2), dtype=np.float32)
    s = np.random.default_rng(3).random((6, 6, 2)).astype(np.float32)
    mem.store(P.Transition(s, 1, 1.0, s, True))
    rng = np.random.default_rng(4)
    deltas = [P.learn_step(on, tg, mem, opt, cfg, i, rng).mean_abs_td for i in range(100)]
    assert all(b <= a + 1e-7 for a, b in zip(deltas, deltas[1:]))
    assert deltas[-1] < 1e-3 < deltas[0]


class _TableNet:
    """Q-table lookup 'network' (the reference test's TableNet): forward maps
    integer state indices to Q rows."""

    def __init__(self, table):
        self.table = np.asarray(table, dtype=np.float64)
        self.output_shape = (self.table.shape[1],)

    def forward(self, states):
        return self.table[np.asarray(states, dtype=np.int64)]


def _value_iteration(trans, rew, term, gamma, tol=1e-10):
    q = np.zeros((len(trans), len(trans[0])))
    while True:
        prev = q.copy()
        for s in range(len(trans)):
            for a in range(len(trans[0])):
                q[s, a] = rew[s][a] + (0.0 if term[s][a] else gamma * prev[trans[s][a]].max())
        if np.max(np.abs(q - prev)) < tol:
            return q


def _batch(P, rewards, next_states, terminals, actions=None):
    k = len(rewards)
    return P.SampleBatch(states=np.zeros(k), actions=np.zeros(k, np.int64) if actions is None
                         else np.asarray(actions), rewards=np.asarray(rewards, np.float64),
                         next_states=np.asarray(next_states),
                         terminals=np.asarray(terminals, bool), indices=np.arange(k),
                         probabilities=np.full(k, 1.0 / k), weights=np.ones(k))


def test_criterion06_bellman_target_oracle(P):
    """compute_target_dqn / _double on the exact Q* of TabularChain reproduce
    Q* (the Bellman fixed point, test_acceptance.py:206-229); the Double-DQN
    bootstrap never exceeds the max bootstrap over 10k random rows."""
    env = P.TabularChain()
    gamma = 0.99
    q_star = _value_iteration(env.TRANSITIONS, env.REWARDS, env.TERMINAL, gamma)
    net = _TableNet(q_star)
    for s in (1, 2, 3):
        for a in (0, 1):
            b = _batch(P, [env.REWARDS[s][a]], [env.TRANSITIONS[s][a]], [env.TERMINAL[s][a]], [a])
            y_dqn = float(P.compute_target_dqn(b, net, gamma)[0])
            y_double = float(P.compute_target_double(b, net, net, gamma)[0])
            assert abs(y_dqn - q_star[s, a]) < 1e-6       # Q in fp32 on the device
            assert abs(y_double - q_star[s, a]) < 1e-6
    rng = np.random.default_rng(17)
    k = 10_000
    online = _TableNet(rng.standard_normal((k, 5)))
    target = _TableNet(rng.standard_normal((k, 5)))
    b = _batch(P, rng.standard_normal(k), np.arange(k), np.zeros(k, dtype=bool))
    yd = P.compute_target_double(b, online, target, 0.99).cpu().numpy()
    ym = P.compute_target_dqn(b, target, 0.99).cpu().numpy()
    assert np.all(yd <= ym + 1e-12)
