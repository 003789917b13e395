"""CPU oracle for the DQN learner hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference ``deepq`` learner
update (``/root/reference/pkg/src/deepq``).  It exists for three reasons and no
others:

* the ``-m gpu`` parity tests compare the CUDA path against it on identical
  inputs (the reference itself is absent on the GPU box);
* ``__graft_entry__.smoke()`` checks one small CUDA invocation against it;
* ``bench.py`` times it as the CPU baseline (``cpu_baseline.kind = "port"``).

The product package (``paper_1804_05834_b200``) never imports this file.

Parity pin: the restatement is checked against golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py``, fixtures in
``tests/golden/*.npz``) and, when ``/root/reference`` is mounted, directly
against the live reference (``tests/test_oracle_pin.py``).

Each function names the reference lines it restates.  Arithmetic order is kept
wherever the north star asks for bit-exactness (sum tree, sampling, priority
update, RMSprop); network GEMMs are fp32 numpy/BLAS like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# errors (restates deepq/errors.py:4-41, only the ones the hot path raises)
# ---------------------------------------------------------------------------


class OracleGeometryError(Exception):
    pass


class OracleNonFiniteError(Exception):
    pass


# ---------------------------------------------------------------------------
# schedules (restates deepq/schedules.py:17-23)
# ---------------------------------------------------------------------------


def linear_value(start: float, end: float, end_step: int, step: int) -> float:
    """Clamped linear interpolation, schedules.py:17-23."""
    if step < 0:
        raise ValueError("negative step")
    if end_step <= 0 or step >= end_step:
        return end
    return start + (end - start) * (step / end_step)


# ---------------------------------------------------------------------------
# fp64 sum tree (restates deepq/replay.py:127-181)
# ---------------------------------------------------------------------------


class HeapTree:
    """1-indexed fp64 heap: ``nodes[base + i]`` is leaf i, ``nodes[n]`` the
    sum of its two children (replay.py:137-143)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = int(capacity)
        # replay.py:141 -- depth = max(1, ceil(log2 cap))
        self.depth = max(1, int(np.ceil(np.log2(capacity))))
        self.base = 1 << self.depth
        self.nodes = np.zeros(2 * self.base, dtype=np.float64)

    @property
    def total(self) -> float:
        return float(self.nodes[1])

    def leaves(self) -> np.ndarray:
        return self.nodes[self.base:self.base + self.capacity]

    def put(self, i: int, value: float) -> None:
        """replay.py:155-165 -- write leaf, recompute each ancestor from its
        two children (no incremental deltas)."""
        if not 0 <= i < self.capacity:
            raise IndexError(f"leaf {i} out of range")
        if value < 0 or not math.isfinite(value):
            raise ValueError("bad priority")
        n = self.base + i
        self.nodes[n] = value
        n >>= 1
        while n:
            self.nodes[n] = self.nodes[2 * n] + self.nodes[2 * n + 1]
            n >>= 1

    def rebuild(self) -> None:
        """Bottom-up rebuild; identical to any sequence of ``put`` calls that
        leaves the same leaves (internal nodes are a pure function of the
        leaves -- SURVEY Appendix B)."""
        lo = self.base
        while lo > 1:
            hi = lo
            lo >>= 1
            self.nodes[lo:hi] = self.nodes[2 * lo:2 * hi:2] + self.nodes[2 * lo + 1:2 * hi:2]

    def descend(self, queries) -> np.ndarray:
        """replay.py:167-181 -- clipped query, per-level compare/subtract."""
        total = self.nodes[1]
        if total <= 0:
            raise ValueError("zero total priority")
        q = np.asarray(queries, dtype=np.float64).copy()
        q = np.minimum(np.maximum(q, 1e-300), np.nextafter(total, 0))
        node = np.ones(q.shape, dtype=np.int64)
        for _ in range(self.depth):
            child = node * 2
            lsum = self.nodes[child]
            right = q > lsum
            q = q - lsum * right
            node = child + right
        return node - self.base


# ---------------------------------------------------------------------------
# replay (restates deepq/replay.py:74-124, 184-241)
# ---------------------------------------------------------------------------


@dataclass
class Batch:
    states: np.ndarray
    actions: np.ndarray
    rewards: np.ndarray
    next_states: np.ndarray
    terminals: np.ndarray
    indices: np.ndarray
    probabilities: np.ndarray
    weights: np.ndarray


class Ring:
    """FIFO ring (replay.py:74-102).  Frames are kept as uint8 and lifted to
    float32 at gather time with the pixel rule of envs.py:300-302,311
    (``float32(float64(u8) / 255)``), which yields exactly the float32 values
    the reference would have stored.  ``float_states`` keeps raw float32
    states (generic state shapes, as the reference tests use)."""

    def __init__(self, capacity: int, state_shape, float_states: bool = False):
        self.capacity = int(capacity)
        self.state_shape = tuple(state_shape)
        dt = np.float32 if float_states else np.uint8
        self.states = np.zeros((capacity,) + self.state_shape, dtype=dt)
        self.next_states = np.zeros_like(self.states)
        self.actions = np.zeros(capacity, dtype=np.int64)
        self.rewards = np.zeros(capacity, dtype=np.float64)
        self.terminals = np.zeros(capacity, dtype=bool)
        self.cursor = 0
        self.size = 0

    def store(self, s, a, r, s2, t) -> int:
        i = self.cursor
        self.states[i] = s
        self.next_states[i] = s2
        self.actions[i] = a
        self.rewards[i] = r
        self.terminals[i] = t
        self.cursor = (i + 1) % self.capacity
        self.size = min(self.size + 1, self.capacity)
        return i

    @staticmethod
    def lift(frames: np.ndarray) -> np.ndarray:
        if frames.dtype == np.uint8:
            return (frames.astype(np.float64) / 255.0).astype(np.float32)
        return frames.astype(np.float32, copy=True)

    def gather(self, idx, prob, w) -> Batch:
        """replay.py:104-115."""
        return Batch(self.lift(self.states[idx]), self.actions[idx],
                     self.rewards[idx].copy(), self.lift(self.next_states[idx]),
                     self.terminals[idx], idx, prob, w)


def uniform_sample(ring: Ring, k: int, rng: np.random.Generator) -> Batch:
    """replay.py:117-124."""
    if ring.size == 0:
        raise ValueError("empty replay")
    idx = rng.integers(0, ring.size, size=k)
    return ring.gather(idx, np.full(k, 1.0 / ring.size), np.ones(k))


def per_indices(tree: HeapTree, size: int, k: int, beta: float, u: np.ndarray):
    """replay.py:215-229 given the uniforms ``u`` (= ``rng.random(k)``)."""
    if size == 0:
        raise ValueError("empty replay")
    total = tree.total
    if total <= 0:
        raise ValueError("zero total priority")
    seg = total / k
    q = (np.arange(k) + np.asarray(u, dtype=np.float64)) * seg
    idx = tree.descend(q)
    prob = tree.leaves()[idx] / total
    w = np.power(size * prob, -beta)
    w = w / w.max()
    return idx, prob, w


class PerReplay:
    """Ring + heap tree (replay.py:184-241)."""

    def __init__(self, capacity, state_shape, alpha=0.6, eps=0.01,
                 beta=(0.4, 1.0, 100_000_000), float_states=False):
        self.ring = Ring(capacity, state_shape, float_states)
        self.tree = HeapTree(capacity)
        self.alpha, self.eps = float(alpha), float(eps)
        self.beta_sched = beta
        self.max_priority = 1.0

    @property
    def size(self):
        return self.ring.size

    def store(self, s, a, r, s2, t) -> int:
        i = self.ring.store(s, a, r, s2, t)
        self.tree.put(i, self.max_priority ** self.alpha)
        return i

    def beta(self, step: int) -> float:
        return linear_value(*self.beta_sched, step)

    def sample(self, k: int, beta: float, rng=None, u=None) -> Batch:
        if self.size == 0:
            raise ValueError("empty replay")
        if u is None:
            u = rng.random(k)
        idx, prob, w = per_indices(self.tree, self.size, k, beta, u)
        return self.ring.gather(idx, prob, w)

    def update_priorities(self, idx, td) -> None:
        """replay.py:232-241: batch order, last write wins, partial update
        before an out-of-range index raises."""
        idx = np.asarray(idx)
        p = np.abs(np.asarray(td, dtype=np.float64)) + self.eps
        for i, raw in zip(idx, p):
            if not 0 <= i < self.size:
                raise IndexError(f"index {i} out of range [0, {self.size})")
            self.tree.put(int(i), float(raw) ** self.alpha)
        self.max_priority = max(self.max_priority, float(p.max()))


# ---------------------------------------------------------------------------
# Q-network (restates deepq/layers.py and deepq/network.py)
# ---------------------------------------------------------------------------

ATARI_TRUNK = [("conv", 32, 8, 4), ("relu",), ("conv", 64, 4, 2), ("relu",),
               ("conv", 64, 3, 1), ("relu",), ("fc", 512), ("relu",)]
DESK_TRUNK = [("conv", 16, 6, 2), ("relu",), ("conv", 32, 3, 1), ("relu",),
              ("fc", 128), ("relu",)]                  # network.py:21-40


class QNet:
    """Functional restatement of Network + layers (network.py:45-205,
    layers.py:99-330).  ``params`` is the registry (name -> array) in the
    reference's order (network.py:74-84); activations of the last forward are
    cached for backward / wgrad."""

    def __init__(self, trunk, input_shape, n_actions, dueling, dtype=np.float32):
        self.dtype = np.dtype(dtype)
        self.input_shape = tuple(input_shape)
        self.n_actions = n_actions
        self.ops = []            # (kind, name, geometry)
        self.params: dict[str, np.ndarray] = {}
        h, w, c = input_shape
        shape = (h, w, c)
        counters = {}
        spec = list(trunk) + ([("duel", n_actions)] if dueling else [("fc", n_actions)])
        for item in spec:
            kind = item[0]
            counters[kind] = counters.get(kind, 0) + 1
            name = "duel" if kind == "duel" else f"{kind}{counters[kind]}"
            if kind == "conv":
                _, cout, f, s = item
                hh, ww, cc = shape
                if hh < f or ww < f or (hh - f) % s or (ww - f) % s:
                    raise OracleGeometryError(f"{name}: infeasible geometry")
                oh, ow = (hh - f) // s + 1, (ww - f) // s + 1
                self.params[name + ".weight"] = np.zeros((f, f, cc, cout), self.dtype)
                self.params[name + ".bias"] = np.zeros((cout,), self.dtype)
                self.ops.append(("conv", name, (f, s)))
                shape = (oh, ow, cout)
            elif kind == "relu":
                self.ops.append(("relu", name, None))
            elif kind == "fc":
                feat = int(np.prod(shape))
                self.params[name + ".weight"] = np.zeros((feat, item[1]), self.dtype)
                self.params[name + ".bias"] = np.zeros((item[1],), self.dtype)
                self.ops.append(("fc", name, None))
                shape = (item[1],)
            elif kind == "duel":
                feat = int(np.prod(shape))
                self.params["duel.value.weight"] = np.zeros((feat, 1), self.dtype)
                self.params["duel.value.bias"] = np.zeros((1,), self.dtype)
                self.params["duel.advantage.weight"] = np.zeros((feat, n_actions), self.dtype)
                self.params["duel.advantage.bias"] = np.zeros((n_actions,), self.dtype)
                self.ops.append(("duel", name, None))
                shape = (n_actions,)
        self.grads = {k: np.zeros_like(v) for k, v in self.params.items()}
        self._acts = []
        self._dq = None

    # -- init (network.py:180-205) ------------------------------------------
    def init(self, seed) -> None:
        rng = np.random.default_rng(seed)
        for name, arr in self.params.items():
            if not name.endswith(".weight"):
                continue
            if arr.ndim == 4:
                rf = arr.shape[0] * arr.shape[1]
                fi, fo = rf * arr.shape[2], rf * arr.shape[3]
            else:
                fi, fo = arr.shape
            lim = np.sqrt(6.0 / (fi + fo))
            arr[...] = rng.uniform(-lim, lim, size=arr.shape).astype(self.dtype)
        for name, arr in self.params.items():
            if name.endswith(".bias"):
                arr[...] = 0

    def copy_from(self, other: "QNet") -> None:
        """optim.py:78-89 bitwise copy."""
        for k in self.params:
            np.copyto(self.params[k], other.params[k])

    # -- forward ---------------------------------------------------------------
    @staticmethod
    def _patches(x, f, s):
        # windows (b, oh, ow, f, f, c) -> rows ordered (fh, fw, c) like the
        # (fh, fw, cin, cout) filter layout (layers.py:210-233)
        win = np.lib.stride_tricks.sliding_window_view(x, (f, f), axis=(1, 2))
        win = win[:, ::s, ::s]                       # (b, oh, ow, c, f, f)
        b, oh, ow = win.shape[:3]
        return np.ascontiguousarray(win.transpose(0, 1, 2, 4, 5, 3)).reshape(b * oh * ow, -1), oh, ow

    def forward(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=self.dtype)
        if x.shape[1:] != self.input_shape:
            raise OracleGeometryError("input shape")
        acts = []
        cur = x
        for kind, name, geo in self.ops:
            if kind == "conv":
                f, s = geo
                w = self.params[name + ".weight"]
                pt, oh, ow = self._patches(cur, f, s)
                y = pt @ w.reshape(-1, w.shape[-1])
                y += self.params[name + ".bias"]
                acts.append((cur, pt))
                cur = y.reshape(cur.shape[0], oh, ow, w.shape[-1])
            elif kind == "relu":
                acts.append((cur, None))
                cur = np.maximum(cur, 0)
            elif kind == "fc":
                flat = cur.reshape(cur.shape[0], -1)
                y = flat @ self.params[name + ".weight"]
                y += self.params[name + ".bias"]
                acts.append((cur, flat))
                cur = y
            else:  # duel, layers.py:302-310
                flat = cur.reshape(cur.shape[0], -1)
                v = flat @ self.params["duel.value.weight"]
                v += self.params["duel.value.bias"]
                a = flat @ self.params["duel.advantage.weight"]
                a += self.params["duel.advantage.bias"]
                q = np.empty_like(a)
                q[...] = v
                q += a
                q -= a.mean(axis=1, keepdims=True)
                acts.append((cur, flat))
                cur = q
        if not np.all(np.isfinite(cur)):
            raise OracleNonFiniteError("non-finite output")
        self._acts = acts
        return cur

    # -- backward + wgrad (layers.py:108-112,152-160,235-255,312-330) --------
    def backward(self, dq: np.ndarray) -> np.ndarray:
        dq = np.asarray(dq, dtype=self.dtype)
        self._dq = dq
        douts = [None] * len(self.ops)
        g = dq
        for li in range(len(self.ops) - 1, -1, -1):
            kind, name, geo = self.ops[li]
            xin, aux = self._acts[li]
            douts[li] = g
            if kind == "relu":
                g = g * (xin > 0)
            elif kind == "fc":
                g = (g @ self.params[name + ".weight"].T).reshape(xin.shape)
            elif kind == "duel":
                gv = g.sum(axis=1, keepdims=True)
                ga = g - gv / self.n_actions
                dx = gv @ self.params["duel.value.weight"].T
                dx += ga @ self.params["duel.advantage.weight"].T
                g = dx.reshape(xin.shape)
            else:  # conv: dpatches then scatter-add each filter tap
                f, s = geo
                w = self.params[name + ".weight"]
                cout = w.shape[-1]
                b, hh, ww, cin = xin.shape
                oh, ow = (hh - f) // s + 1, (ww - f) // s + 1
                dp = (g.reshape(-1, cout) @ w.reshape(-1, cout).T).reshape(b, oh, ow, f, f, cin)
                dx = np.zeros_like(xin)
                for ty in range(f):
                    for tx in range(f):
                        dx[:, ty:ty + s * oh:s, tx:tx + s * ow:s, :] += dp[:, :, :, ty, tx, :]
                g = dx
        self._douts = douts
        return g

    def wgrad(self) -> None:
        for li in range(len(self.ops) - 1, -1, -1):
            kind, name, geo = self.ops[li]
            xin, aux = self._acts[li]
            g = self._douts[li]
            if kind == "conv":
                cout = g.shape[-1]
                gf = g.reshape(-1, cout)
                self.grads[name + ".weight"] += (aux.T @ gf).reshape(self.grads[name + ".weight"].shape)
                self.grads[name + ".bias"] += gf.sum(axis=0)
            elif kind == "fc":
                self.grads[name + ".weight"] += aux.T @ g
                self.grads[name + ".bias"] += g.sum(axis=0)
            elif kind == "duel":
                gv = g.sum(axis=1, keepdims=True)
                ga = g - gv / self.n_actions
                self.grads["duel.value.weight"] += aux.T @ gv
                self.grads["duel.value.bias"] += gv.sum(axis=0)
                self.grads["duel.advantage.weight"] += aux.T @ ga
                self.grads["duel.advantage.bias"] += ga.sum(axis=0)

    def zero_grads(self):
        for g in self.grads.values():
            g[...] = 0


# ---------------------------------------------------------------------------
# optimizer (restates deepq/optim.py:12-89)
# ---------------------------------------------------------------------------


class RmsPropState:
    def __init__(self, net: QNet, lr=0.000625, decay=0.95, eps=1e-6):
        self.net, self.lr, self.decay, self.eps = net, float(lr), float(decay), float(eps)
        self.acc = {k: np.zeros_like(v) for k, v in net.params.items()}

    def step(self) -> None:
        """optim.py:36-47 -- finite scan of every grad first, then per tensor
        acc*=rho; acc+=(1-rho)*g^2; w-=lr*g/(sqrt(acc)+eps); g=0.  All float32
        with numpy weak-scalar promotion (the python floats become float32)."""
        net = self.net
        for k, g in net.grads.items():
            if not np.all(np.isfinite(g)):
                raise OracleNonFiniteError(f"non-finite gradient in {k}")
        for k, g in net.grads.items():
            a = self.acc[k]
            a *= self.decay
            a += (1.0 - self.decay) * np.square(g)
            net.params[k] -= self.lr * g / (np.sqrt(a) + self.eps)
            g[...] = 0


def clip_grads(net: QNet, max_norm: float) -> float:
    """optim.py:61-75 -- fp64 global norm, float32 scale."""
    tot = 0.0
    for g in net.grads.values():
        g64 = g.astype(np.float64).ravel()
        tot += float(np.dot(g64, g64))
    norm = float(np.sqrt(tot))
    if norm > max_norm and norm > 0.0:
        sc = np.asarray(max_norm / norm, dtype=net.dtype)
        for g in net.grads.values():
            g *= sc
    return norm


# ---------------------------------------------------------------------------
# learner step (restates deepq/agent.py:58-132)
# ---------------------------------------------------------------------------


@dataclass
class LearnCfg:
    gamma: float = 0.99
    batch_size: int = 32
    double: bool = True
    huber: bool = False
    reward_clip: bool = False
    grad_clip: float = 0.0


def td_targets(batch: Batch, online: QNet, target: QNet, gamma: float, double: bool):
    """agent.py:58-73."""
    if double:
        a_star = np.argmax(online.forward(batch.next_states), axis=1)
        qn = np.asarray(target.forward(batch.next_states), dtype=np.float64)
        boot = gamma * qn[np.arange(len(batch.actions)), a_star]
    else:
        qn = np.asarray(target.forward(batch.next_states), dtype=np.float64)
        boot = gamma * qn.max(axis=1)
    return batch.rewards + np.where(batch.terminals, 0.0, boot)


def learn_step(online: QNet, target: QNet, mem, opt: RmsPropState, cfg: LearnCfg,
               step: int, rng=None, uniforms=None, indices=None) -> dict:
    """agent.py:91-132.  ``uniforms`` (PER) or ``indices`` (uniform replay)
    may be supplied to teacher-force the draws; otherwise ``rng`` supplies
    them exactly as the reference does."""
    per = isinstance(mem, PerReplay)
    k = cfg.batch_size
    if per:
        batch = mem.sample(k, mem.beta(step), rng=rng, u=uniforms)
    else:
        ring = mem
        if indices is None:
            batch = uniform_sample(ring, k, rng)
        else:
            idx = np.asarray(indices, dtype=np.int64)
            batch = ring.gather(idx, np.full(k, 1.0 / ring.size), np.ones(k))
    out = learn_on_batch(online, target, batch, cfg)
    if cfg.grad_clip > 0.0:
        clip_grads(online, cfg.grad_clip)
    if per:
        mem.update_priorities(batch.indices, np.abs(out["td_errors"]))
    opt.step()
    return out


def learn_on_batch(online: QNet, target: QNet, batch: Batch, cfg: LearnCfg) -> dict:
    """agent.py:102-126 for a given batch: targets, TD errors, losses, output
    gradient, backward and gradient accumulation (no optimizer, no priority
    update).  Used directly by the sharded (data-parallel) restatement."""
    k = len(batch.actions)
    if cfg.reward_clip:
        batch.rewards = np.clip(batch.rewards, -1.0, 1.0)
    y = td_targets(batch, online, target, cfg.gamma, cfg.double)
    q = online.forward(batch.states)
    q_sa = q[np.arange(k), batch.actions].astype(np.float64)
    delta = y - q_sa
    w = batch.weights
    if cfg.huber:
        ad = np.abs(delta)
        losses = w * np.where(ad <= 1.0, 0.5 * delta * delta, ad - 0.5)
        dq = -w * np.clip(delta, -1.0, 1.0)
    else:
        losses = 0.5 * w * delta * delta
        dq = -w * delta
    out_grad = np.zeros((k, online.n_actions), dtype=online.dtype)
    out_grad[np.arange(k), batch.actions] = dq.astype(online.dtype)
    online.backward(out_grad)
    online.wgrad()
    grads = {kk: v.copy() for kk, v in online.grads.items()}
    return dict(batch=batch, targets=y, td_errors=delta, losses=losses, q=q,
                out_grad=out_grad, grads=grads)
