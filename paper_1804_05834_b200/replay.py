"""Device-resident replay: uint8 frame ring + fp64 sum tree in HBM.

Mirrors deepq/replay.py (Transition 20-29, SampleBatch 32-47, PriorityConfig
50-67, anneal_beta 70-71, ReplayMemory 74-124, SumTree 127-181,
PrioritizedReplay 184-241) with the same names, signatures and exceptions.
Differences a caller can see:

* arrays are torch CUDA tensors (``.cpu().numpy()`` gives the reference's
  numpy view); states are stored as uint8 frames (56 GB for 1M Atari
  transitions instead of the reference's 226 GB float32) and the
  network lifts them with the reference's pixel rule ``f32(u8)/255``;
  ``dtype=np.float32`` keeps raw float32 states for generic state shapes;
* the random draws (``rng.random`` / ``rng.integers``) are taken on the host
  from the caller's generator exactly as the reference takes them, so a
  seeded run samples the same indices.

HBM layout per ring: ``states``/``next_states`` [capacity][slot_bytes]
(28,224 B per Atari slot, 16-B aligned), actions i64, rewards f64, terminals
u8; tree ``nodes`` f64[2 * 2^depth] (1-indexed heap, replay.py:141-143);
``size`` and ``max_priority`` are device scalars so a captured CUDA graph
follows them.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .schedules import LinearSchedule


@dataclass
class Transition:
    state: object
    action: int
    reward: float
    next_state: object
    terminal: bool


@dataclass
class SampleBatch:
    states: object
    actions: object
    rewards: object
    next_states: object
    terminals: object
    indices: object
    probabilities: object
    weights: object

    def __len__(self) -> int:
        return len(self.actions)


@dataclass(frozen=True)
class PriorityConfig:
    """alpha, epsilon and the beta schedule (replay.py:50-67)."""

    alpha: float = 0.6
    epsilon: float = 0.01
    beta: LinearSchedule = field(default_factory=lambda: LinearSchedule(0.4, 1.0, 100_000_000))

    def __post_init__(self):
        if self.alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")
        if self.epsilon <= 0:
            raise ValueError(f"priority epsilon must be > 0, got {self.epsilon}")
        for b in (self.beta.start, self.beta.end):
            if not 0.0 <= b <= 1.0:
                raise ValueError(f"beta must stay within [0, 1], got {b}")


def anneal_beta(step: int, schedule: LinearSchedule) -> float:
    return schedule.value(step)


def _torch():
    return _lib.require_cuda()


def _to_device(x, dtype):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype)
    return torch.as_tensor(np.asarray(x), device="cuda").to(dtype)


def _frames(x, dtype):
    """States for the ring.  Float frames produced by the reference's
    preprocess_frame are f32(u8)/255 (envs.py:300-311); rounding x*255 maps
    them back to the exact byte, so a u8 ring reproduces them bit-for-bit."""
    torch = _torch()
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    if dtype == torch.uint8 and t.dtype.is_floating_point:
        t = torch.round(t.to(torch.float64) * 255.0).clamp_(0, 255)
    return t.to(device="cuda", dtype=dtype)


_TYPESTR = {"uint8": "|u1", "bool": "|b1", "int64": "<i8", "float64": "<f8", "float32": "<f4"}


class _SharedAlloc:
    """A plain cudaMalloc allocation (dqn_dev_alloc) so that its CUDA IPC
    handle covers exactly this buffer; viewed as a torch tensor through
    ``__cuda_array_interface__`` (zero copy; the tensor keeps it alive)."""

    def __init__(self, shape, dtype):
        import ctypes as C
        import weakref
        torch = _torch()
        self.dtype = dtype
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.ptr = C.c_void_p()
        _lib.call("dqn_dev_alloc", max(nbytes, 16), C.byref(self.ptr))
        self._fin = weakref.finalize(self, _lib.lib.dqn_dev_free, C.c_void_p(self.ptr.value))
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": _TYPESTR[str(dtype).split(".")[-1]],
            "data": (self.ptr.value, False), "version": 3, "strides": None}

    def handle(self) -> bytes:
        import ctypes as C
        buf = (C.c_uint8 * 64)()
        _lib.call("dqn_ipc_handle", self.ptr, buf)
        return bytes(buf)


def _shared_tensor(shape, dtype):
    torch = _torch()
    a = _SharedAlloc(shape, dtype)
    t = torch.as_tensor(a, device="cuda")
    t.zero_()
    return t, a


class ReplayMemory:
    """FIFO ring with uniform with-replacement sampling (replay.py:74-124).

    ``shareable=True`` allocates the five arrays as plain device allocations
    whose CUDA IPC handles other processes can map (the data-parallel
    learner's peer gather, dp.py)."""

    fused_ok = True           # slots the learner's fused sample + gather can read

    def __init__(self, capacity: int, state_shape: tuple[int, ...], dtype=np.uint8,
                 shareable: bool = False):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        torch = _torch()
        self.capacity = int(capacity)
        self.state_shape = tuple(int(s) for s in state_shape)
        self.np_dtype = np.dtype(dtype)
        if self.np_dtype == np.uint8:
            tdt = torch.uint8
        elif self.np_dtype == np.float32:
            tdt = torch.float32
        else:
            raise ValueError(f"ring dtype must be uint8 or float32, got {self.np_dtype}")
        shapes = {"states": ((self.capacity,) + self.state_shape, tdt),
                  "next_states": ((self.capacity,) + self.state_shape, tdt),
                  "actions": ((self.capacity,), torch.int64),
                  "rewards": ((self.capacity,), torch.float64),
                  "terminals": ((self.capacity,), torch.bool)}
        self.shared = {}
        for name, (shp, dt) in shapes.items():
            if shareable:
                t, self.shared[name] = _shared_tensor(shp, dt)
            else:
                t = torch.zeros(shp, dtype=dt, device="cuda")
            setattr(self, name, t)
        self.slot_bytes = int(self.states[0].numel() * self.states.element_size())
        self.cursor = 0
        self.size = 0
        self._size_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self._scratch = {}

    @property
    def state_dtype(self):
        return self.states.dtype

    # -- insertion ------------------------------------------------------
    def _set_size(self, n: int) -> None:
        self.size = n
        self._size_dev.fill_(n)

    def store(self, transition: Transition) -> int:
        """Insert at the cursor, evicting the oldest (replay.py:91-102)."""
        i = self.cursor
        self.states[i] = _frames(transition.state, self.states.dtype).reshape(self.state_shape)
        self.next_states[i] = _frames(transition.next_state, self.states.dtype).reshape(self.state_shape)
        self.actions[i] = int(transition.action)
        self.rewards[i] = float(transition.reward)
        self.terminals[i] = bool(transition.terminal)
        self.cursor = (i + 1) % self.capacity
        self._set_size(min(self.size + 1, self.capacity))
        return i

    def store_many(self, states, actions, rewards, next_states, terminals) -> np.ndarray:
        """Batched ``store`` (same ring semantics, one copy per field)."""
        torch = _torch()
        n = len(actions)
        slots = (self.cursor + np.arange(n)) % self.capacity
        # a batch longer than the ring keeps its last `capacity` transitions
        # (scatters with repeated slots would leave an unspecified winner)
        m = min(n, self.capacity)
        sl = torch.as_tensor(slots[n - m:], device="cuda")
        tail = slice(n - m, n)
        self.states[sl] = _frames(states, self.states.dtype).reshape((n,) + self.state_shape)[tail]
        self.next_states[sl] = _frames(next_states, self.states.dtype).reshape(
            (n,) + self.state_shape)[tail]
        self.actions[sl] = _to_device(actions, torch.int64)[tail]
        self.rewards[sl] = _to_device(rewards, torch.float64)[tail]
        self.terminals[sl] = _to_device(terminals, torch.bool)[tail]
        self.cursor = int((self.cursor + n) % self.capacity)
        self._set_size(min(self.size + n, self.capacity))
        return slots

    def store_staged(self, states, next_states, actions, rewards, terminals, n: int) -> None:
        """Insert n staged transitions in one launch (dqn_ring_store): tensors
        in the ring's state dtype / int64 / float64 / uint8, pinned host
        memory (read in place by the kernel) or device memory; same ring
        semantics as ``store`` called n times."""
        if n <= 0:
            return
        if n > self.capacity:
            raise ValueError("more staged transitions than slots")
        new_size = min(self.size + n, self.capacity)
        _lib.call("dqn_ring_store", _lib.stream_ptr(), self.states.data_ptr(),
                  self.next_states.data_ptr(), self.slot_bytes, self.actions.data_ptr(),
                  self.rewards.data_ptr(), self.terminals.data_ptr(), self.capacity, self.cursor,
                  int(n), states.data_ptr(), next_states.data_ptr(), actions.data_ptr(),
                  rewards.data_ptr(), terminals.data_ptr(), self._size_dev.data_ptr(), new_size)
        self.cursor = (self.cursor + n) % self.capacity
        self.size = new_size

    def fill_synthetic(self, seed: int, n: int | None = None, n_actions: int = 4) -> None:
        """Bench/test input: hash frames generated in HBM (synth.py), host
        metadata streams.  Fills slots [0, n) and sets size = cursor = n."""
        from . import synth
        torch = _torch()
        n = self.capacity if n is None else int(n)
        if self.states.dtype != torch.uint8:
            raise ValueError("fill_synthetic needs a uint8 ring")
        st = _lib.stream_ptr()
        chunk = 1 << 16
        for kind, buf in ((0, self.states), (1, self.next_states)):
            base = synth.frame_counter_base(seed, kind)
            for s0 in range(0, n, chunk):
                _lib.call("dqn_ring_fill_hash", st, buf.data_ptr(), s0, min(chunk, n - s0),
                          self.slot_bytes, base)
        a, r, t = synth.metadata(seed, n, n_actions)
        self.actions[:n] = torch.as_tensor(a, device="cuda")
        self.rewards[:n] = torch.as_tensor(r, device="cuda")
        self.terminals[:n] = torch.as_tensor(t, device="cuda")
        self.cursor = n % self.capacity
        self._set_size(n)

    # -- sampling -------------------------------------------------------
    def _buf(self, name, shape, dtype):
        torch = _torch()
        t = self._scratch.get(name)
        if t is None or t.shape != shape or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device="cuda")
            self._scratch[name] = t
        return t

    def gather_into(self, indices, k: int, out_states, out_next_states, out_actions,
                    out_rewards, out_terminals) -> None:
        """ReplayMemory._gather into caller buffers (dqn_ring_gather)."""
        _lib.call("dqn_ring_gather", _lib.stream_ptr(), self.states.data_ptr(),
                  self.next_states.data_ptr(), self.slot_bytes, self.actions.data_ptr(),
                  self.rewards.data_ptr(), self.terminals.data_ptr(), indices.data_ptr(), k,
                  _lib.ptr(out_states), _lib.ptr(out_next_states), _lib.ptr(out_actions),
                  _lib.ptr(out_rewards), _lib.ptr(out_terminals))

    def _gather(self, indices, probabilities, weights) -> SampleBatch:
        """replay.py:104-115 -- fresh output tensors (the reference returns
        fancy-indexed copies)."""
        torch = _torch()
        idx = _to_device(indices, torch.int64).contiguous()
        k = idx.numel()
        s = torch.empty((k,) + self.state_shape, dtype=self.states.dtype, device="cuda")
        s2 = torch.empty_like(s)
        a = torch.empty(k, dtype=torch.int64, device="cuda")
        r = torch.empty(k, dtype=torch.float64, device="cuda")
        t = torch.empty(k, dtype=torch.bool, device="cuda")
        self.gather_into(idx, k, s, s2, a, r, t)
        return SampleBatch(s, a, r, s2, t, idx, probabilities, weights)

    def sample_uniform(self, k: int, rng: np.random.Generator) -> SampleBatch:
        """replay.py:117-124: host draws ``rng.integers(0, size, k)``."""
        torch = _torch()
        if self.size == 0:
            raise ValueError("cannot sample from an empty replay memory")
        indices = rng.integers(0, self.size, size=k)
        prob = torch.full((k,), 1.0 / self.size, dtype=torch.float64, device="cuda")
        w = torch.ones(k, dtype=torch.float64, device="cuda")
        return self._gather(indices, prob, w)


class SumTree:
    """fp64 heap in HBM (replay.py:127-181)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        torch = _torch()
        self.capacity = int(capacity)
        self.depth = max(1, int(np.ceil(np.log2(capacity))))
        self._leaf_base = 1 << self.depth
        self.nodes = torch.zeros(2 * self._leaf_base, dtype=torch.float64, device="cuda")
        self._flags = torch.zeros(1, dtype=torch.int32, device="cuda")

    def _check_flags(self) -> None:
        f = int(self._flags.item())
        if f:
            self._flags.zero_()
            if f & _lib.FLAG_ZERO_TOTAL:
                raise ValueError("cannot query a sum tree with zero total priority")
            if f & _lib.FLAG_INDEX:
                raise IndexError("leaf index out of range")
            if f & _lib.FLAG_BAD_PRIORITY:
                raise ValueError("priority must be finite and >= 0")

    @property
    def total(self) -> float:
        return float(self.nodes[1].item())

    def leaf(self, i: int) -> float:
        return float(self.nodes[self._leaf_base + i].item())

    def leaves(self):
        return self.nodes[self._leaf_base:self._leaf_base + self.capacity]

    def set(self, i: int, value: float) -> None:
        """replay.py:155-165 (one leaf, ancestors recomputed)."""
        if not 0 <= i < self.capacity:
            raise IndexError(f"leaf index {i} out of range [0, {self.capacity})")
        if value < 0 or not np.isfinite(value):
            raise ValueError(f"priority must be finite and >= 0, got {value}")
        self.set_many(np.array([i]), np.array([float(value)]))

    def set_many(self, indices, values) -> None:
        torch = _torch()
        idx = _to_device(indices, torch.int64).contiguous()
        val = _to_device(values, torch.float64).contiguous()
        _lib.call("dqn_tree_set", _lib.stream_ptr(), self.nodes.data_ptr(), self.depth,
                  self.capacity, idx.data_ptr(), val.data_ptr(), idx.numel(),
                  self._flags.data_ptr())
        self._check_flags()

    def load_leaves(self, leaves) -> None:
        """Bulk: overwrite all leaves, then rebuild bottom-up.  Bit-identical to
        any sequence of set() calls ending in the same leaves."""
        torch = _torch()
        v = _to_device(leaves, torch.float64).reshape(-1)
        self.nodes[self._leaf_base:self._leaf_base + v.numel()] = v
        _lib.call("dqn_tree_rebuild", _lib.stream_ptr(), self.nodes.data_ptr(), self.depth)

    def find(self, values):
        """replay.py:167-181 -> leaf indices (device int64)."""
        torch = _torch()
        q = _to_device(values, torch.float64).reshape(-1).contiguous()
        out = torch.empty(q.numel(), dtype=torch.int64, device="cuda")
        _lib.call("dqn_tree_find", _lib.stream_ptr(), self.nodes.data_ptr(), self.depth,
                  q.data_ptr(), q.numel(), out.data_ptr(), self._flags.data_ptr())
        self._check_flags()
        return out


class PrioritizedReplay:
    """Ring + sum tree over p^alpha (replay.py:184-241)."""

    def __init__(self, capacity: int, state_shape: tuple[int, ...],
                 config: PriorityConfig | None = None, dtype=np.uint8, shareable: bool = False,
                 frame_dedup: bool = False, frame_capacity: int | None = None):
        """``frame_dedup=True`` keeps each frame once (frame_ring.py; uint8,
        same sampled bytes, ~1/8 of the footprint for episodic streams)."""
        torch = _torch()
        if frame_dedup:
            from .frame_ring import FrameDedupMemory
            if shareable:
                raise ValueError("the frame-deduplicated ring is not shareable")
            self.memory = FrameDedupMemory(capacity, state_shape, dtype=dtype,
                                           frame_capacity=frame_capacity)
        else:
            self.memory = ReplayMemory(capacity, state_shape, dtype=dtype, shareable=shareable)
        self.config = config or PriorityConfig()
        self.tree = SumTree(capacity)
        self._max_p = torch.ones(1, dtype=torch.float64, device="cuda")   # raw p-space
        self._scratch = {}

    @property
    def max_priority(self) -> float:
        return float(self._max_p.item())

    @max_priority.setter
    def max_priority(self, v: float) -> None:
        self._max_p.fill_(float(v))

    @property
    def size(self) -> int:
        return self.memory.size

    @property
    def capacity(self) -> int:
        return self.memory.capacity

    def store(self, transition: Transition) -> int:
        index = self.memory.store(transition)
        _lib.call("dqn_tree_store", _lib.stream_ptr(), self.tree.nodes.data_ptr(),
                  self.tree.depth, self.capacity, index, 1, self._max_p.data_ptr(),
                  float(self.config.alpha))
        return index

    def store_many(self, states, actions, rewards, next_states, terminals) -> np.ndarray:
        slot0 = self.memory.cursor
        slots = self.memory.store_many(states, actions, rewards, next_states, terminals)
        _lib.call("dqn_tree_store", _lib.stream_ptr(), self.tree.nodes.data_ptr(),
                  self.tree.depth, self.capacity, slot0, len(slots), self._max_p.data_ptr(),
                  float(self.config.alpha))
        return slots

    def store_staged(self, states, next_states, actions, rewards, terminals, n: int) -> None:
        """``ReplayMemory.store_staged`` + the new leaves at max priority."""
        if n <= 0:
            return
        slot0 = self.memory.cursor
        self.memory.store_staged(states, next_states, actions, rewards, terminals, n)
        _lib.call("dqn_tree_store", _lib.stream_ptr(), self.tree.nodes.data_ptr(),
                  self.tree.depth, self.capacity, slot0, int(n), self._max_p.data_ptr(),
                  float(self.config.alpha))

    def fill_synthetic(self, seed: int, n: int | None = None, n_actions: int = 4,
                       warmup: bool = True) -> None:
        """Synthetic ring (see ReplayMemory.fill_synthetic) inserted at
        max priority, then one warm-up ``update_priorities(arange(n),
        |N(0,1)|)`` so the tree is non-uniform."""
        from . import synth
        torch = _torch()
        n = self.capacity if n is None else int(n)
        self.memory.fill_synthetic(seed, n, n_actions)
        leaf = float(self.max_priority) ** self.config.alpha
        self.tree.nodes[self.tree._leaf_base:self.tree._leaf_base + n] = leaf
        _lib.call("dqn_tree_rebuild", _lib.stream_ptr(), self.tree.nodes.data_ptr(), self.tree.depth)
        if warmup:
            td = synth.warmup_td(seed, n)
            idx = torch.arange(n, dtype=torch.int64, device="cuda")
            self.update_priorities(idx, torch.as_tensor(td, device="cuda"))

    def beta(self, step: int) -> float:
        return anneal_beta(step, self.config.beta)

    def _buf(self, name, n, dtype):
        torch = _torch()
        t = self._scratch.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(max(n, 1), dtype=dtype, device="cuda")
            self._scratch[name] = t
        return t[:n]

    def sample_indices(self, u_dev, k: int, beta_dev, idx, prob, w, flags) -> None:
        """Device part of ``sample``: stratified descent + IS weights."""
        _lib.call("dqn_tree_sample", _lib.stream_ptr(), self.tree.nodes.data_ptr(), self.tree.depth,
                  self.memory._size_dev.data_ptr(), u_dev.data_ptr(), k, beta_dev.data_ptr(),
                  idx.data_ptr(), prob.data_ptr(), w.data_ptr(), flags.data_ptr())

    def sample(self, k: int, beta: float, rng: np.random.Generator) -> SampleBatch:
        """replay.py:215-230.  ``offsets = rng.random(k)`` on the host."""
        torch = _torch()
        if self.size == 0:
            raise ValueError("cannot sample from an empty replay memory")
        u = torch.as_tensor(rng.random(k), device="cuda")
        beta_dev = torch.full((1,), float(beta), dtype=torch.float64, device="cuda")
        idx = torch.empty(k, dtype=torch.int64, device="cuda")
        prob = torch.empty(k, dtype=torch.float64, device="cuda")
        w = torch.empty(k, dtype=torch.float64, device="cuda")
        self.sample_indices(u, k, beta_dev, idx, prob, w, self.tree._flags)
        self.tree._check_flags()
        return self.memory._gather(idx, prob, w)

    def update_priorities_dev(self, idx, td_abs, k: int, flags) -> None:
        """Device part of ``update_priorities`` (no host sync)."""
        _lib.call("dqn_tree_update", _lib.stream_ptr(), self.tree.nodes.data_ptr(), self.tree.depth,
                  self.memory._size_dev.data_ptr(), idx.data_ptr(), td_abs.data_ptr(), k,
                  float(self.config.alpha), float(self.config.epsilon), self._max_p.data_ptr(),
                  flags.data_ptr())

    def update_priorities(self, indices, td_errors) -> None:
        """replay.py:232-241: leaf = (|td| + eps)^alpha in batch order, last
        write wins; IndexError at the first out-of-range index (earlier
        leaves stay written, as in the reference)."""
        torch = _torch()
        idx = _to_device(indices, torch.int64).reshape(-1).contiguous()
        td = _to_device(td_errors, torch.float64).reshape(-1).contiguous()
        if idx.numel() != td.numel():
            raise ValueError("indices and td_errors differ in length")
        self.update_priorities_dev(idx, td, idx.numel(), self.tree._flags)
        f = int(self.tree._flags.item())
        if f:
            self.tree._flags.zero_()
            if f & _lib.FLAG_INDEX:
                raise IndexError(f"transition index out of range [0, {self.size})")
            raise ValueError("priority must be finite and >= 0")
