"""Frame-deduplicated replay ring.

The reference's ``ReplayMemory`` stores every transition's full state and
next-state stacks (replay.py:83-84; SPEC.md:294 keeps it that way on
purpose): at Atari shapes 2 x 28,224 B per slot, 56 GB per million.
Consecutive transitions of an episode share all but one frame: s_{t+1} is
s_t shifted by one frame, and the next state of transition t is the state of
transition t+1.  ``FrameDedupMemory`` keeps each H x W frame plane once in a
device frame pool and, per ring slot, the 2S pool ids of its stack planes.
For an episodic stream that is about one new 7,056 B frame per transition
instead of 56,448 B: ~7 GB per million.

Sampling semantics are the reference's: ``gather_into`` / ``sample_uniform``
return the same bytes a full-stack ring holding the same transitions returns
(dqn_frame_gather rebuilds the channel-last stacks on the device).  Storage
differs only in footprint.

Host bookkeeping (``FrameIndex``, plain numpy):
* A new transition's planes are matched by content against the previous
  transition's planes and its own earlier planes.  A match reuses the pool
  id; otherwise a free id is taken and the plane uploaded.
* Reference counts per pool slot.  When the ring overwrites a slot, its 2S
  ids are released after the new transition is assigned (an id still
  referenced is never handed out).  A free list supplies new ids.
* The pool is sized ``frame_capacity`` (default 2 x capacity + 4S).
  Exhausting it raises ``ConfigError`` rather than overwriting live frames.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from . import _lib
from .errors import ConfigError, GeometryError
from .replay import ReplayMemory, SampleBatch, Transition, _torch


class FrameIndex:
    """Pool-id assignment, reference counts and the per-slot id table."""

    def __init__(self, capacity: int, frame_capacity: int, stack: int):
        if frame_capacity < 2 * stack:
            raise ConfigError(f"frame_capacity must be >= {2 * stack}, got {frame_capacity}")
        self.capacity, self.frame_capacity, self.stack = int(capacity), int(frame_capacity), int(stack)
        self.ids = np.full((self.capacity, 2 * self.stack), -1, dtype=np.int64)
        self.refs = np.zeros(self.frame_capacity, dtype=np.int64)
        self.free = deque(range(self.frame_capacity))
        self._prev: dict[bytes, int] = {}      # previous transition's planes -> pool id

    @property
    def live_frames(self) -> int:
        return self.frame_capacity - len(self.free)

    def assign(self, slot: int, planes: list[bytes]) -> list[tuple[int, bytes]]:
        """Assign pool ids to the 2S planes (state then next state) of the
        transition stored at ``slot``; returns the (id, plane) pairs that
        must be uploaded (planes not already in the pool)."""
        if len(planes) != 2 * self.stack:
            raise GeometryError(f"expected {2 * self.stack} planes, got {len(planes)}")
        seen = dict(self._prev)
        row = np.empty(2 * self.stack, dtype=np.int64)
        uploads = []
        for j, p in enumerate(planes):
            fid = seen.get(p)
            if fid is None:
                if not self.free:
                    # undo this transition's references before failing
                    for f in row[:j]:
                        self._release(int(f))
                    raise ConfigError(f"frame pool exhausted ({self.frame_capacity} frames); "
                                      "raise frame_capacity (the stream shares fewer frames "
                                      "between transitions than assumed)")
                fid = self.free.popleft()
                uploads.append((fid, p))
                seen[p] = fid
            self.refs[fid] += 1
            row[j] = fid
        old = self.ids[slot].copy()
        self.ids[slot] = row
        for f in old:
            if f >= 0:
                self._release(int(f))
        self._prev = {p: int(f) for p, f in zip(planes, row)}
        return uploads

    def _release(self, fid: int) -> None:
        self.refs[fid] -= 1
        if self.refs[fid] == 0:
            self.free.append(fid)


def _planes(x, stack: int) -> list[bytes]:
    """The S channel planes of one (H, W, S) stack as bytes; float frames
    (f32(u8)/255, envs.py:300-311) map back to their exact byte."""
    a = x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    if a.dtype != np.uint8:
        a = np.clip(np.round(a.astype(np.float64) * 255.0), 0, 255).astype(np.uint8)
    if a.shape[-1] != stack:
        raise GeometryError(f"state shape {a.shape} does not end in the stack depth {stack}")
    return [np.ascontiguousarray(a[..., s]).tobytes() for s in range(stack)]


class FrameDedupMemory(ReplayMemory):
    """``ReplayMemory`` with a frame-deduplicated store (uint8 states only).

    Same API for callers of the learner path: ``store``, ``gather_into``,
    ``sample_uniform``, ``size`` / ``cursor`` / ``capacity``, the
    ``actions`` / ``rewards`` / ``terminals`` device arrays.  There are no
    ``states`` / ``next_states`` arrays (``stack_at`` rebuilds one slot), and
    the batched staging paths of the full-stack ring are not provided."""

    fused_ok = False          # the learner gathers through dqn_frame_gather

    def __init__(self, capacity: int, state_shape: tuple[int, ...], dtype=np.uint8,
                 frame_capacity: int | None = None):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        if np.dtype(dtype) != np.uint8:
            raise ValueError("the frame-deduplicated ring stores uint8 frames")
        if len(state_shape) != 3:
            raise GeometryError(f"state shape must be (H, W, stack), got {state_shape}")
        torch = _torch()
        self.capacity = int(capacity)
        self.state_shape = tuple(int(s) for s in state_shape)
        self.np_dtype = np.dtype(np.uint8)
        h, w, s = self.state_shape
        self.stack = s
        self.frame_bytes = h * w
        fcap = int(frame_capacity) if frame_capacity is not None else 2 * self.capacity + 4 * s
        self.index = FrameIndex(self.capacity, fcap, s)
        self.frames = torch.zeros((fcap, self.frame_bytes), dtype=torch.uint8, device="cuda")
        self.ids = torch.zeros((self.capacity, 2 * s), dtype=torch.int64, device="cuda")
        self.actions = torch.zeros(self.capacity, dtype=torch.int64, device="cuda")
        self.rewards = torch.zeros(self.capacity, dtype=torch.float64, device="cuda")
        self.terminals = torch.zeros(self.capacity, dtype=torch.bool, device="cuda")
        self.shared = {}
        self.slot_bytes = self.frame_bytes * s
        self.cursor = 0
        self.size = 0
        self._size_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self._scratch = {}

    @property
    def state_dtype(self):
        return self.frames.dtype

    @property
    def resident_bytes(self) -> int:
        """Device bytes of frames and ids actually referenced (pool slots
        in use x frame size + the id table + metadata)."""
        return (self.index.live_frames * self.frame_bytes + self.ids.numel() * 8
                + self.capacity * (8 + 8 + 1))

    def store(self, transition: Transition) -> int:
        """Insert at the cursor, evicting the oldest (replay.py:91-102)."""
        torch = _torch()
        i = self.cursor
        planes = _planes(transition.state, self.stack) + _planes(transition.next_state, self.stack)
        for p in planes:
            if len(p) != self.frame_bytes:
                raise GeometryError(f"frame of {len(p)} B, ring holds {self.frame_bytes} B frames")
        for fid, p in self.index.assign(i, planes):
            self.frames[fid] = torch.frombuffer(bytearray(p), dtype=torch.uint8)
        self.ids[i] = torch.as_tensor(self.index.ids[i])
        self.actions[i] = int(transition.action)
        self.rewards[i] = float(transition.reward)
        self.terminals[i] = bool(transition.terminal)
        self.cursor = (i + 1) % self.capacity
        self._set_size(min(self.size + 1, self.capacity))
        return i

    def store_many(self, states, actions, rewards, next_states, terminals) -> np.ndarray:
        """Batched ``store``: ids assigned on the host in order, then the new
        planes in one pinned upload and one scatter per array."""
        torch = _torch()
        n = len(actions)
        if n == 0:
            return np.zeros(0, dtype=np.int64)
        slots = (self.cursor + np.arange(n)) % self.capacity
        new_ids, new_planes = [], []
        for j in range(n):
            planes = _planes(states[j], self.stack) + _planes(next_states[j], self.stack)
            for p in planes:
                if len(p) != self.frame_bytes:
                    raise GeometryError(f"frame of {len(p)} B, ring holds {self.frame_bytes} B frames")
            for fid, p in self.index.assign(int(slots[j]), planes):
                new_ids.append(fid)
                new_planes.append(p)
        # a pool id can be reassigned within the batch only after its last
        # reference went away: the last upload of an id is the one that counts
        if new_ids:
            buf = torch.empty((len(new_ids), self.frame_bytes), dtype=torch.uint8).pin_memory()
            buf.numpy()[:] = np.frombuffer(b"".join(new_planes), dtype=np.uint8).reshape(
                len(new_ids), self.frame_bytes)
            last = {fid: i for i, fid in enumerate(new_ids)}
            keep = torch.as_tensor(sorted(last.values()), dtype=torch.int64)
            ids_t = torch.as_tensor([new_ids[i] for i in keep.tolist()], dtype=torch.int64)
            self.frames.index_copy_(0, ids_t.to("cuda"), buf[keep].to("cuda", non_blocking=True))
        # a batch longer than the ring keeps its last `capacity` transitions
        # (scatters with repeated slots would leave an unspecified winner)
        m = min(n, self.capacity)
        sl = torch.as_tensor(slots[n - m:], device="cuda")
        self.ids.index_copy_(0, sl, torch.as_tensor(self.index.ids[slots[n - m:]]).to("cuda"))
        self.actions[sl] = torch.as_tensor(np.asarray(actions)[n - m:], dtype=torch.int64).to("cuda")
        self.rewards[sl] = torch.as_tensor(np.asarray(rewards)[n - m:], dtype=torch.float64).to("cuda")
        self.terminals[sl] = torch.as_tensor(np.asarray(terminals)[n - m:], dtype=torch.bool).to("cuda")
        self.cursor = int((self.cursor + n) % self.capacity)
        self._set_size(min(self.size + n, self.capacity))
        return slots

    def store_staged(self, *args, **kwargs) -> None:
        raise NotImplementedError("the frame-deduplicated ring stores through store()")

    def gather_into(self, indices, k: int, out_states, out_next_states, out_actions,
                    out_rewards, out_terminals) -> None:
        """ReplayMemory._gather into caller buffers (dqn_frame_gather)."""
        _lib.call("dqn_frame_gather", _lib.stream_ptr(), self.frames.data_ptr(),
                  self.frame_bytes, self.ids.data_ptr(), self.stack, indices.data_ptr(), k,
                  self.actions.data_ptr(), self.rewards.data_ptr(), self.terminals.data_ptr(),
                  _lib.ptr(out_states), _lib.ptr(out_next_states), _lib.ptr(out_actions),
                  _lib.ptr(out_rewards), _lib.ptr(out_terminals))

    def _gather(self, indices, probabilities, weights) -> SampleBatch:
        torch = _torch()
        from .replay import _to_device
        idx = _to_device(indices, torch.int64).contiguous()
        k = idx.numel()
        s = torch.empty((k,) + self.state_shape, dtype=torch.uint8, device="cuda")
        s2 = torch.empty_like(s)
        a = torch.empty(k, dtype=torch.int64, device="cuda")
        r = torch.empty(k, dtype=torch.float64, device="cuda")
        t = torch.empty(k, dtype=torch.bool, device="cuda")
        self.gather_into(idx, k, s, s2, a, r, t)
        return SampleBatch(s, a, r, s2, t, idx, probabilities, weights)

    def stack_at(self, slot: int):
        """(state, next_state) of one slot as device uint8 stacks."""
        torch = _torch()
        b = self._gather(torch.tensor([int(slot)], device="cuda"), None, None)
        return b.states[0], b.next_states[0]
