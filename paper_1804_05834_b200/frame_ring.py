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
from .replay import ReplayMemory, SampleBatch, Transition, _to_device, _torch


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
    ``actions`` / ``rewards`` / ``terminals`` device arrays, the Trainer's
    staged insert (``store_staged``) and checkpoint export / import
    (``host_states`` / ``restore``).  There are no ``states`` /
    ``next_states`` arrays (``stack_at`` rebuilds one slot)."""

    fused_ok = True           # the learner samples + gathers by dqn_frame_sample_gather

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
        # persistent pinned staging for batched plane uploads, reused once the
        # event recorded after its last copy has completed
        self._stage = torch.empty((0, self.frame_bytes), dtype=torch.uint8).pin_memory()
        self._stage_ev = None
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
        """Batched ``store``: ids assigned on the host in batch order, then
        the new planes in one pinned upload and one scatter per array.

        Every transition's planes are built and checked before the first
        assignment (a malformed state raises with nothing changed).  If the
        pool runs out part-way (ConfigError), the transitions assigned so
        far are uploaded and the cursor advances past them before the error
        propagates, so the device table never points at ids the host index
        no longer holds."""
        torch = _torch()
        n = len(actions)
        if n == 0:
            return np.zeros(0, dtype=np.int64)
        planes_all = []
        for j in range(n):
            planes = _planes(states[j], self.stack) + _planes(next_states[j], self.stack)
            for p in planes:
                if len(p) != self.frame_bytes:
                    raise GeometryError(f"frame of {len(p)} B, ring holds {self.frame_bytes} B frames")
            planes_all.append(planes)
        slots = (self.cursor + np.arange(n)) % self.capacity
        new_ids, new_planes = [], []
        done, err = n, None
        for j in range(n):
            try:
                ups = self.index.assign(int(slots[j]), planes_all[j])
            except ConfigError as e:           # pool exhausted: keep transitions 0..j-1
                done, err = j, e
                break
            for fid, p in ups:
                new_ids.append(fid)
                new_planes.append(p)
        if done:
            self._commit(slots[:done], new_ids, new_planes,
                         _to_device(actions, torch.int64)[:done],
                         _to_device(rewards, torch.float64)[:done],
                         _to_device(terminals, torch.bool)[:done])
        if err is not None:
            raise err
        return slots

    def _commit(self, slots, new_ids, new_planes, actions, rewards, terminals) -> None:
        """Upload the planes assigned to ``slots`` (host index already
        updated), write the slots' id rows and metadata, advance the cursor."""
        torch = _torch()
        n = len(slots)
        # a pool id can be reassigned within the batch only after its last
        # reference went away: the last upload of an id is the one that counts
        if new_ids:
            last = {fid: i for i, fid in enumerate(new_ids)}
            keep = sorted(last.values())
            if self._stage_ev is not None:
                self._stage_ev.synchronize()          # the last upload has read the stage
            if self._stage.shape[0] < len(keep):
                self._stage = torch.empty((max(len(keep), 2 * self._stage.shape[0]), self.frame_bytes),
                                          dtype=torch.uint8).pin_memory()
            buf = self._stage[:len(keep)]
            buf.numpy()[:] = np.frombuffer(b"".join(new_planes[i] for i in keep),
                                           dtype=np.uint8).reshape(len(keep), self.frame_bytes)
            ids_t = torch.as_tensor([new_ids[i] for i in keep], dtype=torch.int64, device="cuda")
            self.frames.index_copy_(0, ids_t, buf.to("cuda", non_blocking=True))
            self._stage_ev = torch.cuda.Event()
            self._stage_ev.record()
        # a batch longer than the ring keeps its last `capacity` transitions
        # (scatters with repeated slots would leave an unspecified winner)
        m = min(n, self.capacity)
        sl_np = np.asarray(slots[n - m:])
        sl = torch.as_tensor(sl_np, device="cuda")
        self.ids.index_copy_(0, sl, torch.as_tensor(self.index.ids[sl_np]).to("cuda"))
        self.actions[sl] = actions[n - m:]
        self.rewards[sl] = rewards[n - m:]
        self.terminals[sl] = terminals[n - m:]
        self.cursor = int((self.cursor + n) % self.capacity)
        self._set_size(min(self.size + n, self.capacity))

    def store_staged(self, states, next_states, actions, rewards, terminals, n: int) -> None:
        """The Trainer's staged insert (trainer._Staging): ``n`` transitions
        from pinned host buffers, through the batched host index."""
        n = int(n)
        if n <= 0:
            return
        self.store_many(states[:n].numpy(), actions[:n], rewards[:n], next_states[:n].numpy(),
                        terminals[:n])

    def fill_synthetic(self, *args, **kwargs) -> None:
        raise NotImplementedError("the frame-deduplicated ring is filled through store / "
                                  "store_many (synthetic fills are per slot, not per frame)")

    # -- checkpoint export / import (checkpoint.py:134-177 'memory') ------
    def host_states(self, n: int):
        """(states, next_states) of slots [0, n) as host uint8 arrays -- the
        full stacks, as the full-stack ring's checkpoint holds them."""
        torch = _torch()
        out_s = np.empty((n,) + self.state_shape, dtype=np.uint8)
        out_n = np.empty_like(out_s)
        for a in range(0, n, 4096):
            b = min(n, a + 4096)
            bt = self._gather(torch.arange(a, b, device="cuda"), None, None)
            out_s[a:b] = bt.states.cpu().numpy()
            out_n[a:b] = bt.next_states.cpu().numpy()
        return out_s, out_n

    def restore(self, n: int, states, next_states, actions, rewards, terminals, cursor: int) -> None:
        """Refill slots [0, n) from host arrays (a checkpoint's memory
        section), then set the cursor: the same ring contents as the
        checkpointed one (frames re-deduplicated in slot order)."""
        h, w, s = self.state_shape
        self.index = FrameIndex(self.capacity, self.index.frame_capacity, s)
        self.cursor = 0
        self._set_size(0)
        if n:
            self.store_many(states, actions, rewards, next_states, terminals)
        self.cursor = int(cursor)

    def gather_into(self, indices, k: int, out_states, out_next_states, out_actions,
                    out_rewards, out_terminals) -> None:
        """ReplayMemory._gather into caller buffers (dqn_frame_gather)."""
        _lib.call("dqn_frame_gather", _lib.stream_ptr(), self.frames.data_ptr(),
                  self.frame_bytes, self.ids.data_ptr(), self.stack, indices.data_ptr(), k,
                  self.actions.data_ptr(), self.rewards.data_ptr(), self.terminals.data_ptr(),
                  _lib.ptr(out_states), _lib.ptr(out_next_states), _lib.ptr(out_actions),
                  _lib.ptr(out_rewards), _lib.ptr(out_terminals))

    def sample_gather_fused(self, tree, u, k: int, beta, idx, prob, w, flags, out_states,
                            out_next_states, out_actions, out_rewards, out_terminals) -> None:
        """PrioritizedReplay.sample + _gather in one launch (the learner's
        fused path; dqn_frame_sample_gather)."""
        _lib.call("dqn_frame_sample_gather", _lib.stream_ptr(), tree.nodes.data_ptr(), tree.depth,
                  self._size_dev.data_ptr(), _lib.ptr(u), k, _lib.ptr(beta), _lib.ptr(idx),
                  _lib.ptr(prob), _lib.ptr(w), _lib.ptr(flags), self.frames.data_ptr(),
                  self.frame_bytes, self.ids.data_ptr(), self.stack, self.actions.data_ptr(),
                  self.rewards.data_ptr(), self.terminals.data_ptr(), _lib.ptr(out_states),
                  _lib.ptr(out_next_states), _lib.ptr(out_actions), _lib.ptr(out_rewards),
                  _lib.ptr(out_terminals))

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
