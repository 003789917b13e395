"""Data-parallel prioritized-replay learner (BASELINE cfg5).

The reference has no distributed mode; its comparator is
one ``learn_step`` at the global batch K = k * N.  This
module defines the sharded algorithm and runs it over ``torch.distributed``
(NCCL on GPUs, gloo on CPU for the tests).  Per learner step, with N ranks
and per-rank batch k:

1. shards: global transition g lives on rank g % N at local slot g // N
   (round-robin insertion); each rank owns an fp64 sum tree over its shard;
2. ``all_gather`` of the shard totals t_r; T = sum_r t_r in rank order, so
   every rank holds bit-identical T and prefix masses c_r;
3. global stratification (replay.py:215-229 over the union of shards):
   q_j = (j + u_j) * (T / K) for j < K with the SAME uniforms on every rank
   (a common generator); query j belongs to the first shard r with
   q_j <= c_r + t_r, and its owner descends its own tree with the local mass
   q_j - c_r (clipped like SumTree.find, replay.py:172-173);
4. ``all_reduce`` (sum; every entry has exactly one non-zero writer) of the
   table (owner, local index, leaf priority); P_j = leaf_j / T and
   w_j = (size * P_j)^-beta / max_j w_j are then computed identically on
   every rank with numpy (the reference's own np.power semantics);
5. rank r learns strata j in [r k, (r+1) k): the owners ship those
   transitions with ``all_to_all_single`` (variable splits);
6. the loss is a sum over the batch, so ``all_reduce`` (sum) of the per-rank
   gradients equals the gradient of the global batch (agent.py:110-131);
7. ``all_gather`` of the TD errors; every owner applies
   ``update_priorities`` to its leaves in global batch order (last write
   wins, replay.py:237-240) and every rank updates max_priority with the max
   over all K errors, so shards stay consistent;
8. every rank applies the same RMSprop update to identical gradients.

For N = 1 this is exactly ``learn_step`` (same queries, same clip, same
descent).  The per-rank compute is a ``Backend``: the device backend
(``DeviceBackend``) runs the libdqn_b200 kernels; the CPU tests plug in the
oracle.  The host orchestration here is plain numpy + torch.distributed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# sharding math (host, numpy; identical on every rank)
# ---------------------------------------------------------------------------

def shard_of(g, world: int):
    """(rank, local slot) of global transition g (round-robin insertion)."""
    g = np.asarray(g, dtype=np.int64)
    return g % world, g // world


def global_slot(rank: int, local, world: int):
    return np.asarray(local, dtype=np.int64) * world + rank


def global_total(totals: np.ndarray) -> float:
    """T = t_0 + t_1 + ... in rank order (fp64, sequential)."""
    s = 0.0
    for t in np.asarray(totals, dtype=np.float64):
        s = s + float(t)
    return s


def stratified_queries(totals: np.ndarray, K: int, u: np.ndarray):
    """Owner rank and local query mass of each of the K strata."""
    totals = np.asarray(totals, dtype=np.float64)
    T = global_total(totals)
    if not T > 0.0:
        raise ValueError("zero total priority; nothing can be sampled")
    seg = T / K
    q = (np.arange(K) + np.asarray(u, dtype=np.float64)) * seg
    q = np.minimum(np.maximum(q, 1e-300), np.nextafter(T, 0.0))
    prefix = np.zeros(len(totals) + 1)
    acc = 0.0
    for r, t in enumerate(totals):
        acc = acc + float(t)
        prefix[r + 1] = acc
    # first shard whose cumulative mass reaches q (q <= prefix[r+1])
    owner = np.searchsorted(prefix[1:], q, side="left")
    owner = np.minimum(owner, len(totals) - 1)
    # skip empty shards (possible only through rounding at a boundary)
    for j in np.nonzero(totals[owner] <= 0.0)[0]:
        r = owner[j]
        while r < len(totals) - 1 and totals[r] <= 0.0:
            r += 1
        owner[j] = r
    q_local = q - prefix[owner]
    return owner.astype(np.int64), q_local, T


def is_weights(leaf: np.ndarray, T: float, size_total: int, beta: float):
    """replay.py:227-229 over the global batch."""
    prob = np.asarray(leaf, dtype=np.float64) / T
    w = np.power(size_total * prob, -beta)
    return prob, w / w.max()


@dataclass
class ExchangePlan:
    """Who sends which strata to whom (all ranks compute the same plan)."""
    send_counts: list       # to each destination
    recv_counts: list       # from each source
    send_strata: np.ndarray  # strata this rank ships, grouped by destination, j order
    recv_order: np.ndarray  # batch position b -> row in the receive buffer


def exchange_plan(owner: np.ndarray, rank: int, world: int, k: int) -> ExchangePlan:
    K = len(owner)
    dest = np.arange(K) // k                       # stratum j is learned by rank j // k
    send_strata = np.nonzero(owner == rank)[0]
    send_strata = send_strata[np.argsort(dest[send_strata], kind="stable")]
    send_counts = [int(np.sum((owner == rank) & (dest == d))) for d in range(world)]
    mine = np.arange(rank * k, (rank + 1) * k)
    recv_counts = [int(np.sum(owner[mine] == s)) for s in range(world)]
    # receive buffer = concat over sources s of (my strata owned by s, in j order)
    offsets = np.concatenate([[0], np.cumsum(recv_counts)[:-1]]).astype(np.int64)
    recv_order = np.empty(k, dtype=np.int64)
    seen = [0] * world
    for b, j in enumerate(mine):
        s = int(owner[j])
        recv_order[b] = offsets[s] + seen[s]
        seen[s] += 1
    return ExchangePlan(send_counts, recv_counts, send_strata, recv_order)


# ---------------------------------------------------------------------------
# the orchestrator
# ---------------------------------------------------------------------------

class Backend:
    """Per-rank compute of one sharded learner step (see DeviceBackend)."""

    def shard_total(self) -> float: ...
    def shard_size(self) -> int: ...
    def max_priority(self) -> float: ...
    def descend(self, q_local: np.ndarray) -> tuple: ...          # -> (local idx, leaf)
    def pack(self, local_idx: np.ndarray): ...                     # -> dict of tensors
    def learn(self, batch: dict, weights: np.ndarray): ...         # -> td (k,) np; grads computed
    def grads(self): ...                                           # flat grad tensor (in place)
    def apply_update(self, local_idx: np.ndarray, td: np.ndarray, max_p: float) -> None: ...
    def optimizer_step(self) -> None: ...


@dataclass
class DpStepResult:
    indices: np.ndarray        # global transition ids of the K strata
    weights: np.ndarray        # IS weights of the K strata
    td_errors: np.ndarray      # K TD errors (global batch order)
    owner: np.ndarray


class DataParallelLearner:
    """Runs the sharded step over a torch.distributed process group."""

    def __init__(self, backend: Backend, k: int, alpha: float, eps: float,
                 comm_device: str = "cpu", group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.b = backend
        self.k = int(k)
        self.alpha, self.eps = float(alpha), float(eps)
        self.dev = comm_device
        # the global running max raw priority = max over the shards' maxima
        self.max_p = float(self._all_gather(
            np.array([backend.max_priority()], dtype=np.float64)).max())

    # -- collectives on host-side numpy values -------------------------------
    def _all_gather(self, arr: np.ndarray) -> np.ndarray:
        import torch
        t = torch.as_tensor(np.ascontiguousarray(arr), device=self.dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return np.concatenate([o.cpu().numpy() for o in out])

    def _all_reduce_sum(self, arr: np.ndarray) -> np.ndarray:
        import torch
        t = torch.as_tensor(np.ascontiguousarray(arr), device=self.dev)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def step(self, u: np.ndarray, beta: float) -> DpStepResult:
        """One global update; ``u`` = rng.random(K) from a generator shared by
        all ranks, ``beta`` = the annealed exponent for this step."""
        import torch
        k, N, r = self.k, self.world, self.rank
        K = k * N
        totals = self._all_gather(np.array([self.b.shard_total()], dtype=np.float64))
        sizes = self._all_gather(np.array([self.b.shard_size()], dtype=np.int64))
        owner, q_local, T = stratified_queries(totals, K, u)
        mine = np.nonzero(owner == r)[0]
        table = np.zeros((K, 2), dtype=np.float64)       # (local index, leaf), owner writes
        if len(mine):
            idx, leaf = self.b.descend(q_local[mine])
            table[mine, 0] = idx
            table[mine, 1] = leaf
        table = self._all_reduce_sum(table)
        local_idx = table[:, 0].astype(np.int64)
        prob, w = is_weights(table[:, 1], T, int(sizes.sum()), beta)
        # ship the strata to the ranks that learn them
        plan = exchange_plan(owner, r, N, k)
        packed = self.b.pack(local_idx[plan.send_strata])
        batch = {}
        for name, t in packed.items():
            send = t.reshape(len(plan.send_strata), -1) if t.dim() > 1 else t.reshape(-1, 1)
            send = send.to(self.dev).contiguous()
            recv = torch.empty((k,) + tuple(send.shape[1:]), dtype=send.dtype, device=self.dev)
            self.dist.all_to_all_single(recv, send, plan.recv_counts, plan.send_counts,
                                        group=self.group)
            recv = recv[torch.as_tensor(plan.recv_order, device=self.dev)]
            batch[name] = recv.reshape((k,) + tuple(t.shape[1:])) if t.dim() > 1 else recv.reshape(k)
        mw = w[r * k:(r + 1) * k]
        td_local = self.b.learn(batch, mw)
        g = self.b.grads()
        gd = g if str(g.device).startswith(self.dev.split(":")[0]) else g.to(self.dev)
        self.dist.all_reduce(gd, group=self.group)
        if gd is not g:
            g.copy_(gd)
        td = self._all_gather(np.asarray(td_local, dtype=np.float64))
        # owners update their leaves in global batch order; max over all K
        self.max_p = max(self.max_p, float((np.abs(td) + self.eps).max()))
        if len(mine):
            self.b.apply_update(local_idx[mine], np.abs(td[mine]), self.max_p)
        self.b.optimizer_step()
        gidx = global_slot(owner, local_idx, N)
        return DpStepResult(indices=gidx, weights=w, td_errors=td, owner=owner)


def max_priority_leaf(max_p: float, alpha: float) -> float:
    return math.pow(max_p, alpha)


class DeviceBackend(Backend):
    """The rank-local compute on the GPU: the shard's sum tree and ring in
    HBM, descent/gather/learn/update/RMSprop through libdqn_b200 (the same
    kernels and step plan as ``learn_step``)."""

    def __init__(self, online, target, memory, optimizer, config):
        from . import agent
        from .replay import PrioritizedReplay
        if not isinstance(memory, PrioritizedReplay):
            raise ValueError("the data-parallel learner shards a PrioritizedReplay")
        self.plan = agent._StepPlan(online, target, memory, optimizer, config)
        self.mem, self.on, self.opt = memory, online, optimizer

    def shard_total(self) -> float:
        return self.mem.tree.total

    def shard_size(self) -> int:
        return self.mem.size

    def max_priority(self) -> float:
        return self.mem.max_priority

    def descend(self, q_local):
        tree = self.mem.tree
        idx = tree.find(np.asarray(q_local, dtype=np.float64))
        leaf = tree.nodes[tree._leaf_base + idx]
        return idx.cpu().numpy(), leaf.cpu().numpy()

    def pack(self, local_idx):
        import torch
        ring = self.mem.memory
        n = len(local_idx)
        idx = torch.as_tensor(np.asarray(local_idx, dtype=np.int64), device="cuda")
        s = torch.empty((n,) + ring.state_shape, dtype=ring.states.dtype, device="cuda")
        s2 = torch.empty_like(s)
        a = torch.empty(n, dtype=torch.int64, device="cuda")
        r = torch.empty(n, dtype=torch.float64, device="cuda")
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        if n:
            ring.gather_into(idx, n, s, s2, a, r, t)
        return {"s": s, "s2": s2, "a": a, "r": r, "t": t}

    def learn(self, batch, weights):
        import torch
        p = self.plan
        k = p.k
        p.x[:k].copy_(batch["s"])
        p.x[k:].copy_(batch["s2"])
        p.a.copy_(batch["a"])
        p.r.copy_(batch["r"])
        p.t.copy_(batch["t"].to(torch.bool))
        p.w.copy_(torch.as_tensor(np.asarray(weights, dtype=np.float64)))
        p.enqueue_learn()
        return p.d_out[k:2 * k].cpu().numpy()

    def grads(self):
        return self.on.flat_grads

    def apply_update(self, local_idx, td, max_p):
        self.mem.update_priorities(np.asarray(local_idx, dtype=np.int64), td)
        self.mem.max_priority = max_p

    def optimizer_step(self) -> None:
        self.opt.step()


# ---------------------------------------------------------------------------
# the device pipeline: one CUDA graph per rank, collectives inside
# ---------------------------------------------------------------------------

class _PeerRing:
    """ctypes mirror of dqn_peer_ring (include/dqn_b200.h)."""

    @staticmethod
    def struct():
        import ctypes as C

        class S(C.Structure):
            _fields_ = [("states", C.c_void_p), ("next_states", C.c_void_p),
                        ("actions", C.c_void_p), ("rewards", C.c_void_p),
                        ("terminals", C.c_void_p)]
        return S


_RING_FIELDS = ("states", "next_states", "actions", "rewards", "terminals")


class DeviceDataParallelLearner:
    """The sharded learner of this module as a device pipeline (csrc/dp.cu):
    every step of ``DataParallelLearner.step`` is a fixed-size kernel or NCCL
    collective, captured once into a CUDA graph per rank and replayed.

    * shard infos: ``all_gather`` of [total, size, max_p] (N x 24 B);
    * routing, owner descent, the (index, leaf) table ``all_reduce`` (K x 16 B)
      and the IS weights on the device, identical on every rank;
    * frames: each rank reads its K/N strata straight from the owners' rings
      through CUDA IPC mappings (NVLink peer loads in ``dqn_dp_gather``), so
      no frame bytes go through a collective;
    * the local update (the single-GPU learner's forward/backward/wgrad
      graph), gradient ``all_reduce`` (6.7 MB, NCCL), TD ``all_gather``,
      owner-side priority update in global batch order, flag ``all_reduce``
      (max) so every rank skips a failed step together, RMSprop.

    ``memory`` must be a ``PrioritizedReplay(..., shareable=True)`` when the
    world size is above one.  ``step(u, beta)`` takes the K = k * N uniforms
    from a generator common to all ranks and returns a ``DpStepResult``.
    """

    def __init__(self, online, target, memory, optimizer, config, group=None, *,
                 _emulated=None):
        """``_emulated`` (tests only): ``(rank, world, comm_factory, rings)``
        -- ranks as threads of one process on one GPU, collectives emulated
        on the host by ``comm_factory()``, ``rings`` the N shard memories
        (local pointers instead of IPC mappings)."""
        import ctypes as C
        import torch
        from . import _lib, agent, nccl
        from .replay import PrioritizedReplay
        if not isinstance(memory, PrioritizedReplay):
            raise ValueError("the data-parallel learner shards a PrioritizedReplay")
        if _emulated is None:
            import torch.distributed as dist
            self.rank = dist.get_rank(group)
            self.world = N = dist.get_world_size(group)
            make_comm = lambda: nccl.Communicator(group)  # noqa: E731
        else:
            self.rank, N, make_comm, emu_rings = _emulated
            self.world = N
        self.mem, self.on, self.opt = memory, online, optimizer
        self.k = k = int(config.batch_size)
        self.K = K = k * N
        if K > 1024:
            raise ValueError("global batch above 1024 strata")
        self.alpha, self.eps = float(memory.config.alpha), float(memory.config.epsilon)
        self.grad_clip = float(getattr(config, "grad_clip", 0.0))
        self.plan = agent._StepPlan(online, target, memory, optimizer, config)
        self.plan.grad_clip = 0.0          # clipping applies to the reduced gradient (below)
        self.comm = make_comm()
        # the TD all_gather runs on the priority stream beside the backward
        # pass: a second communicator keeps its order independent of the
        # gradient all_reduce on the main stream
        self.comm_td = make_comm()
        ring = memory.memory
        # peer rings: own arrays locally, the others' through IPC mappings
        own = [getattr(ring, f).data_ptr() for f in _RING_FIELDS]
        if N > 1 and _emulated is None:
            if not ring.shared:
                raise ValueError("world size > 1 needs PrioritizedReplay(..., shareable=True)")
            mine = [ring.shared[f].handle() for f in _RING_FIELDS]
            allh = [None] * N
            dist.all_gather_object(allh, mine, group=group)
        S = _PeerRing.struct()
        table = (S * N)()
        self._opened = []
        for r in range(N):
            if _emulated is not None:
                ptrs = [getattr(emu_rings[r].memory, f).data_ptr() for f in _RING_FIELDS]
            elif r == self.rank:
                ptrs = own
            else:
                ptrs = []
                for h in allh[r]:
                    p = C.c_void_p()
                    _lib.call("dqn_ipc_open", (C.c_uint8 * 64).from_buffer_copy(h), C.byref(p))
                    self._opened.append(p)
                    ptrs.append(p.value)
            table[r] = S(*ptrs)
        raw = bytes(table)
        self.rings = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to("cuda")
        dev = "cuda"
        f64 = torch.float64
        self.h_in = torch.zeros(K + 1, dtype=f64).pin_memory()          # u | beta
        self.d_in = torch.zeros(K + 1, dtype=f64, device=dev)
        self.info = torch.zeros(3, dtype=f64, device=dev)
        self.info_all = torch.zeros(3 * N, dtype=f64, device=dev)
        self.owner = torch.zeros(K, dtype=torch.int64, device=dev)
        self.q_local = torch.zeros(K, dtype=f64, device=dev)
        self.sums = torch.zeros(3, dtype=f64, device=dev)
        self.table = torch.zeros(2 * K, dtype=f64, device=dev)
        self.local_idx = torch.zeros(K, dtype=torch.int64, device=dev)
        self.w_all = torch.zeros(K, dtype=f64, device=dev)
        self.td_all = torch.zeros(K, dtype=f64, device=dev)
        self.idx_c = torch.zeros(K, dtype=torch.int64, device=dev)
        self.td_c = torch.zeros(K, dtype=f64, device=dev)
        self.n_c = torch.zeros(1, dtype=torch.int32, device=dev)
        self.norm = torch.zeros(1, dtype=f64, device=dev)
        # results: td | w | owner | local idx (as f64) + flags
        self.d_res = torch.zeros(4 * K, dtype=f64, device=dev)
        self.h_res = torch.zeros(4 * K, dtype=f64).pin_memory()
        self.h_flags = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.h_in_np, self.h_res_np = self.h_in.numpy(), self.h_res.numpy()
        self.h_flags_np = self.h_flags.numpy()
        self.graph = self.graph_exec = None
        self.calls = 0

    def close(self) -> None:
        from . import _lib
        for p in self._opened:
            _lib.lib.dqn_ipc_close(p)
        self._opened = []
        self.comm.close()
        self.comm_td.close()

    def enqueue(self) -> None:
        """One global update on the current stream (capturable)."""
        from . import _lib, nccl
        p, k, K, N = self.plan, self.k, self.K, self.world
        st = _lib.stream_ptr()
        tree, ring = self.mem.tree, self.mem.memory
        flags = p.flags
        # the draws are read where they are: pinned host memory (zero-copy) or,
        # in the bench's device loop, a device slot
        src = self.h_in
        _lib.call("dqn_dp_shard_info", st, tree.nodes.data_ptr(), ring._size_dev.data_ptr(),
                  self.mem._max_p.data_ptr(), self.info.data_ptr())
        self.comm.all_gather(self.info, self.info_all, st)
        # routing with the owner descent fused in -> (index, leaf) table
        _lib.call("dqn_dp_route", st, self.info_all.data_ptr(), N, src.data_ptr(), K,
                  self.owner.data_ptr(), self.q_local.data_ptr(), self.sums.data_ptr(),
                  flags.data_ptr(), tree.nodes.data_ptr(), tree.depth, self.rank,
                  self.table.data_ptr())
        self.comm.all_reduce(self.table, nccl.NCCL_SUM, st)
        # peer-ring gather of this rank's strata, IS weights in the same launch
        _lib.call("dqn_dp_gather", st, self.rings.data_ptr(), self.owner.data_ptr(),
                  self.table.data_ptr(), k, self.rank, ring.slot_bytes, p.x.data_ptr(),
                  p.a.data_ptr(), p.r.data_ptr(), p.t.data_ptr(), self.sums.data_ptr(),
                  src[K:].data_ptr(), K, self.local_idx.data_ptr(), self.w_all.data_ptr(),
                  p.w.data_ptr())

        def td_branch():
            # beside the backward pass (priority stream): TD errors of all
            # ranks, the owned strata in global order, this shard's update
            s2 = _lib.stream_ptr()
            self.comm_td.all_gather(p.d_out[k:2 * k], self.td_all, s2)
            _lib.call("dqn_dp_owned", s2, self.owner.data_ptr(), self.local_idx.data_ptr(),
                      self.td_all.data_ptr(), K, self.rank, self.eps, self.idx_c.data_ptr(),
                      self.td_c.data_ptr(), self.n_c.data_ptr(), self.mem._max_p.data_ptr(),
                      flags.data_ptr(), self.sums.data_ptr())
            _lib.call("dqn_tree_update_n", s2, tree.nodes.data_ptr(), tree.depth,
                      ring._size_dev.data_ptr(), self.idx_c.data_ptr(), self.td_c.data_ptr(), K,
                      self.n_c.data_ptr(), self.alpha, self.eps, None, flags.data_ptr())

        p.enqueue_learn(td_hook=td_branch)
        g = self.on.flat_grads
        self.comm.all_reduce(g, nccl.NCCL_SUM, st)
        self.comm.all_reduce(flags, nccl.NCCL_MAX, st)
        if self.grad_clip > 0.0:
            _lib.call("dqn_clip_gradients", st, g.data_ptr(), self.on.n_flat, self.grad_clip,
                      self.norm.data_ptr())
            self.opt.enqueue_step(flags)
        else:
            self.opt.enqueue_apply(flags)
        # results and the status word straight into pinned host memory
        _lib.call("dqn_dp_report", st, self.td_all.data_ptr(), self.w_all.data_ptr(),
                  self.owner.data_ptr(), self.local_idx.data_ptr(), K, flags.data_ptr(),
                  self.h_res.data_ptr(), self.h_flags.data_ptr())

    def step(self, u: np.ndarray, beta: float) -> DpStepResult:
        from . import _lib, agent
        from .errors import NonFiniteError
        K = self.K
        self.h_in_np[:K] = np.asarray(u, dtype=np.float64)
        self.h_in_np[K] = float(beta)
        self.h_flags_np[0] = agent._SENTINEL
        if self.graph_exec is None and self.calls >= 1 and agent.USE_GRAPH:
            self.graph, self.graph_exec = agent.capture_graph(self.enqueue,
                                                              self.plan.capture_stream)
        if self.graph_exec is not None:
            self.graph_exec.launch(_lib.stream_ptr())
        else:
            self.enqueue()
        self.calls += 1
        hf = self.h_flags_np
        for _ in range(200_000):               # the report kernel writes it last
            if hf[0] != agent._SENTINEL:
                break
        else:
            agent._device_sync()
        f = int(hf[0])
        if f == agent._SENTINEL:
            agent._device_sync()
            f = int(hf[0])
            if f == agent._SENTINEL:
                raise RuntimeError("data-parallel update finished without its status word")
        if f:
            self.plan.flags.zero_()
            if f & _lib.FLAG_ZERO_TOTAL:
                raise ValueError("zero total priority; nothing can be sampled")
            if f & _lib.FLAG_NONFINITE_OUT:
                raise NonFiniteError("non-finite network output")
            if f & _lib.FLAG_INDEX:
                raise IndexError("transition index out of range")
            if f & _lib.FLAG_BAD_PRIORITY:
                raise ValueError("priority must be finite and >= 0")
            raise NonFiniteError("non-finite gradient; step aborted")
        h = self.h_res_np
        owner = h[2 * K:3 * K].astype(np.int64)
        local = h[3 * K:].astype(np.int64)
        return DpStepResult(indices=global_slot(owner, local, self.world), weights=h[K:2 * K].copy(),
                            td_errors=h[:K].copy(), owner=owner)
