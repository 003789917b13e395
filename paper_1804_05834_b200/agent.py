"""The learner update on the GPU: ``learn_step`` and the target helpers
(deepq/agent.py:58-132) with the reference's signatures.

``learn_step(online, target, memory, optimizer, config, step, rng)`` takes the
replay draws from the caller's ``rng`` on the host exactly as the reference
does (``rng.random(k)`` for PER, ``rng.integers(0, size, k)`` for uniform),
copies them to HBM, runs the whole update on the device and returns a
``TdResult`` of host numpy arrays.  Per (networks, memory, optimizer, config)
tuple a ``_StepPlan`` owns the device buffers; after the first (eager) call
the update is captured into one CUDA graph and replayed, so a step costs one
graph launch plus two small copies (draws in, TdResult out).

Device pipeline of one update:
  dqn_tree_sample -> dqn_ring_gather (s and s' into one [2k] batch)
  -> online forward on [s; s'] -> target forward on s' -> dqn_td_loss
  (argmax, bootstrap, delta, loss, output grad written straight into the
  online net's y.grad) -> backward (conv1 dX skipped) -> wgrad
  -> [clip] -> dqn_tree_update -> dqn_rmsprop_step.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NonFiniteError
from .network import _FORWARD, _GRAD, Network
from .optim import RmsProp, clip_gradients, sync_target  # noqa: F401  (re-export)
from .replay import PrioritizedReplay, ReplayMemory, SampleBatch


@dataclass
class TdResult:
    targets: np.ndarray
    td_errors: np.ndarray
    losses: np.ndarray

    @property
    def mean_abs_td(self) -> float:
        return float(np.mean(np.abs(self.td_errors)))

    @property
    def mean_loss(self) -> float:
        return float(np.mean(self.losses))


def _td_flags(config) -> int:
    f = 0
    if getattr(config, "double", True):
        f |= _lib.TD_DOUBLE
    if getattr(config, "huber", False):
        f |= _lib.TD_HUBER
    if getattr(config, "reward_clip", False):
        f |= _lib.TD_REWARD_CLIP
    return f


def _targets_only(batch: SampleBatch, online, target, gamma: float, double: bool):
    torch = _lib.require_cuda()

    def dev(x, dtype):      # tensors or array-likes (duck-typed nets / batches)
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
        return t.to(device="cuda", dtype=dtype).contiguous()

    k = len(batch.rewards)
    q_tg = dev(target.forward(batch.next_states), torch.float32).clone()
    if double:
        q_on2 = dev(online.forward(batch.next_states), torch.float32).clone()
    else:
        q_on2 = q_tg
    out = [torch.empty(k, dtype=torch.float64, device="cuda") for _ in range(3)]
    dq = torch.empty_like(q_tg)
    acts = torch.zeros(k, dtype=torch.int64, device="cuda")
    r = dev(batch.rewards, torch.float64)
    t = dev(batch.terminals, torch.bool)
    w = torch.ones(k, dtype=torch.float64, device="cuda")
    _lib.call("dqn_td_loss", _lib.stream_ptr(), q_on2.data_ptr(), q_on2.data_ptr(),
              q_tg.data_ptr(), acts.data_ptr(), r.data_ptr(), t.data_ptr(), w.data_ptr(), k,
              q_tg.shape[1], float(gamma), _lib.TD_DOUBLE if double else 0,
              out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), dq.data_ptr(), None)
    return out[0]


def compute_target_dqn(batch: SampleBatch, target_net, gamma: float):
    """``y = r + gamma * max_a Q_target(s', a)``, ``y = r`` on terminals (agent.py:58-63)."""
    return _targets_only(batch, None, target_net, gamma, False)


def compute_target_double(batch: SampleBatch, online_net, target_net, gamma: float):
    """Online net picks a* (first max), target net evaluates it (agent.py:66-73)."""
    return _targets_only(batch, online_net, target_net, gamma, True)


class _StepPlan:
    """Device buffers (and, after warm-up, the CUDA graph) of one learner
    configuration."""

    def __init__(self, online: Network, target: Network, memory, optimizer: RmsProp, config):
        torch = _lib.require_cuda()
        self.online, self.target, self.memory, self.opt = online, target, memory, optimizer
        self.per = isinstance(memory, PrioritizedReplay)
        self.ring: ReplayMemory = memory.memory if self.per else memory
        self.k = k = int(config.batch_size)
        self.double = bool(getattr(config, "double", True))
        self.gamma = float(config.gamma)
        self.flags_td = _td_flags(config)
        self.grad_clip = float(getattr(config, "grad_clip", 0.0))
        self.nA = online.output_shape[-1]
        dev = "cuda"
        ring = self.ring
        self.x = torch.empty((2 * k,) + ring.state_shape, dtype=ring.state_dtype, device=dev)
        self.a = torch.empty(k, dtype=torch.int64, device=dev)
        self.r = torch.empty(k, dtype=torch.float64, device=dev)
        self.t = torch.empty(k, dtype=torch.bool, device=dev)
        self.idx = torch.empty(k, dtype=torch.int64, device=dev)
        self.idx_w = torch.empty(k, dtype=torch.int64, device=dev)   # the weights launch's copy
        self._e_weights = None
        self.prob = torch.empty(k, dtype=torch.float64, device=dev)
        self.w = torch.ones(k, dtype=torch.float64, device=dev)
        # inputs: u[k] + beta (PER) | indices[k] (uniform); pinned staging
        self.d_in = torch.zeros(k + 1, dtype=torch.float64, device=dev)
        self.h_in = torch.zeros(k + 1, dtype=torch.float64).pin_memory()
        self.h_idx = torch.zeros(k, dtype=torch.int64).pin_memory()
        # outputs: targets | td | losses | stats(2)  + flags
        self.d_out = torch.zeros(3 * k + 2, dtype=torch.float64, device=dev)
        self.h_out = torch.zeros(3 * k + 2, dtype=torch.float64).pin_memory()
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.h_flags = torch.zeros(1, dtype=torch.int32).pin_memory()
        # numpy views of the pinned staging buffers (the per-step host path)
        self.h_in_np, self.h_idx_np = self.h_in.numpy(), self.h_idx.numpy()
        self.h_out_np, self.h_flags_np = self.h_out.numpy(), self.h_flags.numpy()
        self.norm = torch.zeros(1, dtype=torch.float64, device=dev)
        on_rows = 2 * k if self.double else k
        self.on_bind = online.binding(on_rows)
        self.on_view = online.prefix_binding(self.on_bind, k) if self.double else self.on_bind
        # wgrad runs on a side stream concurrently with the dgrad chain: it
        # gets a view with its own scratch (split-K partials and counters)
        self.on_wview = online.prefix_binding(self.on_bind, k, own_scratch=True)
        self.tg_bind = target.binding(k)
        # the target trunk (k rows) beside the online one on [s; s'] (2k rows,
        # the critical path): leaner launches for it.  Without Double DQN the
        # two trunks are the same size and share the GPU evenly.
        self.tg_desc = target.hinted(self.x, _lib.NET_HINT_SIDE) if self.double else None
        # the Q heads, TD block, head backward and head wgrad run as one fused
        # launch (dqn_head_td) when the head fits it (nA <= 18, batch <= 1024)
        units = online._units
        self.head_layer = len(units) - 1
        self.fused_head = (len(units) >= 2 and units[-1]["kind"] in (_lib.LAYER_LINEAR,
                                                                     _lib.LAYER_DUELING)
                           and self.nA <= 18 and k <= 1024 and FUSED_HEAD)
        self.head_work = torch.zeros(int(_lib.lib.dqn_head_td_work_bytes(k, self.nA)),
                                     dtype=torch.uint8, device=dev)
        self.on_desc = online.desc_for(self.x)
        self.fused_sample = (ring.fused_ok and ring.slot_bytes % 16 == 0
                             and ring.state_dtype == torch.uint8 and FUSED_SAMPLE)
        # the head's form is fixed when the plan is built (and so in its graph)
        self.head_two_phase = HEAD_TWO_PHASE
        if not self.head_two_phase:
            self.flags_td |= _lib.TD_HEAD_LAST_CTA
        # zero-copy results are written by the two-phase head's kernels
        self.zero_copy = k * (self.nA + 1) <= 2048 and self.head_two_phase
        self._host_out = None
        self.side = torch.cuda.Stream()
        self.tree_stream = torch.cuda.Stream()
        self.capture_stream = torch.cuda.Stream()
        self.graph = None
        self.graph_exec = None
        self.dev = torch.cuda.current_device()
        self.calls = 0
        self.h2d_bytes = (k + 1) * 8 if self.per else k * 8
        self.d2h_bytes = (3 * k + 2) * 8 + 4

    # -- the device pipeline ----------------------------------------------
    def _weights_beside(self, tree, ring, src, k: int) -> None:
        """prob / IS weights of this batch (dqn_tree_sample: the same
        descents as the gather's) on the tree stream once the gather is
        enqueued; the head waits for them (enqueue_learn)."""
        torch = _lib.require_cuda()
        e_fork = torch.cuda.Event()
        e_fork.record(torch.cuda.current_stream())
        with torch.cuda.stream(self.tree_stream):
            self.tree_stream.wait_event(e_fork)
            _lib.call("dqn_tree_sample", _lib.stream_ptr(), tree.nodes.data_ptr(), tree.depth,
                      ring._size_dev.data_ptr(), src.data_ptr(), k, src[k:].data_ptr(),
                      self.idx_w.data_ptr(), self.prob.data_ptr(), self.w.data_ptr(),
                      self.flags.data_ptr())
            self._e_weights = torch.cuda.Event()
            self._e_weights.record(self.tree_stream)

    def enqueue(self, io: bool = True) -> None:
        """Enqueue one update; ``io`` adds the pinned host copies of the
        draws (in) and TdResult + flags (out)."""
        torch = _lib.require_cuda()
        st = _lib.stream_ptr()
        k, ring = self.k, self.ring
        # zero-copy I/O: the draws are read from pinned host memory by the
        # first kernel, TdResult and the flag word are written to pinned host
        # memory by the head and the optimizer kernels -- no memcpy nodes
        zc = (io and self.zero_copy and self.fused_head and self.grad_clip == 0.0
              and (self.fused_sample or not self.per))
        self._host_out = self.h_out if zc else None
        if self.per and self.fused_sample:
            # descent + frame gather in one launch (the IS weights beside it:
            # WEIGHTS_BESIDE), reading the draws where they are (pinned host
            # buffer, or a device slot)
            src = self.h_in
            if not zc and src.device.type == "cpu":
                self.d_in.copy_(self.h_in, non_blocking=True)
                src = self.d_in
            tree = self.memory.tree
            if hasattr(ring, "sample_gather_fused"):       # frame-deduplicated ring
                beside = WEIGHTS_BESIDE
                ring.sample_gather_fused(tree, src, k, src[k:], self.idx,
                                         None if beside else self.prob,
                                         None if beside else self.w,
                                         self.flags, self.x, self.x[k:], self.a, self.r, self.t)
                if beside:
                    self._weights_beside(tree, ring, src, k)
            elif not WEIGHTS_BESIDE:
                _lib.call("dqn_sample_gather", st, tree.nodes.data_ptr(), tree.depth,
                          ring._size_dev.data_ptr(), src.data_ptr(), k,
                          src[k:].data_ptr(), self.idx.data_ptr(), self.prob.data_ptr(),
                          self.w.data_ptr(), self.flags.data_ptr(), ring.states.data_ptr(),
                          ring.next_states.data_ptr(), ring.slot_bytes, ring.actions.data_ptr(),
                          ring.rewards.data_ptr(), ring.terminals.data_ptr(), self.x.data_ptr(),
                          self.x[k:].data_ptr(), self.a.data_ptr(), self.r.data_ptr(),
                          self.t.data_ptr())
            else:
                # the IS weights (a batch-wide max) by their own launch on the
                # tree stream once the gather is done, beside the trunk: only
                # the head reads them, and as the fused launch's extra CTA row
                # they held up conv1
                _lib.call("dqn_sample_gather", st, tree.nodes.data_ptr(), tree.depth,
                          ring._size_dev.data_ptr(), src.data_ptr(), k,
                          src[k:].data_ptr(), self.idx.data_ptr(), None, None,
                          self.flags.data_ptr(), ring.states.data_ptr(),
                          ring.next_states.data_ptr(), ring.slot_bytes, ring.actions.data_ptr(),
                          ring.rewards.data_ptr(), ring.terminals.data_ptr(), self.x.data_ptr(),
                          self.x[k:].data_ptr(), self.a.data_ptr(), self.r.data_ptr(),
                          self.t.data_ptr())
                self._weights_beside(tree, ring, src, k)
        else:
            idx = self.idx
            if self.per:
                self.d_in.copy_(self.h_in, non_blocking=True)
                self.memory.sample_indices(self.d_in[:k], k, self.d_in[k:], self.idx, self.prob,
                                           self.w, self.flags)
            elif zc:
                idx = self.h_idx                  # uniform draws read in place (pinned)
            else:
                self.idx.copy_(self.h_idx, non_blocking=True)
            ring.gather_into(idx, k, self.x[:k], self.x[k:], self.a, self.r, self.t)
        # priorities are updated inside enqueue_learn, beside the backward pass
        self.enqueue_learn(priorities=self.per)
        if self.grad_clip > 0.0:
            self.opt.enqueue_step(self.flags)      # clipping rescales: rescan
        else:
            # every gradient of the update came from launches that flagged
            # non-finite values into self.flags as they wrote them
            self.opt.enqueue_apply(self.flags, flag_out=self.h_flags if zc else None)
        if io and not zc:
            self.h_out.copy_(self.d_out, non_blocking=True)
            self.h_flags.copy_(self.flags, non_blocking=True)
        del torch

    def enqueue_learn(self, priorities: bool = False, td_hook=None) -> None:
        """Targets, TD loss, backward and wgrad from the batch already in
        self.x ([s; s']), self.a/r/t and IS weights self.w.

        Two streams (both captured into the step's CUDA graph): the target
        forward runs beside the online forward, and each layer's wgrad runs
        beside the rest of the dgrad chain as soon as that layer's output
        gradient exists (it has its own scratch / split-K counters); the first
        layer's wgrad, which has no dgrad beside it, stays on the main stream.
        With ``priorities`` the sum-tree update (replay.py:232-241) runs on a
        third stream as soon as the TD errors exist and joins before the
        optimizer, which still sees its error flags first."""
        torch = _lib.require_cuda()
        st = _lib.stream_ptr()
        k = self.k
        on, tg = self.online, self.target
        s0, s1 = torch.cuda.current_stream(), self.side
        ev = torch.cuda.Event
        e_in = ev()
        e_in.record(s0)
        upto = self.head_layer if self.fused_head else None

        def forward(net, x, bind, desc=None):
            net.forward_into(x, bind, upto=upto, desc=desc)
        with torch.cuda.stream(s1):
            s1.wait_event(e_in)
            forward(tg, self.x[k:], self.tg_bind, self.tg_desc)
            e_tg = ev()
            e_tg.record(s1)
        forward(on, self.x if self.double else self.x[:k], self.on_bind)
        s0.wait_event(e_tg)
        nA = self.nA
        out = self.d_out
        for v in (self.on_view, self.on_wview):
            v.x = self.x[:k]
            v.struct.x = self.x.data_ptr()
            v.struct.dx = None                     # conv1 dX is never needed
        if self._e_weights is not None:           # the IS weights' launch (enqueue)
            s0.wait_event(self._e_weights)
            self._e_weights = None
        if self.fused_head:
            # both Q heads + targets/TD/loss + head dX + head wgrad in one launch
            _lib.call("dqn_head_td", st, C.byref(on.desc_for(self.x)), on.flat_values.data_ptr(),
                      on.flat_grads.data_ptr(), C.byref(self.on_bind.struct),
                      C.byref(self.on_view.struct), C.byref(tg.desc_for(self.x)),
                      tg.flat_values.data_ptr(), C.byref(self.tg_bind.struct),
                      self.a.data_ptr(), self.r.data_ptr(), self.t.data_ptr(), self.w.data_ptr(),
                      self.gamma, self.flags_td, out[:k].data_ptr(), out[k:2 * k].data_ptr(),
                      out[2 * k:3 * k].data_ptr(), out[3 * k:].data_ptr(),
                      self.head_work.data_ptr(), self.flags.data_ptr(),
                      None if self._host_out is None else self._host_out.data_ptr())
            first = self.head_layer - 1
        else:
            q_on = self.on_bind.act[-1]
            _lib.call("dqn_td_loss", st, q_on.data_ptr(),
                      q_on[k * nA:].data_ptr() if self.double else None,
                      self.tg_bind.act[-1].data_ptr(), self.a.data_ptr(), self.r.data_ptr(),
                      self.t.data_ptr(), self.w.data_ptr(), k, nA, self.gamma, self.flags_td,
                      out[:k].data_ptr(), out[k:2 * k].data_ptr(), out[2 * k:3 * k].data_ptr(),
                      self.on_view.dact[-1].data_ptr(), out[3 * k:].data_ptr())
            first = len(on._units) - 1
        e = ev()
        e.record(s0)
        e_tree = None
        if priorities or td_hook is not None:
            # ``td_hook`` (the data-parallel learner) replaces the local
            # priority update with its own work on the TD errors
            with torch.cuda.stream(self.tree_stream):
                self.tree_stream.wait_event(e)
                if td_hook is not None:
                    td_hook()
                else:
                    self.memory.update_priorities_dev(self.idx, out[k:2 * k], k, self.flags)
                e_tree = ev()
                e_tree.record(self.tree_stream)
        for layer in reversed(range(first + 1)):
            if layer == 0:
                # conv1 has no dgrad: its wgrad takes the main stream (and the
                # dgrad binding's scratch) instead of queueing behind conv2's
                on.layer_into(self.on_view, 0, 2, self.flags)
                break
            with torch.cuda.stream(s1):           # wgrad of `layer` once its grad exists
                s1.wait_event(e)
                on.layer_into(self.on_wview, layer, 2, self.flags)
            on.layer_into(self.on_view, layer, 1)  # dgrad chain continues on s0
            e = ev()
            e.record(s0)
        e_w = ev()
        e_w.record(s1)
        s0.wait_event(e_w)
        if e_tree is not None:
            s0.wait_event(e_tree)
        if self.grad_clip > 0.0:
            _lib.call("dqn_clip_gradients", st, on.flat_grads.data_ptr(), on.n_flat,
                      self.grad_clip, self.norm.data_ptr())

    def last_indices(self):
        """Replay slots sampled by the last update (device tensor for PER;
        for uniform replay the host draws, which zero-copy reads in place)."""
        return self.idx if self.per else self.h_idx

    def run(self, use_graph: bool) -> None:
        if use_graph and self.graph_exec is not None:   # hot path: one graph launch
            rc = _GRAPH_LAUNCH(self.graph_exec.ptr, _RAW_STREAM(self.dev))
            if rc:
                _lib.raise_status(rc, "dqn_graph_launch")
            self.calls += 1
            return
        torch = _lib.require_cuda()
        if use_graph and self.graph is None and self.calls >= 1:
            self.graph, self.graph_exec = capture_graph(self.enqueue, self.capture_stream)
        if use_graph and self.graph_exec is not None:
            self.graph_exec.launch(_lib.stream_ptr())
        else:
            self.enqueue()
        self.calls += 1


_PLANS: dict = {}
USE_GRAPH = os.environ.get("DQN_B200_GRAPH", "1") != "0"
# Launch-form switches, read when a step plan is built (tests compare the
# forms; each alternative was measured and the defaults are the fastest):
FUSED_HEAD = True       # Q heads + TD block + head backward/wgrad in dqn_head_td
HEAD_TWO_PHASE = True   # its two-phase form (else the last-CTA-ticket form)
FUSED_SAMPLE = True     # sum-tree descent + frame gather in one launch
WEIGHTS_BESIDE = True   # its IS weights by a separate launch on the tree stream
_GRAPH_LAUNCH = _lib.lib.dqn_graph_launch


def _RAW_STREAM(dev: int) -> int:
    # the caller's current stream (raw pointer) without building a Stream object
    import torch
    global _RAW_STREAM
    _RAW_STREAM = torch._C._cuda_getCurrentRawStream
    return _RAW_STREAM(dev)


class _Exec:
    """An instantiated graph (cudaGraphExec_t), destroyed with its owner."""

    def __init__(self, graph):
        self.ptr = C.c_void_p()
        _lib.call("dqn_graph_instantiate", C.c_void_p(graph.raw_cuda_graph()),
                  0, C.byref(self.ptr))
        self._fin = weakref.finalize(self, _lib.lib.dqn_graph_destroy, self.ptr)

    @property
    def _as_parameter_(self):
        return self.ptr

    def launch(self, stream_ptr: int) -> None:
        rc = _GRAPH_LAUNCH(self.ptr, stream_ptr)
        if rc:
            _lib.raise_status(rc, "dqn_graph_launch")


def capture_graph(fn, stream):
    """Capture ``fn()`` on ``stream`` (its priority becomes the priority of
    the kernel nodes launched on it) and instantiate the graph honouring
    node priorities.  Returns (torch CUDAGraph owning the graph and its
    memory pool, _Exec)."""
    torch = _lib.require_cuda()
    g = torch.cuda.CUDAGraph(keep_graph=True)
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            fn()
    torch.cuda.current_stream().wait_stream(stream)
    return g, _Exec(g)


def _CUDAGraph_replay(g) -> None:
    # torch.cuda.CUDAGraph.replay without the Python wrapper (a few us per call)
    type(g).__mro__[1].replay(g)


def _device_sync() -> None:
    # the learner's stream work is all this process has on the device; a plain
    # cudaDeviceSynchronize skips torch's Python stream/device lookups
    import torch
    torch._C._cuda_synchronize()


def _plan_for(online, target, memory, optimizer, config) -> _StepPlan:
    key = (id(online), id(target), id(memory), id(optimizer), int(config.batch_size),
           bool(getattr(config, "double", True)), float(config.gamma), _td_flags(config),
           float(getattr(config, "grad_clip", 0.0)))
    p = _PLANS.get(key)
    if p is None or p.online is not online or p.memory is not memory:
        p = _StepPlan(online, target, memory, optimizer, config)
        _PLANS[key] = p
    return p


def learn_step_enqueue(plan: _StepPlan, step: int, rng: np.random.Generator) -> None:
    """Stage this step's draws and launch the update without waiting."""
    k = plan.k
    plan.h_flags_np[0] = _SENTINEL      # overwritten by the update's last copy
    if plan.per:
        hin = plan.h_in_np
        hin[:k] = rng.random(k)
        hin[k] = plan.memory.beta(step)
    else:
        plan.h_idx_np[:] = rng.integers(0, plan.ring.size, size=k)
    plan.run(USE_GRAPH)


_POLL_SPINS = 200_000          # ~20-50 ms of polling, then a blocking synchronize


def _wait_result(plan: _StepPlan) -> None:
    """The graph's last node copies the flag word to pinned host memory; the
    host set it to a sentinel before the launch, so polling it observes the
    end of the update (the TdResult copy precedes it on the same stream)
    a few microseconds sooner than cudaDeviceSynchronize wakes up.  Errors
    and slow steps fall through to the synchronize, which raises."""
    hf = plan.h_flags_np
    if plan.graph is not None and USE_GRAPH:
        for _ in range(_POLL_SPINS):
            if hf[0] != _SENTINEL:
                return
    _device_sync()


_SENTINEL = -(1 << 30)


def learn_step_collect(plan: _StepPlan) -> TdResult:
    _wait_result(plan)
    k = plan.k
    f = int(plan.h_flags_np[0])
    if f == _SENTINEL:      # the update's completion word was never written
        raise RuntimeError("learner update finished without reporting its status word")
    if f:
        # the step was aborted on the device; let the update's remaining
        # launches finish before raising
        torch = _lib.require_cuda()
        torch.cuda.current_stream().synchronize()
        plan.flags.zero_()
        if f & _lib.FLAG_ZERO_TOTAL:
            raise ValueError("zero total priority; nothing can be sampled")
        if f & _lib.FLAG_NONFINITE_OUT:
            raise NonFiniteError("non-finite network output")
        if f & _lib.FLAG_INDEX:
            raise IndexError("transition index out of range")
        if f & _lib.FLAG_BAD_PRIORITY:
            raise ValueError("priority must be finite and >= 0")
        if f & _lib.FLAG_NONFINITE_GRAD:
            raise NonFiniteError("non-finite gradient; step aborted")
    h = plan.h_out_np
    plan.online._set_current(plan.on_view, _GRAD)
    plan.target._set_current(plan.tg_bind, _FORWARD)
    return TdResult(targets=h[:k].copy(), td_errors=h[k:2 * k].copy(), losses=h[2 * k:3 * k].copy())


def learn_step(online: Network, target: Network, memory, optimizer: RmsProp, config, step: int,
               rng: np.random.Generator) -> TdResult:
    """One optimisation step (agent.py:91-132) on the GPU."""
    if memory.size == 0:
        raise ValueError("cannot sample from an empty replay memory")
    plan = _plan_for(online, target, memory, optimizer, config)
    learn_step_enqueue(plan, step, rng)
    return learn_step_collect(plan)
