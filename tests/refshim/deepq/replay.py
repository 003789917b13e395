"""deepq.replay over the device ring / sum tree (host arrays out)."""

from __future__ import annotations

import numpy as np

import paper_1804_05834_b200 as P
from paper_1804_05834_b200.replay import PriorityConfig, SampleBatch, Transition, anneal_beta  # noqa: F401

from ._host import HostView, to_np


def _host_batch(b):
    return SampleBatch(*(to_np(getattr(b, f)) for f in
                         ("states", "actions", "rewards", "next_states", "terminals", "indices",
                          "probabilities", "weights")))


def _ring_dtype(dtype):
    return np.uint8 if np.dtype(dtype) == np.uint8 else np.float32


class SumTree:
    def __init__(self, capacity=None, _tree=None):
        self._tree = _tree if _tree is not None else P.SumTree(capacity)

    @property
    def total(self):
        return float(self._tree.total)

    @property
    def nodes(self):
        return to_np(self._tree.nodes)

    @property
    def _leaf_base(self):
        return self._tree._leaf_base

    def leaf(self, i):
        return float(self._tree.leaf(i))

    def leaves(self):
        return to_np(self._tree.leaves())

    def set(self, i, p):
        self._tree.set(i, p)

    def find(self, values):
        return to_np(self._tree.find(values))

    def __getattr__(self, name):
        return getattr(self._tree, name)


class ReplayMemory:
    def __init__(self, capacity, state_shape, dtype=np.float32, _mem=None):
        self._mem = _mem if _mem is not None else P.ReplayMemory(capacity, state_shape,
                                                               dtype=_ring_dtype(dtype))

    def store(self, t):
        return self._mem.store(t)

    def sample_uniform(self, k, rng):
        return _host_batch(self._mem.sample_uniform(k, rng))

    @property
    def states(self):
        return HostView(self._mem.states)

    @property
    def next_states(self):
        return HostView(self._mem.next_states)

    def __getattr__(self, name):
        return getattr(self._mem, name)


class PrioritizedReplay:
    def __init__(self, capacity, state_shape, config=None, dtype=np.float32):
        self._mem = P.PrioritizedReplay(capacity, state_shape, config, dtype=_ring_dtype(dtype))

    @property
    def tree(self):
        return SumTree(_tree=self._mem.tree)

    @property
    def memory(self):
        return ReplayMemory(None, None, _mem=self._mem.memory)

    def store(self, t):
        return self._mem.store(t)

    def sample(self, k, beta, rng):
        return _host_batch(self._mem.sample(k, beta, rng))

    def update_priorities(self, indices, td_errors):
        self._mem.update_priorities(np.asarray(list(indices) if not hasattr(indices, "__array__")
                                               else indices), np.asarray(td_errors))

    def __getattr__(self, name):
        return getattr(self._mem, name)


def unwrap_memory(m):
    return m._mem if isinstance(m, (ReplayMemory, PrioritizedReplay)) else m
