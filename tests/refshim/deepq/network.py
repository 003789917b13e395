"""deepq.network over the device Network (host views of its tensors)."""

from __future__ import annotations

import numpy as np

import paper_1804_05834_b200 as P

from ._host import HostView, to_np


def _f32(dtype):
    return np.float32    # the device learner computes in float32 (see package doc)


class Tensor:
    def __init__(self, t):
        self._t = t
        self.shape = t.shape

    @property
    def values(self):
        return HostView(self._t.values)

    @values.setter
    def values(self, v):
        HostView(self._t.values)[...] = v

    @property
    def grad(self):
        return HostView(self._t.grad)

    @grad.setter
    def grad(self, v):
        HostView(self._t.grad)[...] = v

    @property
    def size(self):
        return self._t.size

    @property
    def dtype(self):
        return np.dtype(np.float32)


class Params:
    def __init__(self, p):
        self._p = p
        self.name = p.name
        self.weight = Tensor(p.weight)
        self.bias = Tensor(p.bias) if p.bias is not None else None


class _Port:                    # net.x / net.y: values and grad as host views
    def __init__(self, t):
        self._t = t

    @property
    def values(self):
        return to_np(self._t.values)

    @property
    def grad(self):
        return None if self._t.grad is None else to_np(self._t.grad)


class Network:
    def __init__(self, layers, input_shape, dtype=np.float32, _net=None):
        self._net = _net if _net is not None else P.Network(list(layers), input_shape, dtype=_f32(dtype))

    @classmethod
    def _wrap(cls, net):
        return cls(None, None, _net=net)

    def forward(self, x):
        return to_np(self._net.forward(x))

    def backward(self, g):
        return to_np(self._net.backward(g))

    def calculate_gradient(self):
        self._net.calculate_gradient()

    def params(self):
        return [Params(p) for p in self._net.params()]

    def named_tensors(self):
        return [(n, Tensor(t)) for n, t in self._net.named_tensors()]

    @property
    def x(self):
        return _Port(self._net.x)

    @property
    def y(self):
        return _Port(self._net.y)

    def __getattr__(self, name):
        return getattr(self._net, name)


def build_network(spec, input_shape, n_actions, dueling=False, dtype=np.float32):
    if isinstance(spec, list):
        spec = [s if isinstance(s, tuple) else s for s in spec]
    return Network._wrap(P.build_network(spec, input_shape, n_actions, dueling, dtype=_f32(dtype)))


def init_params(net, seed):
    P.init_params(net._net if isinstance(net, Network) else net, seed)


def unwrap(net):
    return net._net if isinstance(net, Network) else net
