"""Host views for running the reference's own unit tests (written against
numpy arrays) unchanged on the device package: parameter / gradient /
accumulator tensors live in HBM as torch CUDA tensors, the reference tests
read and write them as numpy arrays.  ``HostView`` is that bridge: reads copy
the device tensor to the host, writes go back to the device."""

from __future__ import annotations

import numpy as np


def to_np(x):
    """torch tensor (any device) -> numpy; anything else unchanged."""
    if hasattr(x, "detach") and hasattr(x, "cpu"):
        return x.detach().cpu().numpy()
    return x


class HostView:
    """A numpy-like live view of a device tensor (read = copy to host,
    write = copy back)."""

    __array_priority__ = 100

    def __init__(self, t):
        object.__setattr__(self, "_t", t)

    def __array__(self, dtype=None, copy=None):
        a = self._t.detach().cpu().numpy()
        return a.astype(dtype) if dtype is not None else a

    def _np(self):
        return self.__array__()

    # -- numpy surface ----------------------------------------------------
    @property
    def shape(self):
        return tuple(self._t.shape)

    @property
    def dtype(self):
        return self._np().dtype

    @property
    def size(self):
        return int(self._t.numel())

    @property
    def ndim(self):
        return self._t.dim()

    def copy(self):
        return self._np().copy()

    def __getitem__(self, idx):
        return self._np()[idx]

    def __setitem__(self, idx, value):
        import torch
        a = self._np()
        a[idx] = np.asarray(value)
        self._t.copy_(torch.as_tensor(a, device=self._t.device))

    def __getattr__(self, name):          # max, sum, astype, ravel, ...
        return getattr(self._np(), name)

    def __len__(self):
        return len(self._t)

    def __iter__(self):
        return iter(self._np())

    def __float__(self):
        return float(self._np())

    def __repr__(self):
        return f"HostView({self._np()!r})"

    def _inplace(self, other, op):
        self[...] = op(self._np(), np.asarray(other))
        return self

    def __iadd__(self, o):
        return self._inplace(o, np.add)

    def __isub__(self, o):
        return self._inplace(o, np.subtract)

    def __imul__(self, o):
        return self._inplace(o, np.multiply)


def _binop(name):
    def f(self, other):
        return getattr(self._np(), name)(np.asarray(other) if isinstance(other, HostView) else other)
    return f


for _n in ("__add__", "__radd__", "__sub__", "__rsub__", "__mul__", "__rmul__", "__truediv__",
           "__rtruediv__", "__pow__", "__eq__", "__ne__", "__lt__", "__le__", "__gt__", "__ge__",
           "__and__", "__or__", "__matmul__"):
    setattr(HostView, _n, _binop(_n))
HostView.__neg__ = lambda self: -self._np()
HostView.__abs__ = lambda self: np.abs(self._np())
HostView.__hash__ = None
