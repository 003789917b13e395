"""deepq.optim over the device optimizer."""

from __future__ import annotations

import paper_1804_05834_b200 as P

from ._host import HostView
from .network import unwrap


class RmsProp:
    def __init__(self, net, learning_rate=0.000625, decay=0.95, epsilon=1e-6):
        self._opt = P.RmsProp(unwrap(net), learning_rate, decay, epsilon)

    @property
    def acc(self):
        return {n: HostView(t) for n, t in self._opt.acc.items()}

    def step(self):
        self._opt.step()

    def __getattr__(self, name):
        return getattr(self._opt, name)


def clip_gradients(net, max_norm):
    return P.clip_gradients(unwrap(net), max_norm)


def sync_target(online, target):
    P.sync_target(unwrap(online), unwrap(target))
