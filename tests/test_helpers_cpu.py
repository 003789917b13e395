"""The kink-resolution helper the one-step parity tests use
(tests/helpers.follow_device_relu_kinks), on the oracle alone."""

import numpy as np
import pytest

from oracle import deepq_oracle as O
from tests.helpers import follow_device_relu_kinks


def _net():
    net = O.QNet(O.DESK_TRUNK, (24, 24, 4), 3, False)
    net.init(4)
    x = np.random.default_rng(0).random((2, 24, 24, 4)).astype(np.float32)
    return net, x


def _unit_outputs(net):
    return [np.maximum(z, 0) for (z, aux), (kind, _, _) in zip(net._acts, net.ops) if kind == "relu"]


def test_agreeing_masks_change_nothing():
    net, x = _net()
    net.forward(x)
    dev = _unit_outputs(net)
    g = np.ones((2, 3), np.float32)
    ref = net.backward(g).copy()
    net.forward(x)
    assert follow_device_relu_kinks(net, dev) == []
    assert np.array_equal(net.backward(g), ref)


def test_flip_at_the_kink_is_followed_and_far_flip_raises():
    net, x = _net()
    net.forward(x)
    dev = _unit_outputs(net)
    li = [i for i, op in enumerate(net.ops) if op[0] == "relu"][1]
    z = net._acts[li][0]
    j = np.unravel_index(np.argmin(np.abs(z)), z.shape)
    small = dict(enumerate(dev))
    d1 = small[1].copy()
    d1[j] = 0.0 if z[j] > 0 else 1e-30          # the device resolved the kink the other way
    flips = follow_device_relu_kinks(net, [dev[0], d1] + dev[2:], tol=1.0)
    net.backward(np.ones((2, 3), np.float32))
    assert flips and flips[0][:2] == (li, 1)
    # a disagreement far from the kink is a real error
    net.forward(x)
    k = np.unravel_index(np.argmax(np.abs(z)), z.shape)
    d2 = dev[1].copy()
    d2[k] = 0.0 if z[k] > 0 else 1.0
    follow_device_relu_kinks(net, [dev[0], d2] + dev[2:], tol=1e-5)
    with pytest.raises(AssertionError):
        net.backward(np.ones((2, 3), np.float32))
