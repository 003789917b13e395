"""RMSprop, gradient clipping and target sync on the GPU (deepq/optim.py:12-89).

All three run over the network's flat parameter buffers in one launch chain:
``dqn_rmsprop_step`` (finite scan, then the fp32 update in numpy's operation
order -- bit-exact with the reference given identical gradients),
``dqn_clip_gradients`` (fp64 global norm) and ``dqn_sync_target`` (bitwise
copy).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import GeometryError, NonFiniteError
from .network import Network


class RmsProp:
    """Plain RMSprop (optim.py:12-58); accumulator state lives in HBM."""

    def __init__(self, net: Network, learning_rate: float = 0.000625, decay: float = 0.95,
                 epsilon: float = 1e-6):
        torch = _lib.require_cuda()
        if not 0.0 < decay < 1.0:
            raise ValueError(f"decay must be in (0, 1), got {decay}")
        if epsilon <= 0.0:
            raise ValueError(f"epsilon must be positive, got {epsilon}")
        if learning_rate < 0.0:
            raise ValueError(f"learning rate must be >= 0, got {learning_rate}")
        self.learning_rate = float(learning_rate)
        self.decay = float(decay)
        self.epsilon = float(epsilon)
        self.net = net
        self._tensors = net.named_tensors()
        self.flat_acc = torch.zeros_like(net.flat_values)
        self.acc = {}
        for (name, t) in self._tensors:
            off = t.values.data_ptr() - net.flat_values.data_ptr()
            o = off // 4
            self.acc[name] = self.flat_acc[o:o + t.values.numel()].view(t.shape)
        self._flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        # numpy weak-scalar promotion (NEP 50): the python floats become float32
        self._lr32 = np.float32(self.learning_rate)
        self._rho32 = np.float32(self.decay)
        self._omr32 = np.float32(1.0 - self.decay)
        self._eps32 = np.float32(self.epsilon)

    def enqueue_step(self, flags=None) -> None:
        """Device-side step (no sync): skip + flag on a non-finite gradient."""
        net = self.net
        _lib.call("dqn_rmsprop_step", _lib.stream_ptr(), net.flat_values.data_ptr(),
                  net.flat_grads.data_ptr(), self.flat_acc.data_ptr(), net.n_flat,
                  float(self._lr32), float(self._rho32), float(self._omr32), float(self._eps32),
                  (flags if flags is not None else self._flags).data_ptr())

    def enqueue_apply(self, flags, flag_out=None) -> None:
        """Device-side step without the finiteness scan: for gradients whose
        producers flagged non-finite values into ``flags`` as they wrote them
        (the learner's wgrad / fused-head launches); skipped on any flag.
        ``flag_out`` (pinned host tensor) receives the flag word from the
        kernel itself (the learner's completion signal)."""
        net = self.net
        _lib.call("dqn_rmsprop_apply", _lib.stream_ptr(), net.flat_values.data_ptr(),
                  net.flat_grads.data_ptr(), self.flat_acc.data_ptr(), net.n_flat,
                  float(self._lr32), float(self._rho32), float(self._omr32), float(self._eps32),
                  flags.data_ptr(), None if flag_out is None else flag_out.data_ptr())

    def step(self) -> None:
        """Apply one update from the accumulated gradients, then zero them."""
        self.enqueue_step()
        f = int(self._flags.item())
        if f & _lib.FLAG_NONFINITE_GRAD:
            self._flags.zero_()
            import torch
            bad = [n for n, t in self._tensors if not bool(torch.isfinite(t.grad).all())]
            raise NonFiniteError(f"non-finite gradient in {bad[0] if bad else '?'}; step aborted")

    def state_arrays(self):
        return [(name, self.acc[name]) for name, _ in self._tensors]

    def load_state(self, arrays: dict) -> None:
        import torch
        for name, _ in self._tensors:
            src = arrays[name]
            src = src if isinstance(src, torch.Tensor) else torch.as_tensor(np.asarray(src))
            if tuple(src.shape) != tuple(self.acc[name].shape):
                raise GeometryError(f"optimizer state {name}: shape {tuple(src.shape)} != "
                                    f"{tuple(self.acc[name].shape)}")
            self.acc[name].copy_(src.to(device="cuda", dtype=torch.float32))


def clip_gradients(net: Network, max_norm: float) -> float:
    """Scale all grads so the global L2 norm is <= max_norm (optim.py:61-75).
    Returns the pre-clip norm."""
    torch = _lib.require_cuda()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("dqn_clip_gradients", _lib.stream_ptr(), net.flat_grads.data_ptr(), net.n_flat,
              float(max_norm), out.data_ptr())
    return float(out.item())


def sync_target(net: Network, target: Network) -> None:
    """Bit-exact copy of every parameter of ``net`` into ``target``."""
    src = dict(net.named_tensors())
    dst = dict(target.named_tensors())
    if set(src) != set(dst):
        raise GeometryError(f"parameter registries differ: {sorted(set(src) ^ set(dst))}")
    for name, t in dst.items():
        if src[name].shape != t.shape:
            raise GeometryError(f"{name}: shape {src[name].shape} != {t.shape}")
    if net.n_flat != target.n_flat:
        raise GeometryError("flat layouts differ")
    _lib.call("dqn_sync_target", _lib.stream_ptr(), target.flat_values.data_ptr(),
              net.flat_values.data_ptr(), net.n_flat)
