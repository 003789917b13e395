"""Device frame pipeline: the reference's
``preprocess_frame`` / ``Preprocessor`` (envs.py:289-357) for raw uint8
emulator frames, computed by ``dqn_preprocess_frames`` on the GPU and
bit-identical to the host restatement in envs.py (and so to the reference).

``preprocess_frames(frames, size)`` maps a batch [N, H, W] / [N, H, W, 1|3]
of uint8 frames (host or device) to float32 [N, h, w] in HBM.
``DevicePreprocessor`` keeps the (h, w, stack) frame stack in HBM: each new
frame is written straight into the stack's last channel by the kernel
(pixel stride = stack depth) after a one-channel shift, so a batch of
emulators never round-trips preprocessed frames through the host.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _as_frames(frames):
    torch = _lib.require_cuda()
    t = frames if isinstance(frames, torch.Tensor) else torch.as_tensor(np.asarray(frames))
    if t.dtype != torch.uint8:
        raise ValueError(f"device preprocessing takes uint8 frames, got {t.dtype}")
    if t.dim() == 3:                      # [N, H, W]
        t = t.unsqueeze(-1)
    if t.dim() != 4 or t.shape[-1] not in (1, 3):
        raise ValueError(f"expected [N, H, W] or [N, H, W, 1|3] frames, got {tuple(t.shape)}")
    return t.to("cuda").contiguous()


def preprocess_into(frames, size: tuple[int, int], out, frame_stride: int, pix_stride: int) -> None:
    """Enqueue ``dqn_preprocess_frames`` writing frame f, pixel p to
    ``out[f * frame_stride + p * pix_stride]`` (``out`` a float32 CUDA
    tensor or view start)."""
    t = _as_frames(frames)
    n, h, w, c = (int(s) for s in t.shape)
    _lib.call("dqn_preprocess_frames", _lib.stream_ptr(), t.data_ptr(), n, h, w, c,
              int(size[0]), int(size[1]), out.data_ptr(), int(frame_stride), int(pix_stride))


def preprocess_frames(frames, size: tuple[int, int] = (84, 84)):
    """Batch ``preprocess_frame``: uint8 [N, H, W(, C)] -> float32 [N, h, w] on the GPU."""
    torch = _lib.require_cuda()
    t = _as_frames(frames)
    out = torch.empty((t.shape[0], int(size[0]), int(size[1])), dtype=torch.float32, device="cuda")
    preprocess_into(t, size, out, int(size[0]) * int(size[1]), 1)
    return out


class DevicePreprocessor:
    """Preprocessor (envs.py:314-357) with the frame stack in HBM: the first
    frame after reset fills every channel, later frames shift FIFO with the
    newest in the last channel.  ``reset`` / ``push`` return the (h, w,
    stack) float32 CUDA tensor (a view of the internal stack: copy it to keep
    it across the next push)."""

    def __init__(self, size: tuple[int, int] = (84, 84), stack: int = 4):
        torch = _lib.require_cuda()
        if stack < 1:
            raise ValueError(f"stack depth must be >= 1, got {stack}")
        self.size = (int(size[0]), int(size[1]))
        self.stack = int(stack)
        self.state = torch.zeros(self.size + (self.stack,), dtype=torch.float32, device="cuda")
        self._tmp = torch.empty_like(self.state)
        self._live = False

    @property
    def output_shape(self) -> tuple[int, int, int]:
        return self.size + (self.stack,)

    def _write_last(self, frame) -> None:
        # one frame [H, W] or [H, W, C], written into the last channel
        preprocess_into(_one(frame), self.size, self.state[..., self.stack - 1], 0, self.stack)

    def reset(self, frame):
        self._write_last(frame)
        if self.stack > 1:
            self.state[..., :-1] = self.state[..., -1:]
        self._live = True
        return self.state

    def push(self, frame):
        if not self._live:
            return self.reset(frame)
        if self.stack > 1:
            self._tmp[..., :-1] = self.state[..., 1:]
            self.state[..., :-1] = self._tmp[..., :-1]
        self._write_last(frame)
        return self.state


def _one(frame):
    """A single frame [H, W] or [H, W, C] as a batch of one."""
    a = frame
    torch = _lib.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.unsqueeze(0)
    return np.asarray(a)[None]
