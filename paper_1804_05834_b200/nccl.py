"""Minimal NCCL binding (ctypes) for the data-parallel learner's collectives.

The learner's update is one CUDA graph per rank, collectives included, so
the collectives are issued straight on the capturing stream through NCCL's
own C API (NCCL supports stream capture natively); the communicator is set
up once from a unique id broadcast over the ``torch.distributed`` group.
The library is the NCCL that torch ships (nvidia-nccl, 2.28), falling back
to the system one.
"""

from __future__ import annotations

import ctypes as C
import glob
import os

NCCL_INT32, NCCL_INT64, NCCL_FLOAT32, NCCL_FLOAT64 = 2, 4, 7, 8
NCCL_UINT8 = 1
NCCL_SUM, NCCL_MAX = 0, 2

_DTYPES = None


def _find_lib() -> str:
    env = os.environ.get("DQN_B200_NCCL")
    if env:
        return env
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            hits = sorted(glob.glob(os.path.join(base, "lib", "libnccl.so*")))
            if hits:
                return hits[0]
    except ImportError:
        pass
    return "libnccl.so.2"


class _UniqueId(C.Structure):
    _fields_ = [("internal", C.c_byte * 128)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(_find_lib())
        L.ncclGetUniqueId.argtypes = [C.POINTER(_UniqueId)]
        L.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, _UniqueId, C.c_int]
        L.ncclAllReduce.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                                    C.c_void_p, C.c_void_p]
        L.ncclAllGather.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                                    C.c_void_p]
        L.ncclCommDestroy.argtypes = [C.c_void_p]
        L.ncclGetErrorString.argtypes = [C.c_int]
        L.ncclGetErrorString.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().ncclGetErrorString(rc).decode(errors="replace")
        raise RuntimeError(f"{what}: NCCL error {rc} ({msg})")


def _torch_dtype_code(t) -> int:
    import torch
    return {torch.float32: NCCL_FLOAT32, torch.float64: NCCL_FLOAT64, torch.int32: NCCL_INT32,
            torch.int64: NCCL_INT64, torch.uint8: NCCL_UINT8}[t.dtype]


class Communicator:
    """One NCCL communicator over a torch.distributed group (rank 0 makes
    the unique id and broadcasts it as an object)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = _UniqueId()
        if self.rank == 0:
            _check(lib().ncclGetUniqueId(C.byref(uid)), "ncclGetUniqueId")
        box = [bytes(uid.internal) if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        C.memmove(uid.internal, box[0], 128)
        self.comm = C.c_void_p()
        _check(lib().ncclCommInitRank(C.byref(self.comm), self.world, uid, self.rank),
               "ncclCommInitRank")

    def all_reduce(self, t, op: int, stream: int, out=None) -> None:
        """In place (or into ``out``) on the given raw stream."""
        dst = t if out is None else out
        _check(lib().ncclAllReduce(t.data_ptr(), dst.data_ptr(), t.numel(), _torch_dtype_code(t),
                                   op, self.comm, stream), "ncclAllReduce")

    def all_gather(self, send, recv, stream: int) -> None:
        """``recv`` holds world x send.numel() elements in rank order."""
        _check(lib().ncclAllGather(send.data_ptr(), recv.data_ptr(), send.numel(),
                                   _torch_dtype_code(send), self.comm, stream), "ncclAllGather")

    def close(self) -> None:
        if self.comm:
            lib().ncclCommDestroy(self.comm)
            self.comm = C.c_void_p()
