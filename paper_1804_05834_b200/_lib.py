"""ctypes binding of libdqn_b200.so (include/dqn_b200.h).

There is no CPU fallback: importing this module loads the in-tree CUDA
library or raises ImportError, and ``require_cuda()`` raises when no GPU is
visible.  The structs mirror ``dqn_layer_desc`` / ``dqn_net_desc`` /
``dqn_binding`` field for field.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigError, DeepQError, GeometryError, NonFiniteError

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DQN_B200_LIB", _HERE / "libdqn_b200.so"))

if not LIB_PATH.exists():
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (the CUDA library is required; there is no CPU fallback)")
lib = C.CDLL(str(LIB_PATH))

# status codes / flags (dqn_b200.h)
OK, ERR_INVALID_ARG, ERR_GEOMETRY, ERR_INDEX, ERR_EMPTY, ERR_ZERO_TOTAL, ERR_NONFINITE, \
    ERR_CUDA, ERR_UNSUPPORTED = range(9)
NET_HINT_SIDE = 1          # dqn_net_desc.hints (include/dqn_b200.h)
FLAG_INDEX, FLAG_ZERO_TOTAL, FLAG_NONFINITE_GRAD, FLAG_NONFINITE_OUT, FLAG_BAD_PRIORITY = \
    0x1, 0x2, 0x4, 0x8, 0x10
TD_DOUBLE, TD_HUBER, TD_REWARD_CLIP, TD_HEAD_LAST_CTA = 0x1, 0x2, 0x4, 0x8
LAYER_CONV, LAYER_LINEAR, LAYER_DUELING = 0, 1, 2
MAX_LAYERS = 8

vp, i32, i64, u64, f32, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double


class LayerDesc(C.Structure):
    _fields_ = [("kind", i32), ("relu", i32), ("in_h", i32), ("in_w", i32), ("in_c", i32),
                ("out_h", i32), ("out_w", i32), ("out_c", i32), ("fh", i32), ("fw", i32),
                ("sh", i32), ("sw", i32), ("w_off", i64), ("b_off", i64), ("w2_off", i64),
                ("b2_off", i64)]


class NetDesc(C.Structure):
    _fields_ = [("n_layers", i32), ("input_u8", i32), ("algo", i32), ("hints", i32),
                ("layer", LayerDesc * MAX_LAYERS)]


class Binding(C.Structure):
    _fields_ = [("batch", i32), ("pad_", i32), ("x", vp), ("act", vp * MAX_LAYERS),
                ("dact", vp * MAX_LAYERS), ("dx", vp), ("scratch", vp),
                ("scratch_floats", i64)]


_SIGS = {
    "dqn_last_error": ([], C.c_char_p),
    "dqn_abi_version": ([], C.c_int),
    "dqn_has_tcgen05": ([], C.c_int),
    "dqn_launch_count": ([], i64),
    "dqn_ring_fill_hash": ([vp, vp, i64, i64, i64, u64], C.c_int),
    "dqn_ring_gather": ([vp, vp, vp, i64, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp], C.c_int),
    "dqn_tree_sample": ([vp, vp, i32, vp, vp, i32, vp, vp, vp, vp, vp], C.c_int),
    "dqn_tree_find": ([vp, vp, i32, vp, i64, vp, vp], C.c_int),
    "dqn_tree_update": ([vp, vp, i32, vp, vp, vp, i32, f64, f64, vp, vp], C.c_int),
    "dqn_tree_store": ([vp, vp, i32, i64, i64, i64, vp, f64], C.c_int),
    "dqn_tree_set": ([vp, vp, i32, i64, vp, vp, i32, vp], C.c_int),
    "dqn_tree_rebuild": ([vp, vp, i32], C.c_int),
    "dqn_net_scratch_floats": ([C.POINTER(NetDesc), i32], i64),
    "dqn_head_td_work_bytes": ([i32, i32], i64),
    "dqn_head_td": ([vp, C.POINTER(NetDesc), vp, vp, C.POINTER(Binding), C.POINTER(Binding),
                     C.POINTER(NetDesc), vp, C.POINTER(Binding), vp, vp, vp, vp, f64, i32,
                     vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "dqn_net_forward": ([vp, C.POINTER(NetDesc), vp, C.POINTER(Binding), vp], C.c_int),
    "dqn_net_backward": ([vp, C.POINTER(NetDesc), vp, C.POINTER(Binding), vp], C.c_int),
    "dqn_net_wgrad": ([vp, C.POINTER(NetDesc), vp, C.POINTER(Binding)], C.c_int),
    "dqn_net_layer": ([vp, C.POINTER(NetDesc), vp, vp, C.POINTER(Binding), i32, i32, vp], C.c_int),
    "dqn_td_loss": ([vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, f64, i32, vp, vp, vp, vp, vp],
                    C.c_int),
    "dqn_rmsprop_step": ([vp, vp, vp, vp, i64, f32, f32, f32, f32, vp], C.c_int),
    "dqn_rmsprop_apply": ([vp, vp, vp, vp, i64, f32, f32, f32, f32, vp, vp], C.c_int),
    "dqn_frame_gather": ([vp, vp, i64, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp],
                         C.c_int),
    "dqn_frame_sample_gather": ([vp, vp, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, i64, vp,
                                 C.c_int, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "dqn_clip_gradients": ([vp, vp, i64, f64, vp], C.c_int),
    "dqn_sync_target": ([vp, vp, vp, i64], C.c_int),
    "dqn_dp_shard_info": ([vp, vp, vp, vp, vp], C.c_int),
    "dqn_dp_route": ([vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp],
                     C.c_int),
    "dqn_dp_descend": ([vp, vp, C.c_int, vp, vp, C.c_int, C.c_int, vp], C.c_int),
    "dqn_dp_weights": ([vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp], C.c_int),
    "dqn_dp_gather": ([vp, vp, vp, vp, C.c_int, C.c_int, i64, vp, vp, vp, vp, vp, vp, C.c_int, vp,
                       vp, vp], C.c_int),
    "dqn_dp_owned": ([vp, vp, vp, vp, C.c_int, C.c_int, C.c_double, vp, vp, vp, vp, vp, vp],
                     C.c_int),
    "dqn_dp_report": ([vp, vp, vp, vp, vp, C.c_int, vp, vp, vp], C.c_int),
    "dqn_tree_update_n": ([vp, vp, C.c_int, vp, vp, vp, C.c_int, vp, C.c_double, C.c_double, vp,
                           vp], C.c_int),
    "dqn_dev_alloc": ([i64, C.POINTER(C.c_void_p)], C.c_int),
    "dqn_dev_free": ([vp], C.c_int),
    "dqn_ipc_handle": ([vp, vp], C.c_int),
    "dqn_ipc_open": ([vp, C.POINTER(C.c_void_p)], C.c_int),
    "dqn_ipc_close": ([vp], C.c_int),
    "dqn_ring_store": ([vp, vp, vp, i64, vp, vp, vp, i64, i64, C.c_int, vp, vp, vp, vp, vp, vp,
                        i64], C.c_int),
    "dqn_sample_gather": ([vp, vp, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, i64, vp,
                           vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "dqn_graph_instantiate": ([vp, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "dqn_graph_launch": ([vp, vp], C.c_int),
    "dqn_graph_destroy": ([vp], C.c_int),
    "dqn_preprocess_frames": ([vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, i64,
                               i64], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)          # AttributeError here = header/library mismatch
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTED = tuple(_SIGS)


class CudaError(DeepQError):
    """A CUDA runtime error reported by libdqn_b200."""


_STATUS_EXC = {
    ERR_INVALID_ARG: ValueError, ERR_GEOMETRY: GeometryError, ERR_INDEX: IndexError,
    ERR_EMPTY: ValueError, ERR_ZERO_TOTAL: ValueError, ERR_NONFINITE: NonFiniteError,
    ERR_CUDA: CudaError, ERR_UNSUPPORTED: ConfigError,
}


def call(name: str, *args) -> None:
    """Call an int-returning entry point; map a non-zero status to the
    reference's exception type."""
    st = getattr(lib, name)(*args)
    if st != OK:
        raise_status(st, name)


def raise_status(st: int, name: str) -> None:
    msg = lib.dqn_last_error().decode(errors="replace")
    raise _STATUS_EXC.get(st, DeepQError)(f"{name}: {msg}")


def require_cuda():
    """The product path runs only on the GPU; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1804_05834_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def stream_ptr() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
