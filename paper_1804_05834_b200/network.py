"""Q-network on the GPU: the reference's layer pipeline and parameter registry
(deepq/network.py:45-205, deepq/layers.py:27-344) driving libdqn_b200.

The registry keeps the reference's names and order (``conv1.weight``,
``conv1.bias``, ..., ``duel.value.weight``, ...; network.py:74-84) and shapes
(conv filters (fh, fw, cin, cout), linear (in, out)).  Storage is one flat
fp32 buffer per network (values, grads; each tensor starts on a 128-byte
boundary) so RMSprop and the target sync are single passes over HBM.  ReLU
layers are fused into the producing layer's epilogue (forward) and into the
consumer's dgrad (backward mask); they still appear in ``layers`` with the
reference names for introspection.

Only float32 networks exist on this path; ``dtype=float64`` raises
ConfigError (no CPU fallback).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, GeometryError, NonFiniteError, PhaseOrderError
from .tensor import Params, Tensor


@dataclass(frozen=True)
class LayerSpec:
    """Declarative layer description (layers.py:27-55)."""

    kind: str  # convolution | linear | relu | dueling-head
    geometry: dict = field(default_factory=dict)

    @staticmethod
    def convolution(filters: int, size: int, stride: int) -> "LayerSpec":
        return LayerSpec("convolution", {"filters": filters, "filter_h": size, "filter_w": size,
                                         "stride_h": stride, "stride_w": stride})

    @staticmethod
    def linear(units: int) -> "LayerSpec":
        return LayerSpec("linear", {"units": units})

    @staticmethod
    def relu() -> "LayerSpec":
        return LayerSpec("relu", {})

    @staticmethod
    def dueling_head(n_actions: int) -> "LayerSpec":
        return LayerSpec("dueling-head", {"n_actions": n_actions})


ARCHITECTURES: dict[str, list[LayerSpec]] = {
    "atari": [LayerSpec.convolution(32, 8, 4), LayerSpec.relu(),
              LayerSpec.convolution(64, 4, 2), LayerSpec.relu(),
              LayerSpec.convolution(64, 3, 1), LayerSpec.relu(),
              LayerSpec.linear(512), LayerSpec.relu()],
    "desk": [LayerSpec.convolution(16, 6, 2), LayerSpec.relu(),
             LayerSpec.convolution(32, 3, 1), LayerSpec.relu(),
             LayerSpec.linear(128), LayerSpec.relu()],
}

_IDLE, _FORWARD, _BACKWARD, _GRAD = range(4)
_ALIGN = 32          # floats (128 B) per tensor start


def trunk_layers(arch: str) -> list[LayerSpec]:
    try:
        return list(ARCHITECTURES[arch])
    except KeyError:
        raise ValueError(f"unknown architecture {arch!r}; choose from {sorted(ARCHITECTURES)}") from None


class LayerView:
    """Introspection record for one reference layer (name, kind, output shape)."""

    def __init__(self, name, kind, out_shape, unit):
        self.name, self.kind, self.out_shape, self.unit = name, kind, out_shape, unit
        self.in_features = None
        self.w = None

    def __repr__(self):
        return f"LayerView({self.name!r}, {self.kind}, out={self.out_shape})"


class _Bind:
    """Per-batch activation buffers + the C dqn_binding struct."""

    def __init__(self, net: "Network", batch: int, parent: "_Bind | None" = None,
                 own_scratch: bool = False):
        torch = _lib.require_cuda()
        self.batch = batch
        self.struct = _lib.Binding()
        self.struct.batch = batch
        if parent is None:
            self.act, self.dact = [], []
            for u in net._units:
                n = batch * int(np.prod(u["out_shape"]))
                self.act.append(torch.empty(n, dtype=torch.float32, device="cuda"))
                self.dact.append(torch.zeros(n, dtype=torch.float32, device="cuda"))
            self.dx = torch.zeros((batch,) + net.input_shape, dtype=torch.float32, device="cuda")
            sf = int(_lib.lib.dqn_net_scratch_floats(C.byref(net._desc), batch))
            if sf < 0:
                raise GeometryError("network geometry rejected by libdqn_b200")
            # zeroed: its tail is the split-K tile-counter table (self-resetting)
            self.scratch = torch.zeros(max(sf, 1), dtype=torch.float32, device="cuda")
            self.scratch_floats = sf
        else:                       # prefix view: first `batch` rows of a larger binding
            self.act, self.dact, self.dx = parent.act, parent.dact, parent.dx
            self.scratch, self.scratch_floats = parent.scratch, parent.scratch_floats
            sf = int(_lib.lib.dqn_net_scratch_floats(C.byref(net._desc), batch))
            if sf > self.scratch_floats or own_scratch:
                # own scratch: kernels of this view may run concurrently with
                # the parent's on another stream
                sf = max(sf, self.scratch_floats)
                self.scratch = torch.zeros(sf, dtype=torch.float32, device="cuda")
                self.scratch_floats = sf
        for i in range(len(net._units)):
            self.struct.act[i] = self.act[i].data_ptr()
            self.struct.dact[i] = self.dact[i].data_ptr()
        self.struct.dx = self.dx.data_ptr()
        self.struct.scratch = self.scratch.data_ptr()
        self.struct.scratch_floats = self.scratch_floats
        self.x = None


class Network:
    """Phase-checked layer pipeline (network.py:45-138) over device buffers."""

    def __init__(self, specs: list[tuple[str, LayerSpec]], input_shape: tuple[int, ...],
                 dtype=np.float32):
        torch = _lib.require_cuda()
        self.dtype = np.dtype(dtype)
        if self.dtype != np.float32:
            raise ConfigError("the B200 learner computes in float32 only (float64 nets are "
                              "CPU-reference only)")
        self.input_shape = tuple(int(s) for s in input_shape)
        if len(self.input_shape) not in (1, 3):
            raise GeometryError(f"input must be (H, W, C) or (features,), got {self.input_shape}")
        units, views, reg = [], [], []
        shape = self.input_shape if len(self.input_shape) == 3 else (1, 1, self.input_shape[0])
        spatial = len(self.input_shape) == 3
        for name, spec in specs:
            g = spec.geometry
            if spec.kind == "convolution":
                if not spatial:
                    raise GeometryError(f"{name}: expected 4-d input")
                h, w, c = shape
                fh, fw, sh, sw, co = (int(g["filter_h"]), int(g["filter_w"]), int(g["stride_h"]),
                                      int(g["stride_w"]), int(g["filters"]))
                if min(fh, fw, sh, sw, co) < 1:
                    raise GeometryError(f"{name}: filter/stride extents must be positive")
                if h < fh or w < fw:
                    raise GeometryError(f"{name}: {fh}x{fw} filter does not fit {h}x{w} input")
                if (h - fh) % sh or (w - fw) % sw:
                    raise GeometryError(f"{name}: stride ({sh},{sw}) does not tile {h}x{w} input "
                                        f"with {fh}x{fw} filter (valid padding)")
                oh, ow = (h - fh) // sh + 1, (w - fw) // sw + 1
                u = dict(kind=_lib.LAYER_CONV, name=name, in_shape=shape, out_shape=(oh, ow, co),
                         geo=(fh, fw, sh, sw), relu=0,
                         tensors=[(name + ".weight", (fh, fw, c, co)), (name + ".bias", (co,))])
                shape = (oh, ow, co)
            elif spec.kind == "linear":
                feat = int(np.prod(shape))
                n = int(g["units"])
                u = dict(kind=_lib.LAYER_LINEAR, name=name, in_shape=(1, 1, feat), out_shape=(n,),
                         geo=(1, 1, 1, 1), relu=0,
                         tensors=[(name + ".weight", (feat, n)), (name + ".bias", (n,))])
                shape = (1, 1, n)
                spatial = False
            elif spec.kind == "dueling-head":
                feat = int(np.prod(shape))
                na = int(g["n_actions"])
                if na < 1:
                    raise GeometryError(f"{name}: n_actions must be >= 1, got {na}")
                u = dict(kind=_lib.LAYER_DUELING, name=name, in_shape=(1, 1, feat),
                         out_shape=(na,), geo=(1, 1, 1, 1), relu=0,
                         tensors=[(name + ".value.weight", (feat, 1)), (name + ".value.bias", (1,)),
                                  (name + ".advantage.weight", (feat, na)),
                                  (name + ".advantage.bias", (na,))])
                shape = (1, 1, na)
                spatial = False
            elif spec.kind == "relu":
                if not units:
                    raise ConfigError(f"{name}: a leading ReLU on the raw input is not supported")
                units[-1]["relu"] = 1             # fused (relu after relu is idempotent)
                views.append(LayerView(name, "relu", views[-1].out_shape, len(units) - 1))
                continue
            else:
                raise ValueError(f"unknown layer kind {spec.kind!r}")
            units.append(u)
            views.append(LayerView(name, spec.kind, u["out_shape"], len(units) - 1))
            views[-1].in_features = int(np.prod(u["in_shape"]))
        if not units:
            raise GeometryError("network has no parameterised layer")
        if len(units) > _lib.MAX_LAYERS:
            raise ConfigError(f"at most {_lib.MAX_LAYERS} parameterised layers")
        # flat registry
        off = 0
        for u in units:
            u["offs"] = []
            for tname, tshape in u["tensors"]:
                u["offs"].append(off)
                reg.append((tname, tshape, off))
                off += (int(np.prod(tshape)) + _ALIGN - 1) // _ALIGN * _ALIGN
        self.n_flat = off
        self.flat_values = torch.zeros(off, dtype=torch.float32, device="cuda")
        self.flat_grads = torch.zeros(off, dtype=torch.float32, device="cuda")
        self._registry = []
        for tname, tshape, o in reg:
            n = int(np.prod(tshape))
            self._registry.append((tname, Tensor(self.flat_values[o:o + n].view(tshape),
                                                 self.flat_grads[o:o + n].view(tshape))))
        tmap = dict(self._registry)
        self._params = []
        for u in units:
            names = [t[0] for t in u["tensors"]]
            if u["kind"] == _lib.LAYER_DUELING:
                ps = [Params(u["name"] + ".value", tmap[names[0]], tmap[names[1]]),
                      Params(u["name"] + ".advantage", tmap[names[2]], tmap[names[3]])]
            else:
                ps = [Params(u["name"], tmap[names[0]], tmap[names[1]])]
            u["params"] = ps
            self._params.extend(ps)
        for v in views:
            if v.kind != "relu":
                v.w = units[v.unit]["params"][0]
        self._units = units
        self.layers = views
        self._desc = self._make_desc(input_u8=False)
        self._desc_u8 = self._make_desc(input_u8=True)
        self.output_shape = tuple(units[-1]["out_shape"])
        self._phase = _IDLE
        self._binds: dict[int, _Bind] = {}
        self._views: dict[tuple[int, int], _Bind] = {}
        self._cur: _Bind | None = None
        self._flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.need_input_grad = True

    def _make_desc(self, input_u8: bool):
        d = _lib.NetDesc()
        d.n_layers = len(self._units)
        d.input_u8 = 1 if input_u8 else 0
        # DQN_B200_ALGO=simt forces the generic SIMT kernels (A/B diagnostics)
        d.algo = 1 if os.environ.get("DQN_B200_ALGO", "") == "simt" else 0
        for i, u in enumerate(self._units):
            L = d.layer[i]
            L.kind, L.relu = u["kind"], u["relu"]
            L.in_h, L.in_w, L.in_c = u["in_shape"]
            os_ = u["out_shape"]
            if len(os_) == 3:
                L.out_h, L.out_w, L.out_c = os_
            else:
                L.out_h, L.out_w, L.out_c = 1, 1, os_[0]
            L.fh, L.fw, L.sh, L.sw = u["geo"]
            offs = u["offs"]
            L.w_off, L.b_off = offs[0], offs[1]
            if u["kind"] == _lib.LAYER_DUELING:
                L.w2_off, L.b2_off = offs[2], offs[3]
        return d

    # -- registry -----------------------------------------------------------
    def params(self) -> list[Params]:
        return list(self._params)

    def named_tensors(self) -> list[tuple[str, Tensor]]:
        return list(self._registry)

    def zero_grads(self) -> None:
        self.flat_grads.zero_()

    def layer_output_shapes(self) -> list[tuple[int, ...]]:
        return [tuple(v.out_shape) for v in self.layers]

    # -- bindings -------------------------------------------------------------
    def binding(self, batch: int) -> _Bind:
        b = self._binds.get(batch)
        if b is None:
            b = _Bind(self, batch)
            self._binds[batch] = b
        return b

    def prefix_binding(self, parent: _Bind, batch: int, own_scratch: bool = False) -> _Bind:
        key = (id(parent), batch, own_scratch)
        v = self._views.get(key)
        if v is None:
            v = _Bind(self, batch, parent=parent, own_scratch=own_scratch)
            self._views[key] = v
        return v

    def layer_into(self, bind: _Bind, layer: int, phase: int, flags=None, desc=None) -> None:
        """One phase (0 fwd, 1 bwd to the layer's input, 2 wgrad) of one layer;
        ``flags`` (default: the network's) receives non-finite outputs and,
        for wgrad, non-finite gradients as they are written.  ``desc``: a
        copy of this network's descriptor with launch hints (``hinted``)."""
        _lib.call("dqn_net_layer", _lib.stream_ptr(), C.byref(desc or self.desc_for(bind.x)),
                  self.flat_values.data_ptr(), self.flat_grads.data_ptr(), C.byref(bind.struct),
                  layer, phase, (self._flags if flags is None else flags).data_ptr())

    def desc_for(self, x):
        import torch
        return self._desc_u8 if x.dtype == torch.uint8 else self._desc

    def hinted(self, x, hints: int):
        """A copy of the descriptor for inputs like ``x`` with launch hints
        (``_lib.NET_HINT_SIDE``: this forward runs beside a critical one)."""
        d = _lib.NetDesc.from_buffer_copy(self.desc_for(x))
        d.hints = int(hints)
        return d

    # -- phases (network.py:90-126) --------------------------------------------
    def _input(self, values):
        torch = _lib.require_cuda()
        if isinstance(values, torch.Tensor):
            x = values
            if x.device.type != "cuda":
                x = x.to("cuda")
        else:
            arr = np.asarray(values)
            x = torch.as_tensor(arr if arr.dtype == np.uint8 else arr.astype(np.float32),
                                device="cuda")
        if x.dtype not in (torch.uint8, torch.float32):
            x = x.to(torch.float32)
        if tuple(x.shape[1:]) != self.input_shape:
            raise GeometryError(f"input shape {tuple(x.shape[1:])} != network input {self.input_shape}")
        return x.contiguous()

    def forward_into(self, x, bind: _Bind, upto: int | None = None, flags=None,
                     desc=None) -> None:
        """Enqueue the forward phase for a prepared device input (no sync);
        ``upto`` stops before that layer (the learner's fused head takes over);
        ``flags`` (default: the network's) receives non-finite outputs;
        ``desc``: a hinted descriptor copy (``hinted``)."""
        bind.x = x
        bind.struct.x = x.data_ptr()
        fl = self._flags if flags is None else flags
        if upto is None:
            _lib.call("dqn_net_forward", _lib.stream_ptr(), C.byref(desc or self.desc_for(x)),
                      self.flat_values.data_ptr(), C.byref(bind.struct), fl.data_ptr())
            return
        for layer in range(upto):
            self.layer_into(bind, layer, 0, fl, desc=desc)

    def check_output(self) -> None:
        f = int(self._flags.item())
        if f & _lib.FLAG_NONFINITE_OUT:
            self._flags.zero_()
            raise NonFiniteError("non-finite network output")

    def forward(self, values):
        """Run the forward phase; returns the (batch, n_actions) output."""
        x = self._input(values)
        bind = self.binding(x.shape[0])
        self.forward_into(x, bind)
        self.check_output()
        self._cur = bind
        self._phase = _FORWARD
        return self.y.values

    def backward_from(self, bind: _Bind, need_input_grad: bool) -> None:
        bind.struct.dx = bind.dx.data_ptr() if need_input_grad else None
        _lib.call("dqn_net_backward", _lib.stream_ptr(), C.byref(self.desc_for(bind.x)),
                  self.flat_values.data_ptr(), C.byref(bind.struct),
                  bind.dact[-1].data_ptr())

    def backward(self, output_grad):
        """Run the backward phase; returns the gradient w.r.t. the input."""
        torch = _lib.require_cuda()
        if self._phase != _FORWARD:
            raise PhaseOrderError("backward requires a completed forward phase")
        b = self._cur
        g = output_grad if isinstance(output_grad, torch.Tensor) else torch.as_tensor(np.asarray(output_grad))
        if tuple(g.shape) != (b.batch,) + self.output_shape:
            raise GeometryError(f"output grad shape {tuple(g.shape)} != {(b.batch,) + self.output_shape}")
        n = b.batch * int(np.prod(self.output_shape))
        b.dact[-1][:n].copy_(g.reshape(-1).to(device="cuda", dtype=torch.float32))
        self.backward_from(b, self.need_input_grad)
        self._phase = _BACKWARD
        return self.x.grad

    def wgrad_into(self, bind: _Bind) -> None:
        _lib.call("dqn_net_wgrad", _lib.stream_ptr(), C.byref(self.desc_for(bind.x)),
                  self.flat_grads.data_ptr(), C.byref(bind.struct))

    def calculate_gradient(self) -> None:
        """Accumulate parameter gradients for the current pass (``+=``)."""
        if self._phase != _BACKWARD:
            raise PhaseOrderError("calculate_gradient requires a completed backward phase")
        self.wgrad_into(self._cur)
        self._phase = _GRAD

    def validate_finite(self) -> None:
        for v in self.layers:
            b = self._cur
            if b is not None and v.kind != "relu":
                u = v.unit
                n = b.batch * int(np.prod(self._units[u]["out_shape"]))
                Tensor(b.act[u][:n], b.dact[u][:n]).check_finite(f"{v.name} output")
        for name, t in self.named_tensors():
            t.check_finite(name)

    @property
    def y(self) -> Tensor | None:
        b = self._cur
        if b is None:
            return None
        n = b.batch * int(np.prod(self.output_shape))
        shp = (b.batch,) + self.output_shape
        return Tensor(b.act[-1][:n].view(shp), b.dact[-1][:n].view(shp))

    @property
    def x(self) -> Tensor | None:
        b = self._cur
        if b is None or b.x is None:
            return None
        return Tensor(b.x, b.dx[:b.batch])

    def _set_current(self, bind: _Bind, phase: int) -> None:
        self._cur = bind
        self._phase = phase


def build_network(spec, input_shape: tuple[int, int, int], n_actions: int, dueling: bool,
                  dtype=np.float32) -> Network:
    """Assemble the Q-network (network.py:150-177): trunk + plain or dueling
    head, reference layer names (conv1, relu1, ..., fc2 | duel)."""
    if len(input_shape) != 3 or any(s < 1 for s in input_shape):
        raise GeometryError(f"input shape must be HxWxC with positive extents, got {input_shape}")
    if n_actions < 2:
        raise GeometryError(f"need at least 2 actions, got {n_actions}")
    trunk = trunk_layers(spec) if isinstance(spec, str) else list(spec)
    trunk.append(LayerSpec.dueling_head(n_actions) if dueling else LayerSpec.linear(n_actions))
    short = {"convolution": "conv", "linear": "fc", "relu": "relu", "dueling-head": "duel"}
    counts: dict[str, int] = {}
    named = []
    for s in trunk:
        base = short[s.kind]
        counts[base] = counts.get(base, 0) + 1
        named.append(("duel" if s.kind == "dueling-head" else f"{base}{counts[base]}", s))
    return Network(named, input_shape, dtype=dtype)


def _fan(shape) -> tuple[int, int]:
    if len(shape) == 4:
        rf = shape[0] * shape[1]
        return rf * shape[2], rf * shape[3]
    if len(shape) == 2:
        return shape[0], shape[1]
    raise ValueError(f"no fan rule for weight shape {shape}")


def init_params(net: Network, seed) -> None:
    """Seeded Glorot-uniform weights, zero biases (network.py:190-205): the
    same PCG64 draws in registry order as the reference, uploaded to HBM, so
    a given seed gives bit-identical parameters on both paths."""
    torch = _lib.require_cuda()
    rng = np.random.default_rng(seed)
    host = np.zeros(net.n_flat, dtype=np.float32)
    reg = {n: t for n, t in net.named_tensors()}
    offs = {}
    o = 0
    for u in net._units:
        for (tname, tshape), off in zip(u["tensors"], u["offs"]):
            offs[tname] = (off, tshape)
    for p in net.params():
        off, shape = offs[p.name + ".weight"]
        fi, fo = _fan(shape)
        bound = np.sqrt(6.0 / (fi + fo))
        draw = rng.uniform(-bound, bound, size=shape).astype(np.float32)
        host[off:off + draw.size] = draw.ravel()
    del reg, o
    net.flat_values.copy_(torch.as_tensor(host, device="cuda"))
    net.flat_grads.zero_()


def load_params(net: Network, arrays: dict) -> None:
    """Upload named arrays (e.g. an oracle/reference registry) bit-exactly."""
    torch = _lib.require_cuda()
    for name, t in net.named_tensors():
        src = np.asarray(arrays[name], dtype=np.float32)
        if src.shape != t.shape:
            raise GeometryError(f"{name}: shape {src.shape} != {t.shape}")
        t.values.copy_(torch.as_tensor(src, device="cuda"))
