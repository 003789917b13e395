"""GPU parity of the Q-network phases against the CPU oracle (norm-wise,
fp32): forward, backward (input grads), wgrad, for the Atari trunk with both
heads, the desk preset and a tiny float-input net; plus determinism and the
reference's geometry / phase-order errors."""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import pytest

from oracle import deepq_oracle as O
from tests.helpers import follow_device_relu_kinks, rel_norm

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-5      # fp32 re-ordered sums vs numpy/BLAS


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def _pair(P, trunk_name, shape, nA, dueling, seed=3):
    o_trunk = {"atari": O.ATARI_TRUNK, "desk": O.DESK_TRUNK}[trunk_name]
    on = P.build_network(trunk_name, shape, nA, dueling)
    P.init_params(on, seed)
    ref = O.QNet(o_trunk, shape, nA, dueling)
    ref.init(seed)
    for n, t in on.named_tensors():
        assert np.array_equal(t.values.cpu().numpy(), ref.params[n]), n   # init is bit-exact
    return on, ref


@pytest.mark.parametrize("dueling", [True, False])
def test_atari_forward_backward_wgrad(P, dueling):
    from paper_1804_05834_b200 import synth
    on, ref = _pair(P, "atari", (84, 84, 4), 4, dueling)
    # perturb biases so ReLU masks are non-trivial
    rng = np.random.default_rng(0)
    for n, t in on.named_tensors():
        if n.endswith("bias"):
            v = (rng.standard_normal(t.shape) * 0.01).astype(np.float32)
            t.values.copy_(torch.as_tensor(v, device="cuda"))
            ref.params[n][...] = v
    x8 = synth.frames(4, 0, np.arange(16))
    q = on.forward(torch.as_tensor(x8, device="cuda")).cpu().numpy()
    xf = O.Ring.lift(x8)
    qr = ref.forward(xf)
    assert rel_norm(q, qr) < TOL
    g = rng.standard_normal(q.shape).astype(np.float32)
    dx = on.backward(g).cpu().numpy()
    dxr = ref.backward(g)
    assert rel_norm(dx, dxr) < TOL
    on.calculate_gradient()
    ref.wgrad()
    for n, t in on.named_tensors():
        assert rel_norm(t.grad.cpu().numpy(), ref.grads[n]) < TOL, n


def test_desk_and_float_input(P):
    on, ref = _pair(P, "desk", (24, 24, 4), 3, True, seed=2)
    x = np.random.default_rng(1).random((5, 24, 24, 4), dtype=np.float32)
    q = on.forward(x).cpu().numpy()
    assert rel_norm(q, ref.forward(x)) < TOL
    g = np.random.default_rng(2).standard_normal(q.shape).astype(np.float32)
    assert rel_norm(on.backward(g).cpu().numpy(), ref.backward(g)) < TOL
    on.calculate_gradient()
    ref.wgrad()
    for n, t in on.named_tensors():
        assert rel_norm(t.grad.cpu().numpy(), ref.grads[n]) < TOL, n


def test_tiny_custom_trunk(P):
    trunk = [P.LayerSpec("convolution", {"filters": 2, "filter_h": 2, "filter_w": 2,
                                         "stride_h": 2, "stride_w": 2}),
             P.LayerSpec.relu(), P.LayerSpec.linear(8), P.LayerSpec.relu()]
    on = P.build_network(trunk, (6, 6, 2), 3, True)
    P.init_params(on, 5)
    ref = O.QNet([("conv", 2, 2, 2), ("relu",), ("fc", 8), ("relu",)], (6, 6, 2), 3, True)
    ref.init(5)
    x = np.random.default_rng(3).random((4, 6, 6, 2), dtype=np.float32)
    assert rel_norm(on.forward(x).cpu().numpy(), ref.forward(x)) < TOL


def test_shape_chain_and_registry(P):
    net = P.build_network("atari", (84, 84, 4), 4, dueling=False)
    shapes = net.layer_output_shapes()
    assert shapes[0] == (20, 20, 32) and shapes[2] == (9, 9, 64) and shapes[4] == (7, 7, 64)
    assert shapes[6] == (512,) and shapes[-1] == (4,)
    fc1 = [v for v in net.layers if v.name == "fc1"][0]
    assert fc1.in_features == 3136
    names = [n for n, _ in P.build_network("atari", (84, 84, 4), 6, True).named_tensors()]
    assert names == ["conv1.weight", "conv1.bias", "conv2.weight", "conv2.bias", "conv3.weight",
                     "conv3.bias", "fc1.weight", "fc1.bias", "duel.value.weight", "duel.value.bias",
                     "duel.advantage.weight", "duel.advantage.bias"]
    n_params = sum(t.size for _, t in P.build_network("atari", (84, 84, 4), 4, True).named_tensors())
    assert n_params == 1_686_693


def test_determinism_and_batch_independence(P):
    from paper_1804_05834_b200 import synth
    net = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(net, 1)
    x = torch.as_tensor(synth.frames(9, 0, np.arange(64)), device="cuda")
    q64 = net.forward(x).clone()
    q64b = net.forward(x).clone()
    assert torch.equal(q64, q64b)
    q8 = net.forward(x[:8]).clone()
    assert torch.equal(q8, net.forward(x[:8]))
    # across batch sizes a row's Q agrees to fp32 rounding: conv2 / conv3
    # split K over a cluster sized by the batch (conv_tc.cu)
    assert float((q8 - q64[:8]).norm() / q64[:8].norm()) < 1e-6


def test_errors(P):
    with pytest.raises(P.GeometryError):
        P.build_network("atari", (30, 30, 4), 4, dueling=False)
    with pytest.raises(P.GeometryError):
        P.build_network("atari", (4, 4, 4), 4, dueling=False)
    with pytest.raises(P.GeometryError):
        P.build_network("desk", (24, 24, 4), 1, dueling=False)
    with pytest.raises(ValueError):
        P.trunk_layers("mega")
    with pytest.raises(P.ConfigError):
        P.build_network("desk", (24, 24, 4), 3, False, dtype=np.float64)
    net = P.build_network("desk", (24, 24, 4), 3, dueling=False)
    with pytest.raises(P.PhaseOrderError):
        net.backward(np.zeros((1, 3), np.float32))
    with pytest.raises(P.GeometryError):
        net.forward(np.zeros((1, 24, 24, 3), dtype=np.float32))
    net.forward(np.zeros((2, 24, 24, 4), np.float32))
    with pytest.raises(P.PhaseOrderError):
        net.calculate_gradient()
    net.params()[0].weight.values.fill_(float("nan"))
    with pytest.raises(P.NonFiniteError):
        net.forward(np.ones((1, 24, 24, 4), np.float32))


def _run_tool(script, env_extra=None):
    import subprocess
    import sys
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, script], env=env, capture_output=True, text=True,
                          timeout=300, cwd=str(Path(__file__).resolve().parent.parent))


def test_fc1_dgrad_tiles_correct_and_deterministic(tmp_path):
    """fc1's dgrad through the tcgen05 engine (32-column tiles, the weights by
    TMA tensor loads) against an fp64 reference over repeated launches.
    Regression test for an odd producer ring (3 stages at 32 columns) that
    raced: every launch must agree bit for bit and stay at 3xTF32 accuracy."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run_tool("tools/lin_dgrad_check.py", {"LIN_DGRAD_DUMP": str(tmp_path / "d.pt")})
    line = [l for l in out.stdout.splitlines() if l.startswith("BN=")]
    assert line, out.stdout + out.stderr
    err = float(line[0].split("rel err ")[1].split()[0])
    assert "deterministic True" in line[0] and err < 1e-5, line[0]


def test_conv_dgrad_accuracy():
    """conv2 / conv3 dgrad (stride phases, split K, ragged batch) against an
    fp64 reference: 3xTF32 accuracy and repeatable."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run_tool("tools/conv_dgrad_check.py")
    line = [l for l in out.stdout.splitlines() if l.startswith("WORST")]
    assert line, out.stdout + out.stderr
    assert float(line[0].split()[1]) < 1e-5, out.stdout


def test_small_batch_forward_matches_batched():
    """Small forwards (batch <= 4: tcgen05 layers, the small-batch kernel for
    layers without one) against the same rows inside a batch-64 forward."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run_tool("tools/small_fwd_check.py")
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr


@pytest.mark.parametrize("batch", [1, 6, 12, 32, 64, 130, 300])
def test_conv1_wgrad_from_frames(P, batch):
    """conv1's weight gradient straight from the uint8 frames (csrc/wgrad_u8.cu:
    one CTA per half image up to 64, then up to 144 CTAs looping over units;
    cluster push + ticketed cross-cluster reduction) against the oracle at batch
    sizes that give 1, 2, 4 and 8-CTA clusters, one and several units per CTA
    (130: uneven); a second accumulation doubles it and two runs are
    bit-identical (layers.py:250-255)."""
    from paper_1804_05834_b200 import synth
    on, ref = _pair(P, "atari", (84, 84, 4), 4, True, seed=3)
    x8 = synth.frames(9, 0, np.arange(batch))
    q = on.forward(torch.as_tensor(x8, device="cuda")).cpu().numpy()
    ref.forward(O.Ring.lift(x8))
    g = np.random.default_rng(batch).standard_normal(q.shape).astype(np.float32)
    on.backward(g)
    # pre-activations within fp32 rounding of a ReLU kink take the device's side
    follow_device_relu_kinks(ref, [a.cpu().numpy() for a in on.binding(batch).act])
    ref.backward(g)
    ref.wgrad()
    t1 = dict(on.named_tensors())
    xd = torch.as_tensor(x8, device="cuda")
    runs = []
    for _ in range(2):
        for _, t in on.named_tensors():
            t.grad.zero_()
        on.forward(xd)
        on.backward(g)
        on.calculate_gradient()
        runs.append((t1["conv1.weight"].grad.clone(), t1["conv1.bias"].grad.clone()))
    assert torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1])
    for n in ("conv1.weight", "conv1.bias"):
        assert rel_norm(t1[n].grad.cpu().numpy(), ref.grads[n]) < TOL, n
    on.forward(xd)
    on.backward(g)
    on.calculate_gradient()                       # accumulates: grads += dW
    w2 = t1["conv1.weight"].grad.cpu().numpy()
    assert rel_norm(w2, 2 * ref.grads["conv1.weight"]) < TOL


@pytest.mark.parametrize("batch", [1, 2, 3, 33, 64, 130, 1024])
def test_conv_tc_forward_layers(P, batch):
    """conv2 / conv3 forward (conv_tc.cu: TMA-fed implicit GEMM, tiles of
    whole images, cluster split-K) against an fp64 convolution of the same
    layer input, at batch sizes with partial last tiles and several waves."""
    import torch.nn.functional as F
    from paper_1804_05834_b200 import synth
    on = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 5)
    rng = np.random.default_rng(batch)
    for n, t in on.named_tensors():
        if n.endswith("bias"):
            t.values.copy_(torch.as_tensor((rng.standard_normal(t.shape) * 0.01).astype(np.float32),
                                           device="cuda"))
    x8 = synth.frames(4, 1, np.arange(batch) * 7 + 3)
    on.forward(torch.as_tensor(x8, device="cuda"))
    bind = on.binding(batch)
    tens = dict(on.named_tensors())
    shapes = [tuple(u["out_shape"]) for u in on._units]
    for l, (name, fh, st) in enumerate([("conv2", 4, 2), ("conv3", 3, 1)], start=1):
        h, w, c = shapes[l - 1]
        oh, ow, n = shapes[l]
        xin = bind.act[l - 1][: batch * h * w * c].view(batch, h, w, c).double().permute(0, 3, 1, 2)
        W = tens[f"{name}.weight"].values.double().reshape(fh, fh, c, n).permute(3, 2, 0, 1)
        ref = F.relu(F.conv2d(xin, W, tens[f"{name}.bias"].values.double(), stride=st))
        ref = ref.permute(0, 2, 3, 1)
        got = bind.act[l][: batch * oh * ow * n].view(batch, oh, ow, n).double()
        err = (got - ref).norm() / ref.norm()
        assert err < 2e-6, (name, batch, float(err))
        assert float((got - ref).abs().max()) <= 1e-5 * float(ref.abs().max()) + 1e-7, name


@pytest.mark.parametrize("batch", [1, 3, 32, 33, 130])
def test_conv_tc_dgrad_layers(P, batch):
    """conv2 / conv3 input gradients (conv_tc.cu dgrad: dY and W by TMA, one
    GEMM per stride phase, taps off the dY grid zero-filled by the TMA) against
    an fp64 transposed convolution of the same dY, masked by the layer
    below's ReLU."""
    import torch.nn.functional as F
    from paper_1804_05834_b200 import synth
    on = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 6)
    x8 = synth.frames(5, 0, np.arange(batch) * 3 + 1)
    q = on.forward(torch.as_tensor(x8, device="cuda"))
    g = np.random.default_rng(batch).standard_normal(tuple(q.shape)).astype(np.float32)
    on.backward(g)
    bind = on.binding(batch)
    tens = dict(on.named_tensors())
    shapes = [tuple(u["out_shape"]) for u in on._units]
    for l, (name, fh, st) in enumerate([("conv2", 4, 2), ("conv3", 3, 1)], start=1):
        h, w, c = shapes[l - 1]
        oh, ow, n = shapes[l]
        dy = bind.dact[l][: batch * oh * ow * n].view(batch, oh, ow, n).double().permute(0, 3, 1, 2)
        W = tens[f"{name}.weight"].values.double().reshape(fh, fh, c, n).permute(3, 2, 0, 1)
        ref = F.conv_transpose2d(dy, W, stride=st).permute(0, 2, 3, 1)
        act = bind.act[l - 1][: batch * h * w * c].view(batch, h, w, c).double()
        ref = ref * (act > 0)
        got = bind.dact[l - 1][: batch * h * w * c].view(batch, h, w, c).double()
        err = (got - ref).norm() / ref.norm()
        assert err < 2e-6, (name, batch, float(err))
        assert float((got - ref).abs().max()) <= 1e-5 * float(ref.abs().max()) + 1e-12, name


@pytest.mark.parametrize("batch", [1, 2, 3, 33, 64, 130, 1024])
def test_conv1_tc_forward(P, batch):
    """conv1 forward from the uint8 frames (conv1_tc.cu: frame slab and W by
    bulk copies, integer A, 1/255 on the sum) against an fp64 convolution of
    the frames / 255."""
    import torch.nn.functional as F
    from paper_1804_05834_b200 import synth
    on = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 8)
    tens = dict(on.named_tensors())
    tens["conv1.bias"].values.copy_(torch.linspace(-0.05, 0.05, 32, device="cuda"))
    x8 = torch.as_tensor(synth.frames(6, 1, np.arange(batch) * 5 + 2), device="cuda")
    on.forward(x8)
    bind = on.binding(batch)
    xin = (x8.double() / 255.0).permute(0, 3, 1, 2)
    W = tens["conv1.weight"].values.double().reshape(8, 8, 4, 32).permute(3, 2, 0, 1)
    ref = F.relu(F.conv2d(xin, W, tens["conv1.bias"].values.double(), stride=4)).permute(0, 2, 3, 1)
    got = bind.act[0][: batch * 20 * 20 * 32].view(batch, 20, 20, 32).double()
    err = (got - ref).norm() / ref.norm()
    assert err < 2e-6, (batch, float(err))
    assert float((got - ref).abs().max()) <= 1e-5 * float(ref.abs().max()), batch


def test_side_hint_changes_only_the_launch_shapes(P):
    """dqn_net_desc.hints = DQN_NET_HINT_SIDE (the learner's target trunk):
    smaller K splits / clusters, so the same outputs up to fp32 summation
    order, and bit-identical from run to run."""
    from paper_1804_05834_b200 import _lib, synth
    net = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(net, 4)
    x = torch.as_tensor(synth.frames(2, 1, np.arange(32)), device="cuda")
    bind = net.binding(32)
    outs = []
    for desc in (None, net.hinted(x, _lib.NET_HINT_SIDE), net.hinted(x, _lib.NET_HINT_SIDE)):
        net.forward_into(x, bind, desc=desc)
        torch.cuda.synchronize()
        outs.append([a.clone() for a in bind.act])
    for l in range(len(outs[0])):
        assert torch.equal(outs[1][l], outs[2][l]), l
        # fp32 re-association only (each layer's K split differs): 3e-6 covers the
        # accumulated difference down the trunk
        assert float((outs[1][l] - outs[0][l]).norm() / outs[0][l].norm()) < 3e-6, l


@pytest.mark.parametrize("geom", [(27, 3, 3), (16, 4, 2), (12, 3, 1)])
def test_conv_tc_other_geometries_forward_backward_wgrad(P, geom):
    """Custom trunks whose 64-filter convolutions take the TMA-fed kernel with
    other strides / filters / image sizes than the Atari net (stride 3, one
    and two images per tile, 64-channel input): forward, input gradient and
    weight gradient against the oracle."""
    hw, f, s = geom
    conv = lambda n, ff, ss: P.LayerSpec("convolution", {"filters": n, "filter_h": ff,  # noqa: E731
                                                          "filter_w": ff, "stride_h": ss,
                                                          "stride_w": ss})
    trunk = [conv(32, 1, 1), P.LayerSpec.relu(), conv(64, f, s), P.LayerSpec.relu(),
             conv(64, f, 1) if (hw - f) // s + 1 >= f else conv(64, 1, 1), P.LayerSpec.relu(),
             P.LayerSpec.linear(16), P.LayerSpec.relu()]
    o_trunk = [("conv", 32, 1, 1), ("relu",), ("conv", 64, f, s), ("relu",),
               ("conv", 64, f, 1) if (hw - f) // s + 1 >= f else ("conv", 64, 1, 1), ("relu",),
               ("fc", 16), ("relu",)]
    shape = (hw, hw, 4)
    on = P.build_network(trunk, shape, 3, True)
    P.init_params(on, 7)
    ref = O.QNet(o_trunk, shape, 3, True)
    ref.init(7)
    rng = np.random.default_rng(hw)
    for n, t in on.named_tensors():
        if n.endswith("bias"):
            v = (rng.standard_normal(t.shape) * 0.01).astype(np.float32)
            t.values.copy_(torch.as_tensor(v, device="cuda"))
            ref.params[n][...] = v
    x = rng.random((5,) + shape, dtype=np.float32)
    q = on.forward(x).cpu().numpy()
    assert rel_norm(q, ref.forward(x)) < TOL
    g = rng.standard_normal(q.shape).astype(np.float32)
    dx = on.backward(g).cpu().numpy()
    assert rel_norm(dx, ref.backward(g)) < TOL
    on.calculate_gradient()
    ref.wgrad()
    for n, t in on.named_tensors():
        assert rel_norm(t.grad.cpu().numpy(), ref.grads[n]) < 1e-4, n


@pytest.mark.parametrize("hw,stride", [(64, 4), (36, 2), (44, 4)])
def test_conv1_tc_other_geometries(P, hw, stride):
    """The uint8 first layer (8x8 filters over 4 channels, 32 filters) on other
    frame sizes and strides: conv1_tc tiles of 3-15 output rows; the network's
    forward and gradients against the oracle."""
    trunk = [P.LayerSpec("convolution", {"filters": 32, "filter_h": 8, "filter_w": 8,
                                         "stride_h": stride, "stride_w": stride}),
             P.LayerSpec.relu(), P.LayerSpec.linear(16), P.LayerSpec.relu()]
    shape = (hw, hw, 4)
    on = P.build_network(trunk, shape, 3, False)
    P.init_params(on, 9)
    ref = O.QNet([("conv", 32, 8, stride), ("relu",), ("fc", 16), ("relu",)], shape, 3, False)
    ref.init(9)
    rng = np.random.default_rng(hw + stride)
    x8 = rng.integers(0, 256, size=(6,) + shape, dtype=np.uint8)
    q = on.forward(torch.as_tensor(x8, device="cuda")).cpu().numpy()
    assert rel_norm(q, ref.forward(O.Ring.lift(x8))) < TOL
    g = rng.standard_normal(q.shape).astype(np.float32)
    on.backward(g)
    ref.backward(g)
    on.calculate_gradient()
    ref.wgrad()
    for n, t in on.named_tensors():
        assert rel_norm(t.grad.cpu().numpy(), ref.grads[n]) < 1e-4, n


@pytest.mark.parametrize("batch", [65, 130, 1024])
def test_fc1_lin_tc_large_batch(P, batch):
    """fc1 above learner batch sizes on lin_tc (64-row batch blocks, K split
    for ~128 CTAs): forward against an fp64 product of the same input, and the
    input gradient (W rows K-major by TMA) against the fp64 transposed product
    masked by the layer below's ReLU."""
    from paper_1804_05834_b200 import synth
    on = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, 11)
    x = torch.as_tensor(synth.frames(7, 0, np.arange(batch) % 4096), device="cuda")
    q = on.forward(x)
    on.backward(torch.as_tensor(np.random.default_rng(batch).standard_normal(tuple(q.shape)),
                                dtype=torch.float32, device="cuda"))
    bind = on.binding(batch)
    tens = dict(on.named_tensors())
    W = tens["fc1.weight"].values.double()                   # [3136][512]
    xin = bind.act[2][: batch * 3136].view(batch, 3136).double()
    ref = torch.relu(xin @ W + tens["fc1.bias"].values.double())
    got = bind.act[3][: batch * 512].view(batch, 512).double()
    # fp32-level for a 3,136-long dot product (one K chain of 1,568-3,136 at
    # these batches; the numpy fp32 oracle is at ~1e-6 itself)
    assert float((got - ref).norm() / ref.norm()) < 5e-6
    dy = bind.dact[3][: batch * 512].view(batch, 512).double()
    dref = (dy @ W.T) * (xin > 0)
    dgot = bind.dact[2][: batch * 3136].view(batch, 3136).double()
    assert float((dgot - dref).norm() / dref.norm()) < 5e-6
