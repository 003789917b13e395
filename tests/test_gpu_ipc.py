"""The cross-process half of the data-parallel learner's peer-ring gather
(dp.DeviceDataParallelLearner, csrc/dp.cu dqn_ipc_* / dqn_dp_gather): a
shareable ring's CUDA-IPC handles, opened by ANOTHER process, must give that
process's gather kernel the owner's bytes.

One GPU is available, so both processes use cuda:0 (IPC within one device);
no NCCL communicator and no cross-process kernel waits are involved -- the
owner just keeps its ring alive while the reader gathers from it.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REPO = Path(__file__).resolve().parent.parent

_READER = r"""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1804_05834_b200 import _lib
from paper_1804_05834_b200.dp import _PeerRing, _RING_FIELDS
import paper_1804_05834_b200 as P
handles = [bytes.fromhex(h) for h in open(sys.argv[2]).read().split()]
k, cap, slot = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
opened = []
for h in handles:
    p = C.c_void_p()
    _lib.call("dqn_ipc_open", (C.c_uint8 * 64).from_buffer_copy(h), C.byref(p))
    opened.append(p)
own = P.ReplayMemory(cap, (84, 84, 4))
own.fill_synthetic(99, cap)
S = _PeerRing.struct()
tab = (S * 2)(S(*[p.value for p in opened]),
              S(*[getattr(own, f).data_ptr() for f in _RING_FIELDS]))
dtab = torch.frombuffer(bytearray(bytes(tab)), dtype=torch.uint8).to("cuda")
K = 2 * k
rng = np.random.default_rng(5)
owner = np.zeros(K, dtype=np.int64)           # rank 0's strata all live on the peer
local = rng.integers(0, cap, K)
table = torch.zeros(2 * K, dtype=torch.float64, device="cuda")
table[0::2] = torch.as_tensor(local.astype(np.float64), device="cuda")
table[1::2] = 1.0
sums = torch.tensor([float(K), 100.0, 0.0], dtype=torch.float64, device="cuda")
beta = torch.full((1,), 0.5, dtype=torch.float64, device="cuda")
x = torch.zeros((2 * k, 84, 84, 4), dtype=torch.uint8, device="cuda")
a = torch.zeros(k, dtype=torch.int64, device="cuda")
rw = torch.zeros(k, dtype=torch.float64, device="cuda")
t = torch.zeros(k, dtype=torch.bool, device="cuda")
lidx = torch.zeros(K, dtype=torch.int64, device="cuda")
w_all = torch.zeros(K, dtype=torch.float64, device="cuda")
w_mine = torch.zeros(k, dtype=torch.float64, device="cuda")
_lib.call("dqn_dp_gather", _lib.stream_ptr(), dtab.data_ptr(),
          torch.as_tensor(owner, device="cuda").data_ptr(), table.data_ptr(), k, 0, slot,
          x.data_ptr(), a.data_ptr(), rw.data_ptr(), t.data_ptr(), sums.data_ptr(),
          beta.data_ptr(), K, lidx.data_ptr(), w_all.data_ptr(), w_mine.data_ptr())
torch.cuda.synchronize()
torch.save({"local": torch.as_tensor(local[:k]), "x": x.cpu(), "a": a.cpu(), "r": rw.cpu(), "t": t.cpu()},
           sys.argv[6])
for p in opened:
    _lib.call("dqn_ipc_close", p)
print("reader ok")
"""


def test_peer_ring_gather_through_ipc_in_another_process(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    from paper_1804_05834_b200.dp import _RING_FIELDS
    k, cap = 16, 64
    m = P.ReplayMemory(cap, (84, 84, 4), shareable=True)
    m.fill_synthetic(31, cap)
    torch.cuda.synchronize()
    hfile, out = tmp_path / "handles.txt", tmp_path / "gathered.pt"
    hfile.write_text(" ".join(m.shared[f].handle().hex() for f in _RING_FIELDS))
    script = tmp_path / "reader.py"
    script.write_text(_READER)
    r = subprocess.run([sys.executable, str(script), str(REPO), str(hfile), str(k), str(cap),
                        str(m.slot_bytes), str(out)], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    g = torch.load(out)
    for b, i in enumerate(g["local"]):
        i = int(i)
        assert torch.equal(g["x"][b], m.states[i].cpu())
        assert torch.equal(g["x"][k + b], m.next_states[i].cpu())
        assert g["a"][b].item() == m.actions[i].item()
        assert g["r"][b].item() == m.rewards[i].item()
        assert g["t"][b].item() == m.terminals[i].item()
