"""conv1 wgrad-from-frames alone (product build), for ncu captures."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, synth  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
x = torch.as_tensor(synth.frames(3, 0, np.arange(batch)), device="cuda")
q = net.forward(x)
net.backward(torch.randn(q.shape, device="cuda"))
b = net._cur
desc = _lib.NetDesc.from_buffer_copy(net._desc_u8)
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
args = (_lib.stream_ptr(), C.byref(desc), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
        C.byref(b.struct), 0, 2, flags.data_ptr())
for _ in range(3):
    _lib.call("dqn_net_layer", *args)
torch.cuda.synchronize()
