"""Diagnostic: per-CTA phase marks of the conv1 wgrad-from-frames kernel
(csrc/wgrad_u8.cu, trace build)."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("DQN_B200_LIB", str(ROOT / "paper_1804_05834_b200" / "libdqn_b200_trace.so"))
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1804_05834_b200 as P  # noqa: E402
from paper_1804_05834_b200 import _lib, synth  # noqa: E402

net = P.build_network("atari", (84, 84, 4), 4, True)
P.init_params(net, 1)
for skip in [int(v) for v in (sys.argv[1:] or ['0'])]:
  _lib.lib.dqn_w1_skip(skip)
  print('skip', skip)
  for batch in (32,):
      x = torch.as_tensor(synth.frames(3, 0, np.arange(batch)), device="cuda")
      q = net.forward(x)
      net.backward(torch.randn(q.shape, device="cuda"))
      b = net._cur
      desc = _lib.NetDesc.from_buffer_copy(net._desc_u8)
      flags = torch.zeros(1, dtype=torch.int32, device="cuda")
      args = (_lib.stream_ptr(), C.byref(desc), net.flat_values.data_ptr(), net.flat_grads.data_ptr(),
              C.byref(b.struct), 0, 2, flags.data_ptr())
      for _ in range(5):
          _lib.call("dqn_net_layer", *args)
      torch.cuda.synchronize()
      e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      e0.record()
      for _ in range(20):
          _lib.call("dqn_net_layer", *args)
      e1.record()
      torch.cuda.synchronize()
      print(f"batch {batch}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch (back to back)")
      _lib.call("dqn_net_layer", *args)
      torch.cuda.synchronize()
      buf = (C.c_ulonglong * (256 * 12))()
      _lib.lib.dqn_w1_trace(buf)
      t = np.frombuffer(buf, dtype=np.uint64).reshape(256, 12).astype(np.int64)
      t = t[t[:, 0] > 0]
      t0 = t[:, 0].min()
      print(f"  {len(t)} CTAs")
      names = ["entry", "pdl", "Bbuilt", "img", "mma", "epi", "clred", "ticket", "final", "issue0", "issue1"]
      for i, n in enumerate(names):
          sel = t[:, i] >= t0
          v = (t[sel, i] - t0) / 1e3
          print(f"  {n:7s} mean {v.mean():6.2f} max {v.max():6.2f} us  ({sel.sum()} CTAs)")
