"""Diagnostic: which kernels the trunk phases of a few custom geometries launch."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1804_05834_b200 as P
from torch.profiler import profile, ProfilerActivity
conv = lambda n, ff, ss: P.LayerSpec("convolution", {"filters": n, "filter_h": ff, "filter_w": ff, "stride_h": ss, "stride_w": ss})
for hw, f, s in [(27, 3, 3), (16, 4, 2), (12, 3, 1)]:
    trunk = [conv(32, 1, 1), P.LayerSpec.relu(), conv(64, f, s), P.LayerSpec.relu(),
             conv(64, f, 1) if (hw - f) // s + 1 >= f else conv(64, 1, 1), P.LayerSpec.relu(),
             P.LayerSpec.linear(16), P.LayerSpec.relu()]
    on = P.build_network(trunk, (hw, hw, 4), 3, True)
    P.init_params(on, 7)
    x = np.random.default_rng(1).random((5, hw, hw, 4), dtype=np.float32)
    on.forward(x); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        q = on.forward(x); on.backward(np.ones(q.shape, np.float32)); on.calculate_gradient(); torch.cuda.synchronize()
    names = sorted({e.name.replace("(anonymous namespace)::", "").split("(")[0][-48:]
                    for e in prof.events() if e.device_type.name == "CUDA"})
    print((hw, f, s), [n for n in names if "conv" in n or "gemm" in n])
