"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/dqn_b200.h declares (no compute calls)."""

import ctypes
import re
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "dqn_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(dqn_[a-z0-9_]+)\(", text, re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ["dqn_ring_gather", "dqn_tree_sample", "dqn_tree_update", "dqn_net_forward",
                 "dqn_net_backward", "dqn_net_wgrad", "dqn_td_loss", "dqn_rmsprop_step",
                 "dqn_sync_target"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1804_05834_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.EXPORTED)
    assert lib.dqn_abi_version() == 5


def test_struct_layouts_match_header():
    from paper_1804_05834_b200 import _lib
    # dqn_layer_desc: 12 int32 + 4 int64 = 80 bytes; net desc: 16 + 8*80
    assert ctypes.sizeof(_lib.LayerDesc) == 80
    assert ctypes.sizeof(_lib.NetDesc) == 16 + 8 * 80
    assert ctypes.sizeof(_lib.Binding) == 8 + 8 + 16 * 8 + 8 + 8 + 8   # ... scratch_floats


def test_product_path_refuses_without_gpu(monkeypatch):
    import pytest
    import torch
    from paper_1804_05834_b200 import _lib
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.require_cuda()


def test_product_path_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: importing the package with the CUDA library missing
    raises ImportError; without a GPU every constructor raises."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DQN_B200_LIB=str(tmp_path / "missing.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_1804_05834_b200"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "ImportError" in r.stderr
    probe = ("import torch, paper_1804_05834_b200 as P\n"
             "if torch.cuda.is_available():\n    print('GPU')\nelse:\n"
             "    try:\n        P.build_network('atari', (84, 84, 4), 4, True)\n"
             "        print('NO-RAISE')\n"
             "    except Exception as e:\n        print('RAISED', type(e).__name__)\n")
    r = subprocess.run([sys.executable, "-c", probe], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert r.stdout.startswith("GPU") or r.stdout.startswith("RAISED"), r.stdout + r.stderr


def test_header_constants_match_the_binding():
    """Every DQN_FLAG_* / DQN_TD_* / DQN_NET_HINT_* / DQN_LAYER_* value the
    Python binding uses equals the header's."""
    from paper_1804_05834_b200 import _lib
    text = HEADER.read_text()
    defines = {m.group(1): int(m.group(2), 0)
               for m in re.finditer(r"#define\s+(DQN_\w+)\s+\(?(0x[0-9a-fA-F]+|\d+)", text)}
    pairs = {"DQN_NET_HINT_SIDE": _lib.NET_HINT_SIDE}
    for name in dir(_lib):
        if name.startswith(("FLAG_", "TD_")) and ("DQN_" + name) in defines:
            pairs["DQN_" + name] = getattr(_lib, name)
    assert "DQN_NET_HINT_SIDE" in defines and len(pairs) >= 4, sorted(pairs)
    for k, v in pairs.items():
        assert defines[k] == v, (k, defines[k], v)


def test_sample_gather_weights_pointers_both_or_neither():
    """dqn_sample_gather / dqn_frame_sample_gather: prob and weight are both
    given (the launch's IS-weights row) or both NULL (the caller computes them
    with dqn_tree_sample); one without the other is an argument error, found
    before any device work."""
    from paper_1804_05834_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    p = ctypes.c_void_p(16)                       # never dereferenced: the check comes first
    sg = lib.dqn_sample_gather
    sg.restype = ctypes.c_int
    args = [None, p, ctypes.c_int(20), p, p, ctypes.c_int(32), p, p, p, None, p, p, p,
            ctypes.c_int64(28224), p, p, p, p, p, p, p, p]
    assert sg(*args) == 1                         # DQN_ERR_INVALID_ARG (weight NULL, prob not)
    fg = lib.dqn_frame_sample_gather
    fg.restype = ctypes.c_int
    args = [None, p, ctypes.c_int(20), p, p, ctypes.c_int(32), p, p, None, p, p, p,
            ctypes.c_int64(7056), p, ctypes.c_int(4), p, p, p, p, p, p, p, p]
    assert fg(*args) == 1                         # prob NULL, weight not
