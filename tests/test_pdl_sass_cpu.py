"""Every kernel launched with programmatic dependent launch must not read
global memory before its griddepcontrol.wait (SASS ACQBULK): a hoisted load
reads what the previous kernel of the stream may still be writing (found
once: a __restrict__ index load in the frame gather, wrong only under CUDA
graphs).  Static check of the built library's SASS (cuobjdump, no GPU)."""

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1804_05834_b200" / "libdqn_b200.so"


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not LIB.exists(),
                    reason="needs cuobjdump and the built library")
def test_no_global_load_before_pdl_wait():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "pdl_hoist_scan.py"), str(LIB)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("PDL wait: 0"), out.stdout
