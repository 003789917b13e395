"""Scan libdqn_b200.so's SASS for global loads issued before the PDL wait
(ACQBULK = griddepcontrol.wait): such a load can read data the previous
kernel of the stream has not finished writing."""
import re
import subprocess
import sys
from pathlib import Path

lib = Path(sys.argv[1] if len(sys.argv) > 1 else
           Path(__file__).resolve().parent.parent / "paper_1804_05834_b200" / "libdqn_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
bad = []
for block in sass.split("Function : ")[1:]:
    name = block.split("\n", 1)[0].strip()
    pre = []
    for line in block.splitlines():
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if not m:
            continue
        ins = m.group(1)
        if "ACQBULK" in ins:
            break
        if re.search(r"\b(LDG|LD\.E|LDGSTS|UBLKCP|UTMALDG)\b", ins) or ins.startswith(("LDG", "@P")) and "LDG" in ins:
            pre.append(ins)
    else:
        continue            # no PDL wait in this function
    if pre:
        bad.append((name, pre))
for name, pre in bad:
    print(name[:110], "|", len(pre), "loads before ACQBULK, e.g.", pre[0][:60])
print("functions with loads hoisted above the PDL wait:", len(bad))
