"""Per-kernel SASS instruction histogram of the built library (the evidence
that the hot kernels run on tcgen05 / TMEM / TMA): counts of the
Blackwell-specific mnemonics per kernel from `cuobjdump -sass`.

    python tools/sass_histogram.py [lib] > profiles/<tag>_sass_histogram.md
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_1804_05834_b200" / "libdqn_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP",
        "SYNCS", "ACQBULK", "FFMA", "DFMA", "LDG", "STG", "LDS", "STS"]
per = defaultdict(Counter)
name = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        name = m.group(1)
        continue
    if name is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                per[name][k] += 1


def demangle(n):
    out = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    out = out.replace("(anonymous namespace)::", "").replace("dqn::", "")
    out = re.sub(r"\((?!int\)).*", "", out)
    return out.replace("tc::", "")[:90]


print("# SASS instruction histogram per kernel (`cuobjdump -sass libdqn_b200.so`)\n")
print("tcgen05: UTCHMMA = MMA issue, UTCBAR = commit, LDTM/STTM = TMEM loads/stores;")
print("TMA: UTMALDG = tensor-map loads, UBLKCP = bulk copies; SYNCS = mbarrier ops.\n")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---|" * len(KEYS))
tot = Counter()
for n in sorted(per, key=lambda n: demangle(n)):
    c = per[n]
    tot.update(c)
    print(f"| `{demangle(n)}` | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")
print("| **total** | " + " | ".join(str(tot.get(k, 0)) for k in KEYS) + " |")
