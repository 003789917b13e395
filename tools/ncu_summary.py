"""Summarise an ncu --set full report into a markdown table (per kernel:
duration, DRAM bytes, tensor-pipe %, achieved occupancy, grid)."""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
want = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "B"),
        ("dram__bytes_write.sum", "B"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"), ("launch__grid_size", ""),
        ("launch__registers_per_thread", "")]


def val(r, name):
    i = col.get(name)
    if i is None:
        return float("nan")
    u = units[i]
    v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else float("nan")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(u, 1.0)
    return v * scale


print("| # | kernel | time us | DRAM rd+wr MB | tensor % | warps active % | grid | regs |")
print("|---|---|---|---|---|---|---|---|")
tot = 0.0
for n, r in enumerate(data):
    name = re.sub(r"\(.*", "", r[col["Kernel Name"]])
    name = name.replace("void ", "").replace("dqn::<unnamed>::", "").replace("tc::", "")
    t = val(r, "gpu__time_duration.sum")
    tot += t
    dr = (val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")) / 1e6
    print(f"| {n} | `{name[:60]}` | {t:.2f} | {dr:.3f} | "
          f"{val(r, want[3][0]):.1f} | {val(r, want[4][0]):.1f} | {val(r, want[5][0]):.0f} | "
          f"{val(r, want[6][0]):.0f} |")
print(f"\nserialized total: {tot:.1f} us over {len(data)} kernels")
