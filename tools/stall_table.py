"""Top SASS lines by warp-stall samples for one kernel launch of an ncu report
(`--page source`), as a markdown table.

    python tools/stall_table.py <report.ncu-rep> <kernel regex> <launch-skip> "<title>" [n]
"""
import csv
import io
import subprocess
import sys

rep, regex, skip, title = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{regex}", "--launch-skip", str(skip), "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
name = lines[0].split(",", 1)[1].strip().strip('",')
rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
key = "Warp Stall Sampling (All Samples)"
rows = [r for r in rows if (r.get(key) or "0").isdigit()]   # repeated header lines
tot = sum(int(r[key] or 0) for r in rows)
rows.sort(key=lambda r: -int(r[key] or 0))
L = [f"# {title}", "", f"Kernel `{name}`, {tot} stall samples (ncu source page, SASS).", "",
     "| samples | share | executed | SASS |", "|---|---|---|---|"]
for r in rows[:n]:
    s = int(r[key] or 0)
    L.append(f"| {s} | {100.0 * s / max(tot, 1):.1f}% | {r['Instructions Executed']} | "
             f"`{r['Source'].strip()}` |")
print("\n".join(L))
