"""Turn the outputs of tools/profile_job.sh (gpurun_out/) into the committed
profile evidence:

  profiles/<tag>_bench_launch_list.md   one steady-state update from the ncu
                                        launch list of the bench command
  profiles/<tag>_bench_launches.csv     that raw launch list
  profiles/<tag>_step_gemms.md          ncu --set full of every GEMM of an update
  profiles/roofline_traffic.json        DRAM bytes per launch, read by bench.py

usage: python tools/profile_summaries.py r01_v3 "<build description>"
"""
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1]
build = sys.argv[2] if len(sys.argv) > 2 else ""


def clean(name):
    name = re.sub(r"\(.*", "", name).replace("void ", "")
    for p in ("dqn::<unnamed>::", "dqn::tc::", "<unnamed>::", "dqn::"):
        name = name.replace(p, "")
    return name


# ------------------------------------------------------------- launch list
rows = list(csv.reader(open(OUT / "launches_bench.csv")))
hdr, recs = None, []
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            us = v / 1000 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1000)
            recs.append((clean(d["Kernel Name"]), us))
starts = [i for i, (n, _) in enumerate(recs)
          if n.startswith("tree_sample_kernel") or n.startswith("sample_gather_kernel")]
updates = []
for a in starts:
    seg = []
    for r in recs[a:]:
        seg.append(r)
        if r[0].startswith("rms_apply_kernel"):
            break
    updates.append(seg)
u = updates[-2] if len(updates) > 1 else updates[-1]
tot = sum(v for _, v in u)
L = [f"# {tag} — ncu launch list of the bench command (one learner update)", "",
     "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "
     "launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu` "
     f"(raw list: `{tag}_bench_launches.csv`).", "",
     f"Build: {build}", "",
     "ncu serialises every launch and flushes caches: absolute times are cold-cache and",
     "un-overlapped (the graph runs the target forward, the wgrads and the priority update",
     "beside the critical chain); compare **shares**.",
     f"One steady-state update, {len(u)} launches, serialised sum {tot:.1f} us:", "",
     "| # | kernel | us | share |", "|---|---|---|---|"]
for i, (n, v) in enumerate(u):
    L.append(f"| {i} | `{n[:80]}` | {v:.2f} | {100 * v / tot:.1f}% |")
g = sum(v for n, v in u if "tc_gemm" in n)
conv1w = [v for n, v in u if "WgradPol<unsigned char" in n]
L += ["", f"tcgen05 GEMMs: {g:.1f} us = {100 * g / tot:.1f}% of the serialised update; "
      f"conv1 wgrad (the bench's roofline kernel): "
      + ", ".join(f"{v:.2f} us ({100 * v / tot:.1f}%)" for v in conv1w) + "."]
(PROF / f"{tag}_bench_launch_list.md").write_text("\n".join(L) + "\n")
shutil.copy(OUT / "launches_bench.csv", PROF / f"{tag}_bench_launches.csv")

# ------------------------------------------------------------- GEMM capture
metrics = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "l1tex__m_xbar2l1tex_read_bytes.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,"
           "launch__registers_per_thread,"
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio")
raw = subprocess.run(["ncu", "-i", str(OUT / "step_gemms.ncu-rep"), "--page", "raw", "--csv",
                      "--metrics", metrics], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1, "us": 1, "usecond": 1,
         "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3}


def val(r, n):
    return float(r[col[n]].replace(",", "")) * scale.get(units[col[n]], 1)


labels = ["conv1.fwd (batch 32, target)", "conv2.fwd (batch 32, target)",
          "conv3.fwd (batch 32, target)", "fc1.fwd (batch 32, target)",
          "conv1.fwd (batch 64)", "conv2.fwd (batch 64)", "conv3.fwd (batch 64)",
          "fc1.fwd (batch 64)", "fc1.dgrad (batch 32)",
          "conv3.wgrad (batch 32)", "conv3.dgrad (batch 32)", "conv2.wgrad (batch 32)",
          "conv2.dgrad (batch 32)", "conv1.wgrad (batch 32)"]
L = [f"# {tag} — every tcgen05 GEMM of one learner update, `ncu --set full`", "",
     "Command: `ncu --profile-from-start off --set full --import-source on --clock-control none "
     "-k regex:tc_gemm -o step_gemms python tools/profile_step.py` (eager launches of one cfg4 "
     "update, B = 32, after 5 warm-up updates).", "", f"Build: {build}", "",
     "ncu flushes caches and serialises launches: DRAM bytes are cold-cache per launch.", "",
     "| # | layer phase | policy | grid | us | DRAM rd+wr MB | L2->L1 MB | tensor % | SM thru % "
     "| long-sb stall/issue | regs |", "|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for i, r in enumerate(data):
    name = clean(r[col["Kernel Name"]]).replace("tc_gemm_kernel", "").strip("<>") + ">"
    dr = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    lab = labels[i] if i < len(labels) else f"kernel {i}"
    traffic[lab] = {"dram_bytes": dr, "policy": name, "us_ncu": val(r, "gpu__time_duration.sum")}
    L.append(
        f"| {i} | {lab} | `{name}` | {int(val(r, 'launch__grid_size'))} | "
        f"{val(r, 'gpu__time_duration.sum'):.2f} | {dr / 1e6:.3f} | "
        f"{val(r, 'l1tex__m_xbar2l1tex_read_bytes.sum') / 1e6:.2f} | "
        f"{float(r[col['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']]):.1f} | "
        f"{float(r[col['sm__throughput.avg.pct_of_peak_sustained_elapsed']]):.1f} | "
        f"{float(r[col['smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio']]):.2f} | "
        f"{int(val(r, 'launch__registers_per_thread'))} |")
(PROF / f"{tag}_step_gemms.md").write_text("\n".join(L) + "\n")
json.dump({"source": f"profiles/{tag}_step_gemms.md (ncu --set full, cold cache, "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch)",
           "kernels": traffic}, open(PROF / "roofline_traffic.json", "w"), indent=1)
print("\n".join(L[8:]))
