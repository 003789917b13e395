"""Turn the outputs of tools/profile_job.sh (gpurun_out/) into the committed
profile evidence:

  profiles/<tag>_bench_launch_list.md   one steady-state update from the ncu
                                        launch list of the bench command
  profiles/<tag>_bench_launches.csv     that raw launch list
  profiles/<tag>_step_kernels.md        ncu --set full of every kernel of an update
  profiles/roofline_traffic.json        DRAM bytes per launch, read by bench.py

Inputs: gpurun_out/<tag>/ (tools/profile_job.sh with TAG=<tag>), including
the nvidia-smi clock snapshots taken around the captures.

usage: python tools/profile_summaries.py r02 "<build description>"
"""
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"
tag = sys.argv[1]
OUT = ROOT / "gpurun_out" / tag
build = sys.argv[2] if len(sys.argv) > 2 else ""


def clocks_note():
    out = []
    for f in ("clocks_before.csv", "clocks_after.csv"):
        p = OUT / f
        if p.exists():
            out.append(f"{f[:-4]}: `" + p.read_text().strip().splitlines()[-1] + "`")
    return ("nvidia-smi (name, sm MHz, max sm MHz, mem MHz, W, event reasons) around the "
            "captures -- " + "; ".join(out)) if out else "no clock record"


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
     f"Build: {build}", "", clocks_note(), "",
     "ncu serialises every launch and flushes caches: absolute times are cold-cache and",
     "un-overlapped (the graph runs the target forward, the wgrads and the priority update",
     "beside the critical chain); compare **shares**.",
     f"One steady-state update, {len(u)} launches, serialised sum {tot:.1f} us:", "",
     "| # | kernel | us | share |", "|---|---|---|---|"]
for i, (n, v) in enumerate(u):
    L.append(f"| {i} | `{n[:80]}` | {v:.2f} | {100 * v / tot:.1f}% |")
g = sum(v for n, v in u if "tc_gemm" in n)
conv1w = [v for n, v in u if "conv1_wgrad_u8" in n]
L += ["", f"tcgen05 GEMMs: {g:.1f} us = {100 * g / tot:.1f}% of the serialised update; "
      f"conv1 wgrad (the bench's roofline kernel): "
      + ", ".join(f"{v:.2f} us ({100 * v / tot:.1f}%)" for v in conv1w) + "."]
(PROF / f"{tag}_bench_launch_list.md").write_text("\n".join(L) + "\n")
shutil.copy(OUT / "launches_bench.csv", PROF / f"{tag}_bench_launches.csv")

# ------------------------------------------------------------- every kernel
metrics = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "l1tex__m_xbar2l1tex_read_bytes.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,"
           "launch__registers_per_thread,"
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio")
raw = subprocess.run(["ncu", "-i", str(OUT / "step_all.ncu-rep"), "--page", "raw", "--csv",
                      "--metrics", metrics], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1, "us": 1, "usecond": 1,
         "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3}


def val(r, n):
    return float(r[col[n]].replace(",", "")) * scale.get(units[col[n]], 1)


# eager launch order of one cfg4 update (agent._StepPlan.enqueue); the name
# fragment checks the label against the captured kernel
labels = [("sample+gather (batch 32)", "sample_gather"),
          ("IS weights (batch 32, tree stream)", "tree_sample"),
          ("conv1.fwd (batch 32, target)", ("conv1_tc", "FwdPol<unsigned char")),
          ("conv2.fwd (batch 32, target)", ("conv_tc_kernel<64, 3, 0", "conv_tc_kernel<64, 2, 0>", "FwdPol<float")),
          ("conv3.fwd (batch 32, target)", ("conv_tc_kernel<64, 3, 0", "conv_tc_kernel<64, 2, 0>", "FwdPol<float")),
          ("fc1.fwd (batch 32, target)", "lin_tc"),
          ("conv1.fwd (batch 64)", ("conv1_tc", "FwdPol<unsigned char")),
          ("conv2.fwd (batch 64)", ("conv_tc_kernel<64, 3, 0", "conv_tc_kernel<64, 2, 0>", "FwdPol<float")),
          ("conv3.fwd (batch 64)", ("conv_tc_kernel<64, 3, 0", "conv_tc_kernel<64, 2, 0>", "FwdPol<float")),
          ("fc1.fwd (batch 64)", "lin_tc"),
          ("duel.fwd+td (Q heads)", "head_q"), ("duel.dgrad+wgrad (TD block)", "head_td_bwd"),
          ("tree update (batch 32)", "tree_update"), ("fc1.wgrad (batch 32)", "lin_wgrad"),
          ("fc1.dgrad (batch 32)", "LinDgrad"), ("conv3.wgrad (batch 32)", "WgradPol<float"),
          ("conv3.dgrad (batch 32)", ("conv_tc_kernel<64, 3, 1", "conv_tc_kernel<64, 2, 1>", "ConvDgradPol")),
          ("conv2.wgrad (batch 32)", "WgradPol<float"),
          ("conv2.dgrad (batch 32)", ("conv_tc_kernel<32, 3, 1", "conv_tc_kernel<32, 2, 1>", "ConvDgradPol")),
          ("conv1.wgrad (batch 32)", "conv1_wgrad_u8"),
          ("rmsprop apply", "rms_apply")]
L = [f"# {tag} — every kernel of one learner update, `ncu --set full`", "",
     "Command: `ncu --profile-from-start off --set full --import-source on --clock-control none "
     "-o step_all python tools/profile_step.py` (eager launches of one cfg4 "
     "update, B = 32, after 5 warm-up updates).", "", f"Build: {build}", "", clocks_note(), "",
     "ncu flushes caches and serialises launches: DRAM bytes are cold-cache per launch.", "",
     "| # | phase | kernel | grid | us | DRAM rd+wr MB | L2->L1 MB | tensor % | SM thru % "
     "| long-sb stall/issue | regs |", "|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for i, r in enumerate(data):
    name = clean(r[col["Kernel Name"]])
    lab, frag = labels[i] if i < len(labels) else (f"kernel {i}", "")
    frags = frag if isinstance(frag, tuple) else (frag,)
    if frag and not any(f in name for f in frags):
        lab = f"kernel {i}"
    dr = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    traffic[lab] = {"dram_bytes": dr, "kernel": name, "us_ncu": val(r, "gpu__time_duration.sum")}
    L.append(
        f"| {i} | {lab} | `{name[:60]}` | {int(val(r, 'launch__grid_size'))} | "
        f"{val(r, 'gpu__time_duration.sum'):.2f} | {dr / 1e6:.3f} | "
        f"{val(r, 'l1tex__m_xbar2l1tex_read_bytes.sum') / 1e6:.2f} | "
        f"{float(r[col['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']]):.1f} | "
        f"{float(r[col['sm__throughput.avg.pct_of_peak_sustained_elapsed']]):.1f} | "
        f"{float(r[col['smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio']]):.2f} | "
        f"{int(val(r, 'launch__registers_per_thread'))} |")
(PROF / f"{tag}_step_kernels.md").write_text("\n".join(L) + "\n")
json.dump({"source": f"profiles/{tag}_step_kernels.md (ncu --set full, cold cache, "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch)",
           "kernels": traffic}, open(PROF / "roofline_traffic.json", "w"), indent=1)
print("\n".join(L[10:]))
