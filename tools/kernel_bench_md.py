"""Render tools/kernel_bench.py JSON as the committed markdown table.

usage: python tools/kernel_bench_md.py gpurun_out/kernel_bench.json profiles/<tag>_kernel_bench.md "<title>"
"""
import json
import sys

src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3]
d = json.load(open(src))
L = [f"# {title}", "",
     "Command: `python tools/kernel_bench.py` on one B200 (device time from CUDA events around",
     "CUDA-graph replays of each call, no host launch overhead).  Peaks from MEASURED_PEAKS.json:",
     f"HBM copy {d['hbm_peak_gbps']:.1f} GB/s, dense bf16 {d['bf16_peak_tflops']:.1f} TFLOP/s (the GEMMs",
     "compute 3xTF32: their implementation tensor work is 2-3x the algorithmic FLOPs below).", "",
     f"Clocks during the run (nvidia-smi sampler of bench.py): {d.get('clocks')}", "",
     "| kernel | us | algorithmic | achieved | of peak | note |", "|---|---|---|---|---|---|"]
for r in d["kernels"]:
    if "gbps" in r:
        alg = f"{r['algorithmic_bytes'] / 1e6:.2f} MB"
        ach = f"{r['gbps']:.0f} GB/s"
        frac = f"{100 * r['frac_hbm']:.1f}% HBM"
    else:
        alg = f"{r['algorithmic_flop'] / 1e9:.2f} GFLOP"
        ach = f"{r['tflops']:.1f} TFLOP/s"
        frac = f"{100 * r['frac_bf16']:.2f}% bf16"
    L.append(f"| {r['kernel']} | {r['us']:.2f} | {alg} | {ach} | {frac} | {r['note']} |")
open(dst, "w").write("\n".join(L) + "\n")
print("\n".join(L))
