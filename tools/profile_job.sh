#!/bin/bash
# One GPU job: full default bench line, the ncu launch list of the bench
# command (cold-cache serialised per-launch times), and an ncu --set full
# capture of every tcgen05 GEMM of one eager learner update.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu \
  > gpurun_out/ncu_launch.log 2>&1
python tools/profile_step.py > gpurun_out/plain_step.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:tc_gemm -o gpurun_out/step_gemms python tools/profile_step.py \
  > gpurun_out/ncu_gemms.log 2>&1
tail -2 gpurun_out/ncu_gemms.log
timeout 600 python tools/kernel_bench.py gpurun_out/kernel_bench.json > gpurun_out/kb.log 2>&1
tail -1 gpurun_out/kb.log
