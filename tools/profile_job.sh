#!/bin/bash
# One GPU job (round 2): clocks, the ncu launch list of the bench command
# (cold-cache serialised per-launch times), an ncu --set full capture of
# every kernel of one eager learner update, the large-batch kernel bench.
# Outputs under gpurun_out/$TAG (default r02).
TAG=${TAG:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.active \
  --format=csv > $O/clocks_before.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu \
  > $O/ncu_launch.log 2>&1
python tools/profile_step.py > $O/plain_step.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o $O/step_all python tools/profile_step.py > $O/ncu_step.log 2>&1
tail -2 $O/ncu_step.log
timeout 600 python tools/kernel_bench.py $O/kernel_bench.json > $O/kb.log 2>&1
tail -1 $O/kb.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.active \
  --format=csv > $O/clocks_after.csv
