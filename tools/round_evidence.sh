#!/bin/bash
# The rest of a round's evidence beside tools/profile_job.sh (one GPU):
# the GPU suite, smoke, the lockstep soak, the parity report, the bench line
# of every config, the reference arm, and a graph timeline.  Outputs under
# gpurun_out/$TAG.
TAG=${TAG:-r02}
O=gpurun_out/$TAG
mkdir -p $O/configs $O/parity
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 300 python tools/soak.py 20000 > $O/soak.txt 2>&1
DQN_PARITY_REPORT=$O/parity timeout 1500 python -m pytest tests/test_gpu_lockstep.py \
  tests/test_gpu_parity_1m.py -q -s -p no:cacheprovider > $O/parity/pytest_tail.log 2>&1
timeout 600 python bench.py > $O/configs/bench.json 2> $O/configs/bench.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --no-cpu > $O/configs/bench_$c.json 2>> $O/configs/bench.err
done
timeout 600 python bench.py --mode dp --no-cpu > $O/configs/bench_dp1.json 2>> $O/configs/bench.err
timeout 600 python bench.py --impl reference > $O/configs/bench_ref.json 2>> $O/configs/bench.err
timeout 300 python tools/graph_timeline.py --cap 1000000 --reps 5 > $O/graph_timeline.txt 2>&1
