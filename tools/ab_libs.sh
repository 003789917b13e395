#!/bin/bash
# Interleaved learner A/B of product builds (libdqn_b200.so and every
# libdqn_b200_alt*.so beside it) plus the graph timeline of the first; outputs
# under gpurun_out/ab/.  usage: bash tools/ab_libs.sh [rounds] [pytest -k expr]
R=${1:-3}
O=gpurun_out/ab
mkdir -p $O
rm -f $O/ab.log
if [ -n "$2" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$2" -p no:cacheprovider > $O/test.log 2>&1; fi
for r in $(seq $R); do
  for L in libdqn_b200.so $(cd paper_1804_05834_b200 && ls libdqn_b200_alt*.so); do
    DQN_B200_LIB=$PWD/paper_1804_05834_b200/$L timeout 300 python tools/learner_ab.py --ct=0 --rounds 1 \
      --steps 3000 2>&1 | tail -1 | sed "s/^/$L /" >> $O/ab.log
  done
done
DQN_B200_LIB=$PWD/paper_1804_05834_b200/libdqn_b200.so timeout 300 python tools/graph_timeline.py \
  --cap 1000000 --reps 5 > $O/timeline.txt 2>&1
