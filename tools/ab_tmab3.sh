mkdir -p gpurun_out
for v in 1 0; do DQN_B200_TMA_B_CONV=$v timeout 300 python tools/conv_dgrad_check.py 2>&1 | tail -1 | sed "s/^/CONV_TMA=$v /"; done
for v in 1 0; do DQN_B200_TMA_B=$v timeout 300 python tools/lin_dgrad_check.py 2>&1 | tail -2 | sed "s/^/TMA_B=$v /"; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_tmab.log 2>&1; tail -3 gpurun_out/pytest_gpu_tmab.log | head -2
for i in 1 2 3; do for cfg in "1 1" "1 0" "0 0"; do set -- $cfg; DQN_B200_TMA_B=$1 DQN_B200_TMA_B_CONV=$2 timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH TMA_B $1 CONV $2', round(d['value']), round(d['e2e']['value']))"; done; done
