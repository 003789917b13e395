mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in 0 1; do DQN_B200_PRIO=$v python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/bench_p$v.log 2>&1; tail -1 gpurun_out/bench_p$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('PRIO', '$v', 'VALUE', d['value'], 'E2E', d['e2e']['value'])"; done
