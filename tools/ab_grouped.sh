mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in 1 0 1 0; do DQN_B200_GROUPED_FWD=$v python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('GROUPED', '$v', 'VALUE', d['value'], 'E2E', d['e2e']['value'])"; done
