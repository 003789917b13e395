mkdir -p gpurun_out
python tools/tc_check.py > gpurun_out/tc_check.log 2>&1; tail -1 gpurun_out/tc_check.log
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', d['value'], 'E2E', d['e2e']['value']); print(' '.join('%s.%s=%.1f'%(x['layer'],x['phase'],x['us']) for x in d['layer_phases']))"
