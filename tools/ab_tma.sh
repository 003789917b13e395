mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log | head -1
for v in 1 0; do DQN_B200_TMA_GATHER=$v python tools/kernel_bench.py gpurun_out/kb_tma$v.json 2>&1 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA', '$v', d['kernel'], round(d['us'],2), round(d['gbps']), round(d['frac_hbm'],3))"; done
for v in 1 0 1 0; do DQN_B200_TMA_GATHER=$v python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH TMA', '$v', round(d['value']), round(d['e2e']['value']))"; done
