mkdir -p gpurun_out
for bn in 32 64; do for v in 0 1; do
  DQN_B200_LIN_DGRAD_BN=$bn DQN_B200_TMA_B=$v LIN_DGRAD_DUMP=gpurun_out/ld_${bn}_$v.pt timeout 300 python tools/lin_dgrad_check.py 2>&1 | tail -3 | sed "s/^/TMA_B=$v /"
done
python -c "import torch; a=torch.load('gpurun_out/ld_${bn}_0.pt'); b=torch.load('gpurun_out/ld_${bn}_1.pt'); print('BN $bn bit-identical', torch.equal(a,b))"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_tmab.log 2>&1; tail -2 gpurun_out/pytest_gpu_tmab.log | head -1
for v in 1 0 1 0 1 0; do DQN_B200_TMA_B=$v timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH TMA_B', '$v', round(d['value']), round(d['e2e']['value']))"; done
