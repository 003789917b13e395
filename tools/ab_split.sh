mkdir -p gpurun_out
for i in 1 2; do for v in "1 32" "1 64" "1 90" "0 64"; do set -- $v; DQN_B200_SPLIT_APPLY=$1 DQN_B200_RMS_SPLIT_BLOCKS=$2 timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH SPLIT $1 BLOCKS $2', round(d['value']), round(d['e2e']['value']))"; done; done
