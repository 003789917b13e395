mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), round(d['e2e']['value']), ' '.join('%s.%s=%.1f'%(x['layer'],x['phase'],x['us']) for x in d['layer_phases'] if x['layer'] in ('conv1',) ))"; }
for r in 1 2; do
run X=0
for c in 16 24 48 64; do run DQN_B200_WGRAD_CAP_U8=$c; done
for c in 2 8; do run DQN_B200_CDGRAD_CAP=$c; done
for c in 128 512; do run DQN_B200_FWD_KLEN=$c; done
done
