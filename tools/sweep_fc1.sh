run() { env "$@" timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), round(d['e2e']['value']))"; }
for r in 1 2; do run X=0; run DQN_B200_LIN_DGRAD_BN=64; run DQN_B200_DGRAD_CAP=8; run DQN_B200_DGRAD_CAP=32; done
