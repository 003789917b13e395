mkdir -p gpurun_out
for i in 1 2; do
python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DEFAULT', d['value'], d['e2e']['value'], d['steps'], d['clocks'])"
python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NOCPU', d['value'], d['e2e']['value'], d['steps'])"
done
