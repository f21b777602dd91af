python -m pytest tests -q -m gpu -x 2>&1 | tail -1
python bench.py --config 4 --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4', d['value'], d['e2e']['value'], d['stages_ms_per_step'], d['config'].get('plan_s'))"
