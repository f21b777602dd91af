set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -5
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FWD', d['value'], d['e2e']['value'], d['stages_ms_per_step'])"
python bench.py --direction back --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BP', d['value'], d['e2e']['value'], d['stages_ms_per_step'])"
