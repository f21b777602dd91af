# A/B experiments: bp bench under spread-warp overrides
python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for w in 2 4; do
  CBN_SPREAD_W=$w python bench.py --direction back --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('W=$w', d['value'], d['stages_ms_per_step']['bp_spread'])"
done
