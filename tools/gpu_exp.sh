# A/B experiments: backprojector Grangeat gather views per CTA
for vg in 4 8 16; do
  CBN_GR_VG=$vg python bench.py --direction back --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('VG=$vg', d['value'], d['stages_ms_per_step']['grangeat_forward'])"
done
