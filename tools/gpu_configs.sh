# per-config bench lines (DESIGN.md measurements table)
mkdir -p gpurun_out/configs
for c in 0 3; do
  for d in forward back; do
    timeout 900 python bench.py --config $c --direction $d --no-cpu-baseline > gpurun_out/configs/c${c}_${d}.json 2> gpurun_out/configs/c${c}_${d}.err
    python -c "import json; d=json.loads(open('gpurun_out/configs/c${c}_${d}.json').read().strip().splitlines()[-1]); print('cfg $c $d', d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))" || tail -3 gpurun_out/configs/c${c}_${d}.err
  done
done
