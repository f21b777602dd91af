# quick GPU check: gpu tests, fwd/bp bench stages, optional ncu metrics of one kernel ($1 regex)
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FWD', d['value'], d['e2e']['value'], d['stages_ms_per_step'])"
python bench.py --direction back --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BP', d['value'], d['e2e']['value'], d['stages_ms_per_step'])"
if [ -n "$1" ]; then
  mkdir -p gpurun_out/quick
  ncu --profile-from-start off --clock-control none -k regex:"$1" -c ${3:-2} --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct --csv python tools/profile_step.py ${2:-} 2>/dev/null | grep -v "^==" | tail -20
fi
