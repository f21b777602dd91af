# repeat the backprojector bench line
for i in 1 2 3; do
  python bench.py --direction back --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BP', d['value'], d['e2e']['value'])"
done
