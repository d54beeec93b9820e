# bench.py at the other BASELINE configurations (one B200): Glint360K, 10M/B=2048, 2M K=1
set -u
for a in "--classes 360000" "--classes 10000000 --batch 2048" "--classes 2000000 --shards 1"; do
  timeout 600 python bench.py $a --no-cpu --no-diag 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$a', round(d['value']), 'samples/s', round(d['ms_per_step'],4), 'ms; e2e', round(d['e2e']['value']), d['config']['workload'])"
done
