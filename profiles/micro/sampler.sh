# bitmap sampler: sampler parity (all BASELINE configs), full GPU suite, bench A/B at three sizes
set -u
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_step.py -q -x -k "sampler or errors or filter_all or pinned or async" > gpurun_out/r2/t_sampler.log 2>&1; echo "sampler tests rc=$?"; tail -15 gpurun_out/r2/t_sampler.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2/t_all.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/r2/t_all.log
for cfg in "" "--classes 360000" "--classes 10000 --batch 128 --shards 1"; do
  timeout 300 python bench.py $cfg --no-cpu --no-diag > gpurun_out/r2/b.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/r2/b.log').read().strip().splitlines()[-1]);print('$cfg', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2/launches2.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/r2/ncu_launch2.log 2>&1; echo "launches rc=$?"
