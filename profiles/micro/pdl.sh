# PDL on/off A/B at three sizes, the streaming-store dW probe, and the GPU parity tests.
set -u
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2/t_pdl.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2/t_pdl.log
for cfg in "" "--classes 360000" "--classes 10000 --batch 128 --shards 1"; do
  for pdl in "" "--no-pdl"; do
    timeout 300 python bench.py $cfg $pdl --no-cpu --no-diag > gpurun_out/r2/b.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/r2/b.log').read().strip().splitlines()[-1]);print('$cfg $pdl', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
  done
done
bash profiles/micro/varbench.sh var_exp5
