# A/B of library variants at the 10M / B = 2048 and 2M / B = 1024 configurations
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for rep in 1 2; do
  for cfg in "--classes 10000000 --batch 2048" ""; do
    for v in "$@"; do
      cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
      timeout 600 python bench.py $cfg --steps 10 --warmup 3 --no-cpu --no-diag --no-e2e > gpurun_out/v10.log 2>&1
      VNAME=$v CFG="$cfg" python -c "import json,os;d=json.loads(open('gpurun_out/v10.log').read().strip().splitlines()[-1]);print(os.environ['VNAME'], repr(os.environ['CFG']), round(d['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
    done
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
