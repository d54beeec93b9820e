# A/B of the diagnostics call (apcs / amncs at 2M) between library variants
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for rep in 1 2; do
  for v in "$@"; do
    cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/vd.log 2>&1
    VNAME=$v python -c "import json,os;d=json.loads(open('gpurun_out/vd.log').read().strip().splitlines()[-1]);g=d['diagnostics'];print(os.environ['VNAME'], round(d['ms_per_step'],4), 'diag', round(g['ms_per_call'],3), g['apcs'], g['amncs'])"
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
