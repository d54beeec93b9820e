# A/B of library variants in the tf32 mode at the north star
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for rep in 1 2; do
  for v in "$@"; do
    cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
    timeout 600 python bench.py --precision tf32 --steps 10 --warmup 3 --no-cpu --no-diag --no-e2e > gpurun_out/vt.log 2>&1
    VNAME=$v python -c "import json,os;d=json.loads(open('gpurun_out/vt.log').read().strip().splitlines()[-1]);print(os.environ['VNAME'], round(d['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
