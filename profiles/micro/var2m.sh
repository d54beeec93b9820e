# A/B at the north star only, 4 alternating repetitions of 50 steps
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for rep in 1 2 3 4; do
  for v in "$@"; do
    cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
    timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-diag > gpurun_out/v2.log 2>&1
    VNAME=$v python -c "import json,os;d=json.loads(open('gpurun_out/v2.log').read().strip().splitlines()[-1]);print(os.environ['VNAME'], round(d['ms_per_step'],4), round(d['phases_ms']['dw_update_gemm']['ms'],4))"
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
