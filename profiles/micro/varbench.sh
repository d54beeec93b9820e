# A/B timing of library variants: bash profiles/micro/varbench.sh var_a var_b ... (each
# paper_2203_15565_b200/<name>.so is swapped in for libpfc_gpu.so, two bench runs each)
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for v in "$@"; do
  cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$v.log 2>&1
    VNAME=$v python -c "import json,os;d=json.loads(open('gpurun_out/bench_'+os.environ['VNAME']+'.log').read().strip().splitlines()[-1]);print(os.environ['VNAME'], round(d['value']), round(d['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
