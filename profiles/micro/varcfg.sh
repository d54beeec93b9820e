# A/B timing of library variants at three sizes (2M north star, 360k, 10k):
#   bash profiles/micro/varcfg.sh var_a var_b ...  (paper_2203_15565_b200/<name>.so swapped in)
set -u
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for rep in 1 2; do
  for cfg in "" "--classes 360000" "--classes 10000 --batch 128 --shards 1"; do
    for v in "$@"; do
      cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
      timeout 300 python bench.py $cfg --steps 30 --warmup 5 --no-cpu --no-diag > gpurun_out/vb.log 2>&1
      VNAME=$v CFG="$cfg" python -c "import json,os;d=json.loads(open('gpurun_out/vb.log').read().strip().splitlines()[-1]);print(os.environ['VNAME'], repr(os.environ['CFG']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k:round(x['ms'],4) for k,x in d['phases_ms'].items()})"
    done
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
