# same-box A/B of whole-library variants at three sizes (device path + e2e), then ncu of the sampler
set -u
mkdir -p gpurun_out/r2
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for cfg in "" "--classes 360000" "--classes 10000 --batch 128 --shards 1"; do
  for v in "$@"; do
    cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
    timeout 300 python bench.py $cfg --no-cpu --no-diag > gpurun_out/r2/ab.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/r2/ab.log').read().strip().splitlines()[-1]);print('$v $cfg', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))"
  done
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:fill_kernel|walk_kernel|mark_kernel' -c 3 \
  -o gpurun_out/r2/samp python bench.py --steps 1 --warmup 3 --profile > gpurun_out/r2/ncu_samp.log 2>&1; echo "ncu rc=$?"
