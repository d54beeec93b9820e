# ncu --set full of the three sampler kernels and the small fixed-cost kernels (one north-star step)
set -u
mkdir -p gpurun_out/r2s
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:mark_kernel|fill_kernel|walk_kernel|finalize|xs_kernel' -c 12 \
  -o gpurun_out/r2s/small python bench.py --steps 1 --warmup 3 --profile --no-cpu --no-e2e --no-diag > gpurun_out/r2s/ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2s/launches_10k.csv python bench.py --classes 10000 --batch 128 --shards 1 --steps 2 --warmup 3 --profile --no-cpu --no-diag > gpurun_out/r2s/ncu10k.log 2>&1; echo "launches rc=$?"
