# Round-2 measurement refresh (one B200): bench lines (north star + the other BASELINE configs,
# tf32 mode), the reference arm, the ncu launch list of a north-star step and one --set full
# capture of the gather + three GEMM launches.
set -u
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --precision tf32 --no-cpu > $O/bench_tf32.log 2>&1; echo "bench tf32 rc=$?"
for cfg in "--classes 10000 --batch 128 --shards 1" "--classes 360000 --shards 8" \
           "--classes 360000 --shards 8 --r 1.0 --margin cosface" "--classes 10000000 --batch 2048 --shards 8 --no-cpu"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 900 python bench.py $cfg --no-diag > $O/bench_$tag.log 2>&1; echo "bench $cfg rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --profile > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:umma_gemm|gather_w' -c 4 \
  -o $O/full python bench.py --steps 1 --warmup 3 --profile > $O/ncu_full.log 2>&1; echo "full rc=$?"
