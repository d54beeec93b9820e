# Round-2 measurement pass (one B200): compute-sanitizer on small configs, bench lines for the
# BASELINE configs, the ncu launch list of a north-star step and one ncu --set full capture.
set -u
O=gpurun_out/r2
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for case in bf16 fp32 loopback; do
    timeout 600 $CS --tool $tool --error-exitcode 9 --print-limit 50 python profiles/sanitize_step.py $case \
      > $O/sanitize_${tool}_${case}.log 2>&1; echo "sanitize $tool $case rc=$?"; tail -2 $O/sanitize_${tool}_${case}.log
  done
done
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench.log | cut -c1-400
for cfg in "--classes 10000 --batch 128 --shards 1" "--classes 360000 --shards 8" \
           "--classes 360000 --shards 8 --r 1.0 --margin cosface" "--classes 10000000 --batch 2048 --shards 8 --no-cpu"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 900 python bench.py $cfg --no-diag > $O/bench_$tag.log 2>&1; echo "bench $cfg rc=$?"; tail -1 $O/bench_$tag.log | cut -c1-300
done
