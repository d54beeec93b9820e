# Round-end measurement refresh (one B200): bench line (ours + reference arm), the ncu launch list
# of a bench step, and one ncu --set full capture of the gather + three GEMM launches.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --profile > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:umma_gemm|gather_w' -c 4 \
  -o $O/full python bench.py --steps 1 --warmup 3 --profile > $O/ncu_full.log 2>&1; echo "full rc=$?"
tail -1 $O/bench.log | cut -c1-300
tail -1 $O/ref.log | cut -c1-300
