# Round 2: parity subset after the stats/finalize changes, a bench line, the bulk-copy update
# microbenchmark, ncu launch list and a source-level capture of the small per-step kernels.
set -u
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x -k "step or edges or multirank or soak" > $O/t_small.log 2>&1; echo "tests rc=$?"; tail -2 $O/t_small.log
timeout 600 python bench.py --no-cpu --no-diag > $O/bench_small.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench_small.log | cut -c1-250
timeout 300 ./profiles/micro/bulkupd > $O/bulkupd.log 2>&1; echo "bulkupd rc=$?"; cat $O/bulkupd.log
timeout 300 ./profiles/micro/rowupd > $O/rowupd.log 2>&1; echo "rowupd rc=$?"; grep -i "dW ownership\|ring emulation" $O/rowupd.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --profile > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:positives|draws|walk|finalize|local_sums' -c 6 \
  -o $O/small python bench.py --steps 1 --warmup 3 --profile > $O/ncu_small.log 2>&1; echo "ncu small rc=$?"
