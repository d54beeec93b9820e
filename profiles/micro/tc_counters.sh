# Tensor-pipe counter calibration (pure-MMA microkernel of known FLOP rate) and the same
# counters for the step's three GEMMs (one ncu pass over one bench step).
set -u
O=gpurun_out/r2
mkdir -p $O
M="gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tc.sum,TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,sm__mem_tensor_reads_op_utcmma_matrix_c.sum"
./profiles/micro/mma_rate 20000 > $O/mma_rate.log 2>&1; cat $O/mma_rate.log
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $O/mma_rate_ncu.csv ./profiles/micro/mma_rate 20000 > /dev/null 2>&1; echo "ncu micro rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:umma_gemm -c 3 --csv --log-file $O/gemm_tc_ncu.csv python bench.py --steps 1 --warmup 3 --profile > /dev/null 2>&1; echo "ncu gemms rc=$?"
