# logits GEMM in column chunks whose gathers overlap the previous chunk's GEMM (PFC_FWD_CHUNKS)
set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_ch4.so paper_2203_15565_b200/libpfc_gpu.so
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_fuzz.py -x -q -m gpu > gpurun_out/t_ch4.log 2>&1; echo "ch4 tests rc=$?"; tail -1 gpurun_out/t_ch4.log
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
bash profiles/micro/varbench.sh var_ch1 var_ch2 var_ch4 var_ch8 var_ch1
