# dW update epilogue timing probes (PFC_DW_EXP=1..4 in epilogues.cuh) against the product build,
# plus the guard-region tests.
set -u
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_guard.py -q -x > gpurun_out/r2/t_guard.log 2>&1; echo "guard tests rc=$?"; tail -15 gpurun_out/r2/t_guard.log
cp paper_2203_15565_b200/libpfc_gpu.so paper_2203_15565_b200/var_main.so
bash profiles/micro/varbench.sh var_main var_exp1 var_exp2 var_exp3 var_exp4
