set -u
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_edges.py -q -x > gpurun_out/r2/t_dw.log 2>&1; echo "step tests rc=$?"; tail -2 gpurun_out/r2/t_dw.log
bash profiles/micro/varbench.sh var_main var_cap4 var_cap3 var_exp6 var_main
