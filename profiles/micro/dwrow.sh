# dW row-major epilogue variants (DwRowEpi) vs the current epilogue (var_cur)
set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_r8s2.so paper_2203_15565_b200/libpfc_gpu.so
timeout 240 python -m pytest tests/test_gpu_step.py -x -q -m gpu -k "step_matches or northstar or repeatable or graph_replay" > gpurun_out/t_row.log 2>&1; echo "row tests rc=$?"; tail -1 gpurun_out/t_row.log
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
bash profiles/micro/varbench.sh var_cur var_r8s2 var_r6s2 var_r4s3
