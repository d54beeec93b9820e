set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for v in var_c22 var_c21; do
  cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
  timeout 300 python -m pytest tests/test_gpu_step.py -x -q -m gpu > gpurun_out/t_$v.log 2>&1; echo "$v tests rc=$?"; tail -3 gpurun_out/t_$v.log
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
bash profiles/micro/varbench.sh var_c11 var_c21 var_c12 var_c22
