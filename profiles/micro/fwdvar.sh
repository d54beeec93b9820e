set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_n4s3.so paper_2203_15565_b200/libpfc_gpu.so
timeout 300 python -m pytest tests/test_gpu_step.py -x -q -m gpu > gpurun_out/t_n4s3.log 2>&1; echo "n4s3 tests rc=$?"; tail -2 gpurun_out/t_n4s3.log
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
bash profiles/micro/varbench.sh var_main var_n4s3 var_n2s3
