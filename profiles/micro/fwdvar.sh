# logits epilogue variants: warpgroups (NWG), operand stages, E^T staging buffers per warp
set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_w4s4b1.so paper_2203_15565_b200/libpfc_gpu.so
timeout 300 python -m pytest tests/test_gpu_step.py -x -q -m gpu > gpurun_out/t_w4.log 2>&1; echo "w4s4b1 tests rc=$?"; tail -1 gpurun_out/t_w4.log
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
bash profiles/micro/varbench.sh var_cur var_w4s4b1 var_w2s4b1 var_w4s3b2
