# CTA-pair GEMMs after the per-warp accumulator release: parity, then A/B timing
set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
cp paper_2203_15565_b200/var_c22.so paper_2203_15565_b200/libpfc_gpu.so
timeout 300 python -m pytest tests/test_gpu_step.py -x -q -m gpu > gpurun_out/t_c22.log 2>&1; echo "c22 tests rc=$?"; tail -1 gpurun_out/t_c22.log
cp paper_2203_15565_b200/var_d2.so paper_2203_15565_b200/libpfc_gpu.so
timeout 300 python -m pytest tests/test_gpu_diag.py -x -q -m gpu > gpurun_out/t_d2.log 2>&1; echo "d2 tests rc=$?"; tail -1 gpurun_out/t_d2.log
timeout 300 python profiles/micro/diag_time.py 2>&1 | tail -1 | sed "s/^/d2 /"
timeout 300 python profiles/micro/mics_time.py 2>&1 | tail -1 | sed "s/^/d2 /"
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
timeout 300 python profiles/micro/diag_time.py 2>&1 | tail -1 | sed "s/^/main /"
timeout 300 python profiles/micro/mics_time.py 2>&1 | tail -1 | sed "s/^/main /"
bash profiles/micro/varbench.sh var_main var_c21 var_c12 var_c22
