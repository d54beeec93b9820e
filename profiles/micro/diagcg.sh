# A/B of the diagnostics / mics screening GEMMs: one CTA per tile (var_d1) vs CTA pairs (var_d2)
set -u
mkdir -p gpurun_out
cp paper_2203_15565_b200/libpfc_gpu.so /tmp/main.so
for v in var_d2 var_d1; do
  cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
  timeout 300 python -m pytest tests/test_gpu_diag.py -x -q -m gpu > gpurun_out/t_$v.log 2>&1; echo "$v diag tests rc=$?"; tail -2 gpurun_out/t_$v.log
  timeout 300 python profiles/micro/diag_time.py 2>&1 | tail -2 | sed "s/^/$v /"
  timeout 300 python profiles/micro/mics_time.py 2>&1 | tail -1 | sed "s/^/$v /"
done
cp /tmp/main.so paper_2203_15565_b200/libpfc_gpu.so
