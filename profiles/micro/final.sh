# Full GPU test suite, then the round-end measurement refresh (profiles/micro/refresh.sh)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
bash profiles/micro/refresh.sh
