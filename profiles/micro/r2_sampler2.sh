set -u
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_step.py -q -x -k "sampler or errors or filter_all or pinned or async or northstar" > gpurun_out/r2/t_sampler.log 2>&1; echo "sampler tests rc=$?"; tail -3 gpurun_out/r2/t_sampler.log
bash profiles/micro/varcfg.sh var_old var_new
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2/t_all.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2/t_all.log
