set -u
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "step_matches or northstar or repeatable or graph" > gpurun_out/r2/t_fwd.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2/t_fwd.log
bash profiles/micro/varbench.sh "$@"
