set -u
for v in var_half var_head var_half; do
  cp paper_2203_15565_b200/$v.so paper_2203_15565_b200/libpfc_gpu.so
  echo "== $v"; CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_step.py -q -x -k "glint360k_k8 and sampler" 2>&1 | grep -E "passed|failed|Error at" | head -3
done
