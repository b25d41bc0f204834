#!/bin/bash
# One gpurun iteration: GPU tests (optional) and the C2..C5 full-size configs with oracle parity.
#   tools/gpu_iter.sh [tests] [configs...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
if [ "$1" = "tests" ]; then
  shift
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
for c in "$@"; do
  timeout 1200 python tools/run_config.py $c --sample 96 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
  cat gpurun_out/cfg_$c.json; tail -3 gpurun_out/cfg_$c.err
done
