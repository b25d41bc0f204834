#!/bin/bash
# One gpurun call: the parameter-selection GPU tests and the depth sweep against the cost model.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_select_params.py -m gpu -x -q > gpurun_out/pytest_select.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_select.log
timeout 900 python tools/depth_sweep.py C2 C3 C4 > gpurun_out/depth_sweep.jsonl 2> gpurun_out/depth_sweep.err; echo "sweep rc=$?"
