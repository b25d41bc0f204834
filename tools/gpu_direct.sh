cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/direct_speedup.py C2 C3 > gpurun_out/speedup.jsonl 2> gpurun_out/speedup.err
CYLFMM_P2P_VARIANT=1 timeout 900 python tools/direct_speedup.py C2 >> gpurun_out/speedup.jsonl 2>> gpurun_out/speedup.err
