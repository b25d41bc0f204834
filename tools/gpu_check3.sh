cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python tools/diag_stations.py 16 65 > gpurun_out/diag_st.json 2>&1
timeout 300 python tools/diag_stations.py 6 5 >> gpurun_out/diag_st.json 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/run_config.py C5 --sample 64 > gpurun_out/cfg_C5.json 2>&1
timeout 600 python tools/run_config.py C4 --sample 64 > gpurun_out/cfg_C4.json 2>&1
