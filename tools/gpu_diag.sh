cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python tools/diag_c5c.py > gpurun_out/diag_c5.log 2>&1; echo "rc=$?" >> gpurun_out/diag_c5.log
