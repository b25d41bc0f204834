cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/win_var.jsonl gpurun_out/win_par.jsonl
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1; do CYLFMM_P2P_VARIANT=$v timeout 600 python tools/phase_bench.py C5 --reps 2 >> gpurun_out/win_var.jsonl 2>>gpurun_out/win_var.err; done
timeout 900 python tools/run_config.py C5 --sample 96 --reps 1 >> gpurun_out/win_par.jsonl 2>>gpurun_out/win_var.err
