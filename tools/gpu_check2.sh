cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMD="python tools/run_config.py C5 --no-oracle --reps 1 --sample 8"
timeout 600 $CMD > gpurun_out/c5_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/c5_launches.csv $CMD > gpurun_out/c5_ncu.log 2>&1
echo "ncu rc=$?"
