cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in C3 C4; do timeout 600 python tools/run_config.py $c --sample 32 --reps 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; done
