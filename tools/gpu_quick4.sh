cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/phase.jsonl
for c in C2 C3 C4 C5; do timeout 600 python tools/phase_bench.py $c --reps 3 >> gpurun_out/phase.jsonl 2>>gpurun_out/phase.err; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
