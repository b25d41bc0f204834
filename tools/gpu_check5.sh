cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python tools/diag_stations.py 16 65 > gpurun_out/diag_st.json 2>&1
timeout 300 python tools/diag_stations.py 8 17 >> gpurun_out/diag_st.json 2>&1
rm -f gpurun_out/phase.jsonl
for c in C2 C3; do timeout 300 python tools/phase_bench.py $c --reps 5 >> gpurun_out/phase.jsonl 2>>gpurun_out/phase.err; done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
