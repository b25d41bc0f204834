cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/s2lq.jsonl
for c in C2 C3 C4; do timeout 300 python tools/phase_bench.py $c --reps 5 >> gpurun_out/s2lq.jsonl 2>>gpurun_out/s2lq.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
