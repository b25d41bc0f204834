cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/l2p.jsonl
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in C2 C3 C4 C5; do timeout 600 python tools/phase_bench.py $c --reps 3 >> gpurun_out/l2p.jsonl 2>>gpurun_out/l2p.err; done
timeout 900 python tools/run_config.py C5 --sample 96 > gpurun_out/cfg_C5.json 2> gpurun_out/cfg_C5.err
