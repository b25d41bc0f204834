cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/s2l_var.jsonl
for v in 0 1 2; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py C2 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
for v in 0 1 2; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py C3 --reps 3 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
for v in 0 1 2; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py C4 --reps 3 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
