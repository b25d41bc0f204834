cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in C3 C5; do timeout 900 python tools/run_config.py $c --sample 96 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; done
for v in 0 1 2 3; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py C2 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
for v in 0 1 2; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py C4 --reps 3 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
