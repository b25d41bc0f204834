cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/s2l_var.jsonl gpurun_out/s2l_par.jsonl
for v in 0 1; do
  for c in C2 C3 C4; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/phase_bench.py $c --reps 4 >> gpurun_out/s2l_var.jsonl 2>>gpurun_out/s2l_var.err; done
  for c in C2 C3; do CYLFMM_S2L_VARIANT=$v timeout 300 python tools/run_config.py $c --sample 256 --reps 1 >> gpurun_out/s2l_par.jsonl 2>>gpurun_out/s2l_var.err; done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
