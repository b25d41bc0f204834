cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/p2pw_var.jsonl gpurun_out/p2pw_par.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm or near" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for v in 0 2; do
  for c in C2 C3 C4; do CYLFMM_P2P_VARIANT=$v timeout 300 python tools/phase_bench.py $c --reps 4 >> gpurun_out/p2pw_var.jsonl 2>>gpurun_out/p2pw_var.err; done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"p2p" -s 2 -c 1 \
   -o gpurun_out/p2pw_c2 python tools/phase_bench.py C2 --reps 1 > gpurun_out/ncu_p2pw.log 2>&1; echo "rc=$?"
