cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/phase.jsonl
for c in C2 C3; do timeout 300 python tools/phase_bench.py $c --reps 5 >> gpurun_out/phase.jsonl 2>>gpurun_out/phase.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor or fmm_small or c2" > gpurun_out/pytest_t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t.log
CMD="python tools/phase_bench.py C2 --reps 1"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:tensor_seed -c 1 -o gpurun_out/prof_seed $CMD > gpurun_out/ncu_seed.log 2>&1
echo "ncu rc=$?"
