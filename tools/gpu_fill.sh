cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/fill.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor or fmm_small" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for t in 256 128 64 32; do
  for c in C2 C3 C4; do CYLFMM_FILL_THREADS=$t timeout 300 python tools/phase_bench.py $c --reps 4 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print('threads=$t', d['config'], d['ms_tensor'])" >> gpurun_out/fill.txt; done
  CYLFMM_FILL_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('threads=$t bench', d['ms_per_step'])" >> gpurun_out/fill.txt
done
